python scripts/shard_calib.py rmat26 > gpurun_out/shard_calib_r2j.jsonl 2> gpurun_out/shard_calib_r2j.err; echo rc=$?; tail -3 gpurun_out/shard_calib_r2j.err
python scripts/shard_calib.py rmat24 > gpurun_out/shard_calib24_r2j.jsonl 2>> gpurun_out/shard_calib_r2j.err; echo rc=$?
