# shard calibration data; staged copy threads
python scripts/shard_calib.py rmat26 > gpurun_out/shard_calib_r2f.jsonl 2> gpurun_out/shard_calib_r2f.err; echo calib_rc=$?
tail -2 gpurun_out/shard_calib_r2f.err
for t in 8 12 16; do echo "copy_threads=$t"; TC_COPY_THREADS=$t python scripts/pageable_e2e.py 26 2>&1 | grep pageable; done
