set -x
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_r2q.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_r2q.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2q.json 2> gpurun_out/bench_r2q.err; echo bench_rc=$?
tail -2 gpurun_out/bench_r2q.err
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dram_step_s26_r2q.csv python scripts/fused_step.py 26 2 > gpurun_out/ncu_dram_r2q.log 2>&1; echo ncu_rc=$?
