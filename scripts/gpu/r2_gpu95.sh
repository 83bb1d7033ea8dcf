set -x
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_r2w.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_r2w.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2w.json 2> gpurun_out/bench_r2w.err; echo bench_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r2w.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_r2w.log 2>&1; echo ncu1_rc=$?
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dram_step_s26_r2w.csv python scripts/fused_step.py 26 2 > gpurun_out/ncu_dram_r2w.log 2>&1; echo ncu2_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count_vhub -c 1 -o gpurun_out/vhub_final_w python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo ncu3_rc=$?
