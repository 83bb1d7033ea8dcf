set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_s26.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --csv -k regex:'k_count_|k_classify|k_range_init|k_vin_' --log-file gpurun_out/dram_count_s26.csv python scripts/fused_step.py 26 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_count_vmajor' -c 1 -o gpurun_out/vmajor_full_s26 python scripts/fused_step.py 26 1 > /dev/null 2>&1
tail -c 3000 gpurun_out/bench_r01b.json
