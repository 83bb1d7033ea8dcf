timeout 400 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
TC_LIB_PATH=variants/lib_b16w8.so timeout 400 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/vhub_e16.csv -k regex:"k_count_vhub" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
