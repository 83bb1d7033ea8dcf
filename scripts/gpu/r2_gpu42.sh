TC_LIB_PATH=variants/lib_hubminb5.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
TC_LIB_PATH=variants/lib_hubminb5.so timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/hubminb5.csv -k regex:"k_count_hub" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
