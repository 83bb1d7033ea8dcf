timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree or headline or huge_rmat" 2>&1 | tail -2
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
TC_LIB_PATH=variants/lib_hubunfused.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/hubfused.csv -k regex:"k_count_hub" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
