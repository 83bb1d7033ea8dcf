timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree or headline or prebuilt or huge_rmat" 2>&1 | tail -2
timeout 600 python scripts/ab_opts.py rmat26 7 "" "vhub_async=0" "" "vhub_async=0" 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/vhub_async.csv -k regex:"k_count_vhub" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
