timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree or headline or prebuilt or huge_rmat" 2>&1 | tail -3
timeout 400 python scripts/ab_opts.py rmat26 5 "" "vband=0" 2>&1 | tail -2
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/vhub_band.csv -k regex:"k_count_vhub|k_seg_sort" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
