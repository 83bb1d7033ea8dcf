timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree or headline or forced" 2>&1 | tail -2
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
TC_LIB_PATH=variants/lib_vlx0.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/vlow_x1.csv -k regex:"k_count_vlow" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
timeout 300 python scripts/two_call.py 26 2>&1 | tail -3
TC_VIX=0 timeout 300 python scripts/two_call.py 26 2>&1 | tail -2
