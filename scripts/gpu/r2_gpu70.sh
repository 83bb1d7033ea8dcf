timeout 400 python scripts/ab_opts.py rmat26 7 "" 2>&1 | tail -1
TC_LIB_PATH=variants/lib_vmwpt1.so timeout 400 python scripts/ab_opts.py rmat26 7 "" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree or headline or forced" 2>&1 | tail -2
