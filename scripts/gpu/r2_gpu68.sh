timeout 400 python scripts/ab_opts.py rmat26 7 "" 2>&1 | tail -1
TC_LIB_PATH=variants/lib_wpt1.so timeout 400 python scripts/ab_opts.py rmat26 7 "" 2>&1 | tail -1
TC_LIB_PATH=variants/lib_wpt4.so timeout 400 python scripts/ab_opts.py rmat26 7 "" 2>&1 | tail -1
