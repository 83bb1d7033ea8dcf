timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
TC_LIB_PATH=variants/lib_vminb5.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | sed 's/^/minb5 /'
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
TC_LIB_PATH=variants/lib_vminb5.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | sed 's/^/minb5 /'
