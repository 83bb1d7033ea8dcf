for v in depth2 depth2b4; do TC_LIB_PATH=variants/lib_$v.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1; done
