TC_LIB_PATH=variants/lib_head.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | sed 's/^/head /'
timeout 900 python scripts/ab_opts.py rmat26 5 "" "vix_small=512" "vix_small=2048" "vix_small=4096" "vix_small=8192" 2>&1 | tail -6
TC_LIB_PATH=variants/lib_head.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | sed 's/^/head /'
