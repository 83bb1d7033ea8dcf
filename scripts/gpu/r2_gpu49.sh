timeout 400 python scripts/ab_opts.py rmat26 5 "" "vband=1" 2>&1 | tail -2
