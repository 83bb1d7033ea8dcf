timeout 600 python scripts/ab_opts.py rmat26 5 "" "concurrent=1" "concurrent=1,share=2" 2>&1 | tail -3
