timeout 900 python scripts/ab_opts.py rmat26 5 "pdl=0" "pdl=1" "pdl=2" "pdl=4" "pdl=8" "pdl=0" 2>&1 | tail -6 | cut -c1-150
