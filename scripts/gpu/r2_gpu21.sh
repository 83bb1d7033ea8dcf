timeout 900 python scripts/ab_opts.py rmat26 5 "" "vhub_unroll=4" "vhub_unroll=1" "vhub=0" "seg_w2k=0" 2>&1 | tail -6
