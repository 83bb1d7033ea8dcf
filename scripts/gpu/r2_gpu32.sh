timeout 600 python scripts/ab_opts.py rmat26 5 "" "vzone_log2=21" "vzone_log2=20" "vzone_log2=19" "vix=0,vzone_log2=21" 2>&1 | tail -5
