timeout 600 python scripts/ab_opts.py rmat26 5 "" "vin_overlap=0" "vin_grid=1" "vin_grid=4" "vin_grid=8" "seg_k16=0" 2>&1 | tail -8
timeout 300 python scripts/ab_opts.py rmat24 5 "" "vin_overlap=0" 2>&1 | tail -3
