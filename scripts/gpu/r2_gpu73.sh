timeout 900 python scripts/ab_opts.py rmat26 5 "" "vm_stage=2" "vm_stage=4" "vm_stage=8" 2>&1 | tail -20
