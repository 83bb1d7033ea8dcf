timeout 600 python scripts/ab_opts.py rmat26 5 "" "vm_entry=32" "vm_entry=64" "vm_entry=128" "vm_entry=256" 2>&1 | tail -5
