timeout 900 python scripts/ab_opts.py rmat26 7 "" "vm_bias=3,vzone_log2=23" "" "vm_bias=3,vzone_log2=23" "vm_bias=3" 2>&1 | tail -5
