timeout 900 python scripts/ab_opts.py rmat26 5 "" "vm_bias=3" "vm_bias=5" "vhub_b16w=3" "vhub_b16w=2" "dense_factor=2" "dense_factor=4" "vzone_log2=23" 2>&1 | tail -8
