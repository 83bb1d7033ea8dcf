timeout 600 python scripts/ab_opts.py rmat26 5 "" "vhub_b16w=3" "vhub_b16w=2" "hub_cap_div=2" "hub_cap_div=4" 2>&1 | tail -5
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree" 2>&1 | tail -2
