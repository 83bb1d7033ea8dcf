timeout 600 python scripts/ab_opts.py rmat26 5 "" "pdl=0" "" "pdl=0" 2>&1 | tail -4 | cut -c1-150
timeout 300 python scripts/ab_opts.py rmat24 5 "" "pdl=0" 2>&1 | tail -2 | cut -c1-150
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
