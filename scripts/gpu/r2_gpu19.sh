python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree or headline or huge_rmat" 2>&1 | tail -5
timeout 600 python scripts/ab_opts.py rmat26 5 "" "vhub=0" 2>&1 | tail -3
