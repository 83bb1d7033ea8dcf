timeout 400 python scripts/ab_opts.py rmat26 7 "" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree or headline or prebuilt" 2>&1 | tail -2
