timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree or headline or prebuilt or huge_rmat or forced" 2>&1 | tail -3
timeout 400 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
