timeout 900 python scripts/ab_opts.py rmat26 5 "" "vhub_blocks=1" "vhub_blocks=8" "vhub_blocks=32" "vhub_blocks=64" 2>&1 | tail -5
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules_agree or headline or huge_rmat" 2>&1 | tail -3
