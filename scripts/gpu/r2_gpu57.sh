timeout 300 python scripts/small_probe.py 2>&1 | tail -4
