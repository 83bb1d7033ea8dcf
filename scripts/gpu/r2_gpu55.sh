timeout 300 python scripts/mix_probe.py 26 fffttttff 2>&1 | tail -9
timeout 300 python scripts/mix_probe.py 26 fffttttff k 2>&1 | tail -9
