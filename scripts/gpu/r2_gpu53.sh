timeout 300 python scripts/two_call.py 26 2>&1 | tail -3
