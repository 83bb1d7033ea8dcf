timeout 600 python scripts/two_call.py 26 8 --bench-like 2>&1 | tail -24
