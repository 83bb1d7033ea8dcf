export TC_COUNT_STATS=1
timeout 900 python scripts/configs.py rmat24 rmat26 2>&1 | grep -E "config|Error|error"
