export TC_COUNT_STATS=1
for V in 1; do echo "TC_VMAJOR=$V"; TC_VMAJOR=$V timeout 600 python scripts/configs.py rmat20 rmat22 ba1e7 rgg2e7 rmat24 rmat26 2>&1 | grep -E "config|Error|error"; done
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
