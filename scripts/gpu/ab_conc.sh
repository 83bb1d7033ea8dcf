for C in 0 1; do echo "TC_CONCURRENT=$C"; TC_CONCURRENT=$C timeout 900 python scripts/configs.py rmat24 rmat26 2>&1 | grep -E "config|Error|error" | cut -c1-130; done
TC_CONCURRENT=1 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k schedules 2>&1 | tail -1
