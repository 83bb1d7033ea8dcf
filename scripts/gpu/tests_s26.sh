export TC_COUNT_STATS=1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python scripts/configs.py rmat26 2>&1 | grep config
TC_LIGHT=0 python scripts/configs.py rmat26 2>&1 | grep config
