python scripts/shard_balance.py rmat26 8 2 2>&1 | grep config | cut -c1-260
python scripts/shard_balance.py rmat26 4 1 2>&1 | grep config | cut -c1-220
TC_COUNT_STATS=1 python scripts/configs.py rmat26 rmat24 2>&1 | grep -E "config|rror"
