python scripts/shard_balance.py rmat26 8 3 2>&1 | grep config | cut -c1-200
python scripts/shard_balance.py rmat26 4 2 2>&1 | grep config | cut -c1-200
python scripts/shard_balance.py rmat26 2 2 2>&1 | grep config | cut -c1-200
for lib in vm5; do echo "lib=$lib"; TC_LIB_PATH=variants/lib_$lib.so TC_COUNT_STATS=1 python scripts/configs.py rmat26 2>&1 | grep -E "config|rror"; done
TC_COUNT_STATS=1 python scripts/configs.py rmat26 2>&1 | grep -E "config|rror"
