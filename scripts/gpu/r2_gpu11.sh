for P in 2 4 8 16; do TC_COUNT_STATS=1 python scripts/shard_balance.py rmat26 $P 2>&1 | tail -1 | cut -c1-300; done
TC_COUNT_STATS=1 python scripts/shard_balance.py rmat24 8 2>&1 | tail -1 | cut -c1-300
