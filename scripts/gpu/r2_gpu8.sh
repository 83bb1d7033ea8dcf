for f in 0 1; do echo "seg_fork=$f"; TC_SEG_FORK=$f TC_COUNT_STATS=1 python scripts/configs.py rmat26 ba1e7 rgg2e7 2>&1 | grep -E "config|rror"; done
for wl in 16 32; do echo "wlight=$wl"; TC_COUNT_STATS=1 TC_SHARD_WLIGHT=$wl python scripts/shard_balance.py rmat26 8 2>&1 | tail -1; done
TC_COUNT_STATS=1 python scripts/shard_balance.py rmat26 4 2>&1 | tail -1
