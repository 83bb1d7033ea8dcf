# head-sharded v-major plan: correctness + serial shard balance; hub window prefetch timing
set -x
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "shard_plan or schedules or headline or huge" > gpurun_out/pytest_r2g.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_r2g.log
TC_COUNT_STATS=1 python scripts/configs.py rmat26 rmat24 2>&1 | grep -E "config|rror"
TC_MIDWARP=2 TC_COUNT_STATS=1 python scripts/configs.py rmat26 2>&1 | grep -E "config|rror"
for P in 2 4 8; do python scripts/shard_balance.py rmat26 $P 2>&1 | tail -1; done
