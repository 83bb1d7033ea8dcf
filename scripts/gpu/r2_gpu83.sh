TC_BENCH_MEMTRACE=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mt.json 2> gpurun_out/bench_mt.err; echo rc=$?
grep memtrace gpurun_out/bench_mt.err
