timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_r2r.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_r2r.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2r.json 2> gpurun_out/bench_r2r.err; echo bench_rc=$?
tail -2 gpurun_out/bench_r2r.err
