timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pool0.json 2>/dev/null; echo rc=$?
TC_LIB_PATH=variants/lib_onepool.so timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pool1.json 2>/dev/null; echo rc=$?
for f in pool0 pool1; do python -c "import json;d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]);e=d['e2e'];print('$f', d['ms_per_step'], e['ms_per_step'], {k:(v['ms_per_step'],v['step_wall_ms']) for k,v in e['variants'].items()})"; done
