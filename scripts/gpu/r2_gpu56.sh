timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2t.json 2> gpurun_out/bench_r2t.err; echo rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_r2t.json').read().strip().splitlines()[-1]);print(d['e2e']['variants'])"
