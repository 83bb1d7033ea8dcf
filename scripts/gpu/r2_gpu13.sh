python scripts/head_costs.py rmat26 2>&1 | tail -32
for w in er ba rgg; do python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 3 --cpu-seconds 8 > gpurun_out/bench_${w}_r2m.json 2> gpurun_out/bench_${w}_r2m.err; echo "$w rc=$?"; tail -2 gpurun_out/bench_${w}_r2m.err; done
python bench.py --workload rmat --scale 20 --steps 10 --warmup 3 --e2e-steps 3 --cpu-seconds 8 > gpurun_out/bench_s20_r2m.json 2> gpurun_out/bench_s20_r2m.err; echo "s20 rc=$?"
