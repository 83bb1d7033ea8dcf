timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2s.json 2> gpurun_out/bench_r2s.err; echo rc=$?
for w in "er" "rmat --scale 20" "ba" "rgg"; do
  n=$(echo $w | tr ' ' '_' | tr -d '-')
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_cfg_$n.json 2> gpurun_out/bench_cfg_$n.err; echo $n rc=$?
  tail -1 gpurun_out/bench_cfg_$n.json | cut -c1-300
done
