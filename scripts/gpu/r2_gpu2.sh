# round 2, GPU call 2: full GPU suite, both bench arms, reference conformance suite,
# ncu DRAM capture of one s26 step, compute-sanitizer over the small-graph workload
set -x
nproc; free -g | head -2
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_r2b.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_r2b.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench_r2b.json; tail -5 gpurun_out/bench_r2b.err
/usr/bin/time -v python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref_r2b.json 2> gpurun_out/bench_ref_r2b.err; echo ref_rc=$?
tail -c 1500 gpurun_out/bench_ref_r2b.json; grep -E "Elapsed|Maximum resident" gpurun_out/bench_ref_r2b.err
python -m pytest -p scripts.conformance_plugin baseline/_ref_tests/test_count.py baseline/_ref_tests/test_preprocess.py baseline/_ref_tests/test_acceptance.py -v -s -p no:cacheprovider > gpurun_out/conformance_r2b.log 2>&1; echo conf_rc=$?
grep -E "ACCEPTANCE|passed|failed" gpurun_out/conformance_r2b.log | tail -12
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dram_step_s26_r2b.csv python scripts/fused_step.py 26 2 > gpurun_out/ncu_dram_r2b.log 2>&1; echo ncu_rc=$?
for tool in memcheck initcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_workload.py > gpurun_out/sanitizer_${tool}_r2b.log 2>&1; echo ${tool}_rc=$?
  tail -3 gpurun_out/sanitizer_${tool}_r2b.log
done
