# round 2: full validation + measurement at HEAD
set -x
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_r2o.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_r2o.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2o.json 2> gpurun_out/bench_r2o.err; echo bench_rc=$?
tail -3 gpurun_out/bench_r2o.err
s=$(date +%s); python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r2o.json 2> gpurun_out/bench_ref_r2o.err; echo ref_rc=$? wall=$(( $(date +%s) - s ))
python -m pytest -p scripts.conformance_plugin baseline/_ref_tests/test_count.py baseline/_ref_tests/test_preprocess.py baseline/_ref_tests/test_acceptance.py -v -s -p no:cacheprovider > gpurun_out/conformance_r2o.log 2>&1; echo conf_rc=$?
tail -1 gpurun_out/conformance_r2o.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r2o.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_r2o.log 2>&1; echo ncu1_rc=$?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dram_step_s26_r2o.csv python scripts/fused_step.py 26 2 > gpurun_out/ncu_dram_r2o.log 2>&1; echo ncu2_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_count_vmajor -s 1 -c 1 -o gpurun_out/vmajor_r2o python scripts/fused_step.py 26 1 > gpurun_out/ncu_full_r2o.log 2>&1; echo ncu3_rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_count_hub -s 0 -c 1 -o gpurun_out/hub_r2o python scripts/fused_step.py 26 1 > gpurun_out/ncu_full_hub_r2o.log 2>&1; echo ncu4_rc=$?
python scripts/shard_balance.py rmat26 8 2 > gpurun_out/shard_r2o.jsonl 2>&1; echo shard_rc=$?
for tool in memcheck initcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_workload.py > gpurun_out/sanitizer_${tool}_r2o.log 2>&1; echo ${tool}_rc=$?
  tail -1 gpurun_out/sanitizer_${tool}_r2o.log
done
