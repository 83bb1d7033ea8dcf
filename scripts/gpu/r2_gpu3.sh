# round 2, GPU call 3: packed hub suffixes (hubpack) -- GPU suite, bench, reference arm,
# reference conformance suite, ncu DRAM of one s26 step
set -x
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_r2c.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_r2c.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err; echo bench_rc=$?
tail -5 gpurun_out/bench_r2c.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_r2c.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step")}, d["phases_ms"], d["e2e"]["value"], d["roofline"]["frac"])
PY
start=$(date +%s); python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench_ref_r2c.json 2> gpurun_out/bench_ref_r2c.err; echo ref_rc=$? wall=$(( $(date +%s) - start ))
tail -c 600 gpurun_out/bench_ref_r2c.json; tail -3 gpurun_out/bench_ref_r2c.err
python -m pytest -p scripts.conformance_plugin baseline/_ref_tests/test_count.py baseline/_ref_tests/test_preprocess.py baseline/_ref_tests/test_acceptance.py -v -s -p no:cacheprovider > gpurun_out/conformance_r2c.log 2>&1; echo conf_rc=$?
grep -E "ACCEPTANCE|passed|failed" gpurun_out/conformance_r2c.log | tail -12
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dram_step_s26_r2c.csv python scripts/fused_step.py 26 2 > gpurun_out/ncu_dram_r2c.log 2>&1; echo ncu_rc=$?
