timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/memcheck_r2w.log 2>&1; echo memcheck_rc=$?; tail -3 gpurun_out/memcheck_r2w.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/racecheck_r2w.log 2>&1; echo racecheck_rc=$?; tail -3 gpurun_out/racecheck_r2w.log
