for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_workload.py > gpurun_out/sanitizer_${tool}_r2s.log 2>&1; echo ${tool}_rc=$?
  tail -2 gpurun_out/sanitizer_${tool}_r2s.log
done
