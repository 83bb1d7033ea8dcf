for i in 1 2; do
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-140
for u in 1 2; do TC_LIB_PATH=variants/lib_vpipe$u.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-140 | sed "s/^/vpipe$u /"; done
done
for u in 1 2; do TC_LIB_PATH=variants/lib_vpipe$u.so timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/vpipe$u.csv -k regex:"k_count_vlow" python scripts/fused_step.py 26 1 > /dev/null 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/vpipe0.csv -k regex:"k_count_vlow" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
