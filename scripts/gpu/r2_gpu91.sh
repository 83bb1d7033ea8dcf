for i in 1 2; do
TC_LIB_PATH=variants/lib_prev.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-140 | sed "s/^/prev /"
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-140 | sed "s/^/sa /"
for m in 3 4 5; do TC_LIB_PATH=variants/lib_vmsa$m.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-140 | sed "s/^/vmsa$m /"; done
done
for v in prev vmsa4 vmsa5; do TC_LIB_PATH=variants/lib_$v.so timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/vm_$v.csv -k regex:"k_count_vmajor" python scripts/fused_step.py 26 1 > /dev/null 2>&1; done; echo rc=$?
