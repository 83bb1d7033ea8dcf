for i in 1 2; do
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-140 | sed "s/^/base /"
for m in 5 6; do TC_LIB_PATH=variants/lib_mid$m.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-140 | sed "s/^/mid$m /"; done
done
for v in mid5 mid6; do TC_LIB_PATH=variants/lib_$v.so timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/m_$v.csv -k regex:"k_count_mid" python scripts/fused_step.py 26 1 > /dev/null 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/m_base.csv -k regex:"k_count_mid" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
