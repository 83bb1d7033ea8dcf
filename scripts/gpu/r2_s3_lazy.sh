# A/B: cuckoo probes with the h2 load only when the h1 slot holds another key (TC_CUCKOO_LAZY=1)
for i in 1 2; do
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-200 | sed "s/^/head /"
TC_LIB_PATH=variants/lib_lazy.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-200 | sed "s/^/lazy /"
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed
for v in base lazy; do
L=""; [ $v = lazy ] && L=variants/lib_lazy.so
TC_LIB_PATH=$L timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/lazy_$v.csv -k regex:"k_count" python scripts/fused_step.py 26 1 > gpurun_out/lazy_ncu_$v.log 2>&1; echo rc=$?
done
