# A/B: k_count_vlow_warp skips probes of items outside [min adj(v), max adj(v)] (TC_VLOW_RANGE=1)
for i in 1 2; do
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-200 | sed "s/^/head /"
TC_LIB_PATH=variants/lib_vrange.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-200 | sed "s/^/vrange /"
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed
for v in vrange; do
L=""; [ $v = vrange ] && L=variants/lib_vrange.so
TC_LIB_PATH=$L timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vrange_$v.csv -k regex:"k_count" python scripts/fused_step.py 26 1 > gpurun_out/vrange_ncu_$v.log 2>&1; echo rc=$?
done
