# A/B: k_count_vhub 16-bit sweep read lane-strided (TC_VHUB_LANE=1) vs HEAD
for i in 1 2; do
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-200 | sed "s/^/head /"
TC_LIB_PATH=variants/lib_lane.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-200 | sed "s/^/lane /"
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
TC_LIB_PATH=variants/lib_lane.so timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/lane_vhub.csv -k regex:"k_count_vhub" python scripts/fused_step.py 26 1 > gpurun_out/lane_ncu.log 2>&1; echo rc=$?
tail -1 gpurun_out/lane_ncu.log
