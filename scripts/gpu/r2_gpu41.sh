M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/pre_base.csv -k regex:"k_degree_hist|k_orient|k_bucket_scatter" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
for v in deg16 deg4; do TC_LIB_PATH=variants/lib_$v.so timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/pre_$v.csv -k regex:"k_degree_hist" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?; done
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
