M=dram__bytes_read.sum,gpu__time_duration.sum,smsp__inst_executed.sum
for v in noload noprobe; do TC_LIB_PATH=variants/lib_$v.so timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vh_$v.csv -k regex:"k_count_vhub" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?; done
