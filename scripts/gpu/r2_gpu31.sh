M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vix_base.csv -k regex:"k_seg_sort|k_big_back|k_hub_count" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
TC_VIX=0 timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vix_off.csv -k regex:"k_seg_sort|k_big_back" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
TC_LIB_PATH=variants/lib_vinp1.so timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vix_p1.csv -k regex:"k_seg_sort|k_big_back" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
