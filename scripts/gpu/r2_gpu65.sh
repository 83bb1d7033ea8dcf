timeout 900 python scripts/ab_opts.py rmat26 5 "" "vm_bias=3" "vm_bias=3,vzone_log2=23" "vm_bias=2" 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sort_batch.csv -k regex:"k_seg_sort" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
