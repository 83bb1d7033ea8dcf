M=dram__bytes_read.sum,gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct,smsp__cycles_active.avg
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vhub_b16.csv -k regex:"k_count_vhub|k_band" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
TC_VHUB_BLOCKS=1 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vhub_b1.csv -k regex:"k_count_vhub" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
TC_VHUB_BLOCKS=4 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vhub_b4.csv -k regex:"k_count_vhub" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
