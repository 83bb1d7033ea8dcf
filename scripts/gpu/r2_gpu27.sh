M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for v in vinp1 vinp2; do TC_LIB_PATH=variants/lib_$v.so ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vin_$v.csv -k regex:"k_vin_pass" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?; done
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/vin_base.csv -k regex:"k_vin_pass" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
timeout 900 python scripts/ab_opts.py rmat26 5 "" "vhub_b16w=3" "vhub_b16w=2" "vhub_b16w=5" 2>&1 | tail -4
