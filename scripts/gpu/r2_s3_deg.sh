# A/B: degree histogram with the next iteration's pairs in flight (TC_DEG_PIPE=1; 8 / 4 pairs per lane)
for v in "" variants/lib_degp.so variants/lib_degp4.so; do
TC_LIB_PATH=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:k_degree_hist python scripts/fused_step.py 26 2 2>/dev/null | grep k_degree_hist | awk -F'","' '{print "'$v' " $(NF-2) " " $NF}'
done
for i in 1 2; do
for v in "" variants/lib_degp.so variants/lib_degp4.so; do
TC_LIB_PATH=$v timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-120 | sed "s|^|$v |"
done; done
