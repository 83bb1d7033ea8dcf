# A/B: k_orient at 6 / 8 CTAs per SM (__launch_bounds__ min blocks) vs HEAD (5)
for i in 1 2; do
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-120 | sed "s/^/head /"
TC_LIB_PATH=variants/lib_or6.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-120 | sed "s/^/or6 /"
TC_LIB_PATH=variants/lib_or8.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-120 | sed "s/^/or8 /"
done
for v in "" variants/lib_or6.so; do
TC_LIB_PATH=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_orient python scripts/fused_step.py 26 1 2>/dev/null | grep k_orient | tail -1 | awk -F'","' '{print "'$v' " $NF}'
done
