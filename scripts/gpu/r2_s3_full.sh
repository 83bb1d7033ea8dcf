# ncu --set full of the second count kernel (k_count_vlow_warp) and the top preprocess kernel (k_orient) at s26
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count_vlow_warp -c 1 -o gpurun_out/vlow_full python scripts/fused_step.py 26 1 > gpurun_out/vlow_full.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_orient -c 1 -o gpurun_out/orient_full python scripts/fused_step.py 26 1 > gpurun_out/orient_full.log 2>&1; echo rc=$?
for r in vlow_full orient_full; do ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/$r.csv 2>/dev/null; ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null; done; ls -la gpurun_out/
