timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count_vhub -c 1 -o gpurun_out/vhub_full3 python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
