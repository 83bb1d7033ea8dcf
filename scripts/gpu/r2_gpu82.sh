timeout 600 ncu --set full --clock-control none -k regex:"k_degree_hist|k_orient|k_bucket_scatter" -c 3 -o gpurun_out/pre_full python scripts/fused_step.py 26 1 > gpurun_out/pre_full.log 2>&1; echo rc=$?
timeout 600 python scripts/two_call.py 26 8 2>&1 | tail -20
