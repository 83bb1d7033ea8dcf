ncu --set full --clock-control none --import-source on -k regex:"k_count_hub|k_count_light_tpe" -c 3 -o gpurun_out/hub_s26 python scripts/step.py rmat26 1 > gpurun_out/ncu_hub.log 2>&1
