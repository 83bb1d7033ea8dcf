export TC_COUNT_STATS=1
for cfg in "TC_LIGHT=0" "TC_LIGHT=1"; do echo "$cfg"; env $cfg python scripts/configs.py rgg2e7 rmat24 2>&1 | grep config; done
TC_LIGHT=1 ncu --set full --clock-control none --import-source on -k regex:k_count_light_tpe -s 1 -c 1 -o gpurun_out/rgg_tpe python scripts/step.py rgg2e7 2 > gpurun_out/ncu_rgg_tpe.log 2>&1
TC_LIGHT=1 ncu --set full --clock-control none --import-source on -k regex:k_count_light_tpe -s 1 -c 1 -o gpurun_out/ba_tpe python scripts/step.py ba1e7 2 > gpurun_out/ncu_ba_tpe.log 2>&1
