set -x
python scripts/configs.py rmat20 rmat22 ba1e7 rgg2e7 rmat24 > gpurun_out/configs.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_ba.csv python scripts/step.py ba1e7 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_rgg.csv python scripts/step.py rgg2e7 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_count_window -s 1 -c 1 -o gpurun_out/ba_window python scripts/step.py ba1e7 2 > gpurun_out/ncu_ba.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_count -s 2 -c 2 -o gpurun_out/rgg_count python scripts/step.py rgg2e7 2 > gpurun_out/ncu_rgg.log 2>&1
cat gpurun_out/configs.log
