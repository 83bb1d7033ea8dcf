ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_bucket_s26.csv python scripts/step.py rmat26 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_bucket_s24.csv python scripts/step.py rmat24 1 > /dev/null 2>&1
