export TC_COUNT_STATS=1
TC_BUCKET=1 python scripts/csr_hash.py rmat12 rmat16 rmat20 ba1e6 rgg2e6 rmat24 2>&1 | tail -6
TC_BUCKET=1 timeout 900 python scripts/configs.py rmat20 rmat22 ba1e7 rgg2e7 rmat24 rmat26 2>&1 | grep -E "config|Error|error"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_bucket_s26.csv python scripts/step.py rmat26 1 > /dev/null 2>&1
