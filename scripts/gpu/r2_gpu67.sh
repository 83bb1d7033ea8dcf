timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_r2v.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_r2v.log
timeout 400 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
timeout 400 python scripts/ab_opts.py rmat24 5 "" "vm_bias=4,vzone_log2=22" 2>&1 | tail -2
