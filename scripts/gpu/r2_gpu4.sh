set -x
python -m pytest tests/test_gpu_parity.py tests/test_api_contract_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_r2d.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_r2d.log
for hp in 0 2 1; do echo "hubpack=$hp"; TC_HUBPACK=$hp TC_COUNT_STATS=1 python scripts/configs.py rmat26 rmat24 2>&1 | grep -E "config|rror"; done
python scripts/two_call.py 26 2>&1 | tail -4
python scripts/pageable_e2e.py 26 2>&1 | tail -6
