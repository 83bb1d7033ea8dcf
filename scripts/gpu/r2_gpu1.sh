set -x
nproc; free -g | head -2; nvidia-smi -L
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_r2a.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_r2a.log
timeout 2400 python tests/golden/make_golden_s26.py 26 > gpurun_out/golden_s26.log 2>&1; echo golden_rc=$?
cp tests/golden/golden_s26.json gpurun_out/ 2>/dev/null
tail -3 gpurun_out/golden_s26.log | cut -c1-400
python -m pytest tests -q -m gpu -k headline -p no:cacheprovider > gpurun_out/pytest_s26.log 2>&1; echo s26_rc=$?
tail -15 gpurun_out/pytest_s26.log
