# round 2 session 2: validation + measurement at HEAD (re-entry baseline)
set -x
nproc; free -g | head -2; nvidia-smi -L
python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/pytest_r2p.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_r2p.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2p.json 2> gpurun_out/bench_r2p.err; echo bench_rc=$?
tail -3 gpurun_out/bench_r2p.err
s=$(date +%s); python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r2p.json 2> gpurun_out/bench_ref_r2p.err; echo ref_rc=$? wall=$(( $(date +%s) - s ))
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dram_step_s26_r2p.csv python scripts/fused_step.py 26 2 > gpurun_out/ncu_dram_r2p.log 2>&1; echo ncu2_rc=$?
