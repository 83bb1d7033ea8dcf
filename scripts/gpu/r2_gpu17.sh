python scripts/hub16_stats.py 26 > gpurun_out/hub16_s26.json 2>&1; echo rc=$?
python scripts/seg_stats.py 26 > gpurun_out/seg_s26.json 2>&1; echo rc=$?
cat gpurun_out/hub16_s26.json gpurun_out/seg_s26.json
