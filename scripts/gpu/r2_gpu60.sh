timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/pre_new.csv -k regex:"k_orient|k_seg_sort|k_bucket_scatter|k_degree" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "rank_space or schedules_agree or headline or substeps or shuffled" 2>&1 | tail -2
