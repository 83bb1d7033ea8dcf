for i in 1 2; do
timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-140 | sed "s/^/ww /"
TC_LIB_PATH=variants/lib_ww0.so timeout 300 python scripts/ab_opts.py rmat26 5 "" 2>&1 | tail -1 | cut -c1-140 | sed "s/^/ww0 /"
done
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/ww.csv -k regex:"k_count_vhub" python scripts/fused_step.py 26 1 > /dev/null 2>&1; echo rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "schedules or headline or rmat or prebuilt" 2>&1 | tail -2
