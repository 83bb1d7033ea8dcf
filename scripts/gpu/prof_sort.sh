# one radix pass of the rank-space key sort at s26 (skip the generator's sort passes)
ncu --set full --clock-control none --import-source on -k regex:"k_radix_pass|k_orient" -s 30 -c 4 -o gpurun_out/sort_s26 python scripts/step.py rmat26 1 > gpurun_out/ncu_sort.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_sort_s26.csv python scripts/step.py rmat26 1 > /dev/null 2>&1
