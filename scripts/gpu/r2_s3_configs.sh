# per-config bench lines at HEAD (BASELINE configs[0..4]) + the headline s26 line
timeout 900 python bench.py --workload er --steps 10 --warmup 3 > gpurun_out/c_er.json 2> gpurun_out/c_er.err; echo er=$?
timeout 900 python bench.py --workload rmat --scale 20 --steps 10 --warmup 3 > gpurun_out/c_s20.json 2> gpurun_out/c_s20.err; echo s20=$?
timeout 900 python bench.py --workload ba --steps 10 --warmup 3 > gpurun_out/c_ba.json 2> gpurun_out/c_ba.err; echo ba=$?
timeout 900 python bench.py --workload rgg --steps 10 --warmup 3 > gpurun_out/c_rgg.json 2> gpurun_out/c_rgg.err; echo rgg=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c_s26.json 2> gpurun_out/c_s26.err; echo s26=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/c_ref.json 2> gpurun_out/c_ref.err; echo ref=$?
