timeout 300 python scripts/pre_probe.py rmat26 5
for g in 32 128 512 4096 1000000000; do TC_LIB_PATH=variants/lib_skip$g.so timeout 300 python scripts/pre_probe.py rmat26 5 | sed "s/^/skip$g /"; done
timeout 300 python scripts/pre_probe.py rmat26 5
