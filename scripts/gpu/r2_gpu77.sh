timeout 300 python scripts/pre_probe.py rmat26 5
for x in a b c d; do TC_LIB_PATH=variants/lib_sw$x.so timeout 300 python scripts/pre_probe.py rmat26 5 | sed "s/^/sw$x /"; done
timeout 300 python scripts/pre_probe.py rmat26 5
