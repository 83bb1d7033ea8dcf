export TC_COUNT_STATS=1
for v in "$@"; do echo "== $v"; TC_LIB_PATH=build_variants/lib_$v.so timeout 300 python scripts/configs.py rmat24 rmat26 2>&1 | grep -E "config|rror" | cut -c1-250; done
