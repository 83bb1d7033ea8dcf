# packed-sweep variants, v-major bias, shard model 2
for lib in pu4 pu8 pu8b5; do for hp in 1 2; do echo "lib=$lib hubpack=$hp"; TC_LIB_PATH=variants/lib_$lib.so TC_HUBPACK=$hp TC_COUNT_STATS=1 python scripts/configs.py rmat26 2>&1 | grep -E "config|rror"; done; done
for b in 3 5; do for hp in 0 1; do echo "bias=$b hubpack=$hp"; TC_VM_BIAS=$b TC_HUBPACK=$hp TC_COUNT_STATS=1 python scripts/configs.py rmat26 2>&1 | grep -E "config|rror"; done; done
for model in 0 2; do echo "shard model $model"; TC_SHARD_MODEL=$model python scripts/shard_balance.py rmat26 8 2>&1 | tail -1; done
