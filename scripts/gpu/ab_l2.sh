export TC_COUNT_STATS=1
for cfg in "TC_L2_PERSIST_MB=32" "TC_L2_PERSIST_MB=0" "TC_L2_TARGET=1 TC_L2_PERSIST_MB=32" "TC_L2_TARGET=1 TC_L2_PERSIST_MB=64" "TC_L2_TARGET=1 TC_L2_PERSIST_MB=96"; do echo "$cfg"; env $cfg timeout 900 python scripts/configs.py rmat26 2>&1 | grep -E "config|Error|error" | cut -c1-260; done
