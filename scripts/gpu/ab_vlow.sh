export TC_COUNT_STATS=1
for cfg in "TC_VZONE_LOG2=19 TC_VLOW_ALL=1" "TC_VZONE_LOG2=21 TC_VLOW_ALL=1" "TC_VZONE_LOG2=22 TC_VLOW_ALL=1" "TC_VZONE_LOG2=23 TC_VLOW_ALL=1"; do echo "$cfg"; env $cfg timeout 900 python scripts/configs.py rmat22 rmat24 rmat26 2>&1 | grep -E "config|Error|error" | cut -c1-230; done
