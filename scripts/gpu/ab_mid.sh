export TC_COUNT_STATS=1
for M in 1 2; do echo "TC_MIDWARP=$M"; TC_MIDWARP=$M timeout 900 python scripts/configs.py rmat24 rmat26 2>&1 | grep -E "config|Error|error" | cut -c1-230; done
