export TC_COUNT_STATS=1
for cfg in "TC_LIGHT=1" "TC_LIGHT=2" "TC_LIGHT=2 TC_SKEW=8" "TC_LIGHT=2 TC_SKEW=128"; do echo "$cfg"; env $cfg python scripts/configs.py ba1e7 rgg2e7 rmat20 rmat24 2>&1 | grep config; done
