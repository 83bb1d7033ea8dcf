# A/B: rank-space vs original-id fused path on the low-skew configs (RGG keeps spatial id locality)
# result (session 3): identical times -- rank_primary only selects what tc_preprocess builds; the fused device path always counts in rank space
timeout 600 python scripts/ab_opts.py rgg2e7 5 "" "rank_primary=0" 2>&1 | tail -2 | cut -c1-330
timeout 600 python scripts/ab_opts.py ba1e7 5 "" "rank_primary=0" 2>&1 | tail -2 | cut -c1-330
timeout 600 python scripts/ab_opts.py rmat20 5 "" "rank_primary=0" 2>&1 | tail -2 | cut -c1-330
