#!/bin/bash
# A/B of the gather implementation / geometry on one config (args passed to bench.py).
# SWEEP="impl ctas threads|..." overrides the list.
SWEEP=${SWEEP:-"tma 16 32 32|tma 32 32 16|tma 64 32 8|tma 48 32 16|tma 96 32 8|tma 32 32 32"}
IFS='|' read -ra CFGS <<< "$SWEEP"
for cfg in "${CFGS[@]}"; do
  read -r impl ctas thr rows <<< "$cfg"
  python bench.py "$@" --fetch-impl $impl --fetch-ctas $ctas --fetch-threads $thr --fetch-rows ${rows:-32} --no-cpu-baseline --no-hbm-variant 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$impl ctas=$ctas thr=$thr rows=${rows:-32}', round(d['value'],2), 'tok/s', round(d['ms_per_step'],2), 'ms', 'fetch', round(d['roofline']['achieved'],2), 'share', round(d['roofline']['step_share'],3), 'gather', round(d['kernel_stats'].get('fetch_gather',{}).get('gbs',0),2))" || echo "$cfg failed"
done
