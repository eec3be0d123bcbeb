#!/bin/bash
# A/B of environment switches on the default bench (no CPU baseline / variant).
# Usage: tools/ab.sh TAG "ENV=1 ENV2=x" "ENV=0" ...   -> gpurun_out/TAG_<i>.json
TAG=$1; shift
i=0
for v in "$@"; do
  env $v timeout 400 python bench.py --no-cpu-baseline --no-variant > gpurun_out/${TAG}_$i.json 2>/dev/null
  echo "$i $v" >> gpurun_out/${TAG}_index.txt
  i=$((i+1))
done
