#!/bin/bash
# A/B at C4 (Llama-2-7B shape, B 4, 32K): tools/ab_c4.sh TAG "ENV=.." ...
TAG=$1; shift
i=0
for v in "$@"; do
  env $v timeout 600 python bench.py --shape llama-2-7b --batch 4 --prompt 32768 --no-cpu-baseline --no-variant > gpurun_out/${TAG}_$i.json 2>/dev/null
  echo "$i $v" >> gpurun_out/${TAG}_index.txt
  i=$((i+1))
done
