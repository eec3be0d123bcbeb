#!/bin/bash
# Full ncu captures of the path kernels inside the bench's timed steps.
# Usage: tools/profile_kernels.sh r01c [kernels...]
#   LAYERS (default 4: identical launch sizes, short setup) and SKIP (default 2:
#   launches skipped per kernel before the 2 captured ones).  LAYERS=40 SKIP=20
#   captures the middle of the full C3 model (layer ~20: ~820-row selections).
R=${1:-r01c}
shift
KS=${@:-"fetch_slots_kernel rehearse_count_kernel attend512_wp_kernel attend512_mma_kernel select_kernel append_kernel sgemm_packed_kernel resident_plan_kernel layernorm_kernel"}
LAYERS=${LAYERS:-4}
SKIP=${SKIP:-2}
export IG_PROFILE_WINDOW=1
for K in $KS; do
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:${K} -s ${SKIP} -c 2 -o gpurun_out/prof_${R}_${K} -f \
      python bench.py --layers ${LAYERS} --steps 1 --warmup 1 --no-cpu-baseline --no-variant \
      > /dev/null 2> gpurun_out/prof_${R}_${K}.err
done
