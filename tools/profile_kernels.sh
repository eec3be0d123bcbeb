#!/bin/bash
# Full ncu captures of the path kernels at the C3 per-layer size (4 layers of the
# OPT-13B shape: identical launches, short setup).  Usage: tools/profile_kernels.sh r01c [kernels...]
R=${1:-r01c}
shift
KS=${@:-"fetch_slots_kernel rehearse_count_kernel attend512_wp_kernel attend512_mma_kernel select_kernel append_kernel sgemm_tcw_kernel resident_plan_kernel layernorm_kernel"}
export IG_PROFILE_WINDOW=1
for K in $KS; do
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:${K} -s 2 -c 2 -o gpurun_out/prof_${R}_${K} -f \
      python bench.py --layers 4 --steps 1 --warmup 1 --no-cpu-baseline --no-variant \
      > /dev/null 2> gpurun_out/prof_${R}_${K}.err
done
