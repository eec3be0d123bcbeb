#!/bin/bash
# ncu evidence for one round: launch list of the timed bench steps and full
# captures of the path kernels.  Usage (on the GPU box): tools/profile_round.sh r01
R=${1:-r01}
mkdir -p gpurun_out
export IG_PROFILE_WINDOW=1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${R}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/launches_${R}.bench.json 2> gpurun_out/launches_${R}.err
for K in fetch_kernel rehearse_kernel attend_kernel select_kernel count_kernel; do
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:${K} -s 2 -c 2 -o gpurun_out/prof_${R}_${K} -f \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/prof_${R}_${K}.err
done
ls -la gpurun_out/
