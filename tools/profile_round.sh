#!/bin/bash
# ncu launch list of the timed steps of the bench command (C3 default).
# Usage (on the GPU box): tools/profile_round.sh r01
R=${1:-r01}
mkdir -p gpurun_out
IG_PROFILE_WINDOW=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${R}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-variant \
    > gpurun_out/launches_${R}.bench.json 2> gpurun_out/launches_${R}.err
