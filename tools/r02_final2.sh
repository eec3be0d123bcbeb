#!/bin/bash
# Round-2 closing validation (second pass): every GPU test, smoke, default bench
# with CPU baseline + parity leg, reference arm, C1/C2/C4 bench lines, the ncu
# launch list of the default bench and one full ncu capture of the select.
R=${1:-r02fin}
bash tools/round_check.sh $R
timeout 600 python bench.py --shape llama-2-7b --batch 4 --prompt 32768 --no-cpu-baseline > gpurun_out/${R}_bench_c4.json 2> gpurun_out/${R}_bench_c4.err
timeout 600 python bench.py --shape opt-6.7b --batch 8 --prompt 2048 --no-cpu-baseline > gpurun_out/${R}_bench_c2.json 2> gpurun_out/${R}_bench_c2.err
timeout 600 python bench.py --shape opt-125m --batch 1 --prompt 2048 --no-cpu-baseline > gpurun_out/${R}_bench_c1.json 2> gpurun_out/${R}_bench_c1.err
timeout 900 bash tools/profile_round.sh $R
timeout 600 ncu --set full --clock-control none --import-source on -k regex:select_kernel -s 3 -c 1 \
    -o gpurun_out/${R}_select_ncu python tools/select_probe.py --layers 2 --chain 1 > gpurun_out/${R}_select_ncu.log 2>&1
echo done
