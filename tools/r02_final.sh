#!/bin/bash
bash tools/round_check.sh r02z
timeout 600 python bench.py --shape llama-2-7b --batch 4 --prompt 32768 --no-cpu-baseline > gpurun_out/r02z_bench_c4.json 2> gpurun_out/r02z_bench_c4.err
timeout 600 python bench.py --shape opt-6.7b --batch 8 --prompt 2048 --no-cpu-baseline > gpurun_out/r02z_bench_c2.json 2> gpurun_out/r02z_bench_c2.err
timeout 600 python bench.py --shape opt-125m --batch 1 --prompt 2048 --no-cpu-baseline > gpurun_out/r02z_bench_c1.json 2> gpurun_out/r02z_bench_c1.err
