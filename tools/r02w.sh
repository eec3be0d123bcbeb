timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -k "select" > gpurun_out/r02w_select.log 2>&1; echo rc=$? >> gpurun_out/r02w_select.log
timeout 600 python bench.py --shape llama-2-7b --batch 4 --prompt 32768 --no-cpu-baseline > gpurun_out/r02w_bench_c4.json 2> gpurun_out/r02w_bench_c4.err
IG_SELECT_CLUSTER=0 timeout 600 python bench.py --shape llama-2-7b --batch 4 --prompt 32768 --no-cpu-baseline --no-variant > gpurun_out/r02w_bench_c4_nocluster.json 2> /dev/null
timeout 600 python bench.py --shape opt-6.7b --batch 8 --prompt 2048 --no-cpu-baseline > gpurun_out/r02w_bench_c2.json 2> gpurun_out/r02w_bench_c2.err
timeout 600 python bench.py --shape opt-125m --batch 1 --prompt 2048 --no-cpu-baseline > gpurun_out/r02w_bench_c1.json 2> gpurun_out/r02w_bench_c1.err
