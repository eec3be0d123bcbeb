#!/bin/bash
# Full validation on the GPU box: every GPU test, smoke(), the default bench
# line (with the CPU baseline), the reference arm.  Usage: tools/round_check.sh r02s
R=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${R}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/${R}_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/${R}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${R}_smoke.log
timeout 900 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${R}_bench_reference.json 2> gpurun_out/${R}_bench_reference.err
