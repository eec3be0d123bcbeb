timeout 300 python -m pytest tests/test_tc05_gpu.py -x -q -s > gpurun_out/r02e_tc05_tests.log 2>&1; echo rc=$? >> gpurun_out/r02e_tc05_tests.log
timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_resident_gpu.py -x -q > gpurun_out/r02e_engine_tests.log 2>&1; echo rc=$? >> gpurun_out/r02e_engine_tests.log
for v in "IG_APPEND_FIRST=1" "IG_APPEND_FIRST=0" "IG_STREAM_PRIO=-1,0" "IG_STREAM_PRIO=0,0" "IG_STREAM_PRIO=-1,0 IG_APPEND_FIRST=0"; do
  env $v timeout 400 python bench.py --no-cpu-baseline --no-variant > gpurun_out/r02e_bench_$(echo $v | tr ' =,' '___').json 2>/dev/null
done
