timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "attend or attention" > gpurun_out/r02m_attn_tests.log 2>&1; echo rc=$? >> gpurun_out/r02m_attn_tests.log
timeout 200 python tools/attend_trace.py > gpurun_out/r02m_trace.json 2>&1
timeout 100 python tools/attend_trace.py --rows 4096 --cap 4100 > gpurun_out/r02m_trace4k.json 2>&1
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_resident_gpu.py -x -q > gpurun_out/r02m_engine_tests.log 2>&1; echo rc=$? >> gpurun_out/r02m_engine_tests.log
timeout 400 python bench.py --no-cpu-baseline --no-variant > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err
