# dynamic item claiming in the warp-persistent attention: parity, alone, in the C3 step
IG_WP_DYN=1 timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_fullsize_gpu.py -q -x -k "attend or attention or graph_replay" > gpurun_out/r02_latedyn_tests.log 2>&1
tail -2 gpurun_out/r02_latedyn_tests.log
for dy in 0 1; do IG_WP_DYN=$dy python tools/attend_probe.py --sweep 256,512,819,2048 > gpurun_out/r02_latedyn_probe_$dy.jsonl 2>&1; done
cat gpurun_out/r02_latedyn_probe_*.jsonl
tools/ab.sh r02_latedyn "IG_WP_DYN=0" "IG_WP_DYN=1" "IG_WP_DYN=0" "IG_WP_DYN=1"
python tools/ab_show.py r02_latedyn
