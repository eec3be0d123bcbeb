# LN2 / next LN1 fused into the residual GEMMs' tails: parity, then the C3 step A/B
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -x -k "packed or layernorm or graph_replay or f32_pool or c1 or step_host or hook or trace or prefill" > gpurun_out/r02_lnfuse_tests.log 2>&1
tail -3 gpurun_out/r02_lnfuse_tests.log
tools/ab.sh r02_lnfuse "IG_LN_FUSE=0" "IG_LN_FUSE=1" "IG_LN_FUSE=0" "IG_LN_FUSE=1"
python tools/ab_show.py r02_lnfuse
