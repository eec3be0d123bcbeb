timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "attend" > gpurun_out/r02ae_attn.log 2>&1; echo rc=$? >> gpurun_out/r02ae_attn.log
for cfg in "--B 4 --Hg 32 --rows 6553 --cap 6556" "--rows 819 --cap 820" "--rows 4096 --cap 4100"; do
  n=$(echo $cfg | tr -d ' -' | cut -c1-24)
  IG_ATTEND_IMPL=c timeout 200 python tools/attend_trace.py $cfg > gpurun_out/r02ae_c_$n.json 2>&1
  IG_ATTEND_IMPL=mma timeout 200 python tools/attend_trace.py $cfg > gpurun_out/r02ae_m_$n.json 2>&1
done
bash tools/ab.sh r02ae "IG_ATTEND_IMPL=mma" "IG_ATTEND_IMPL=c"
bash tools/ab_c4.sh r02ae4 "IG_ATTEND_IMPL=mma" "IG_ATTEND_IMPL=c"
