timeout 600 python -m pytest tests/test_cli.py -q -m gpu > gpurun_out/r02u_cli.log 2>&1; echo rc=$? >> gpurun_out/r02u_cli.log
bash tools/profile_round.sh r02u
LAYERS=4 SKIP=0 timeout 600 bash tools/profile_kernels.sh r02u attend_tc05_kernel sgemm_packed_kernel attend512_wp_kernel select_kernel rehearse_count_kernel
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc05_kernel -s 1 -c 1 -o gpurun_out/prof_r02u_gemm_tc05 -f python tools/gemm_tc05_probe.py 65536x15360x5120 > /dev/null 2> gpurun_out/prof_r02u_gemm_tc05.err
cuobjdump -sass paper_2406_19707_b200/libinfinigen_b200.so | grep -oE "UTCHMMA|UTCQMMA|UTCBAR|UTCCP|LDTM|STTM|UTMALDG|UTMASTG|UBLKCP|HMMA\.[0-9A-Z.]+" | sort | uniq -c > gpurun_out/r02u_sass_mnemonics.txt
