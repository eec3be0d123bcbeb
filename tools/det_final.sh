timeout 600 python tools/determinism_probe.py --case c2 --configs 0,1 --runs 3 > gpurun_out/r02fix_det.jsonl 2>&1
bash tools/round_check.sh r02fix
