# attention work-item size: alone (attend_probe) and in the C3 step
for sg in 128 64; do IG_WP_SEG=$sg python tools/attend_probe.py > gpurun_out/r02_lateseg_probe_$sg.jsonl 2>&1; done
tools/ab.sh r02_lateseg "IG_WP_SEG=128" "IG_WP_SEG=64" "IG_WP_SEG=128" "IG_WP_SEG=64"
python tools/ab_show.py r02_lateseg
head -3 gpurun_out/r02_lateseg_probe_*.jsonl
