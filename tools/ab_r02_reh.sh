set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
tools/ab.sh r02_latereh "IG_REHEARSE_CTAS=0" "IG_REHEARSE_CTAS=1" "IG_REHEARSE_CTAS=2" "IG_REHEARSE_CTAS=4" "IG_REHEARSE_CTAS=0" "IG_REHEARSE_CTAS=2"
python tools/ab_show.py r02_latereh
