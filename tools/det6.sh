for e in "IG_DBG_NONE=1" "IG_DBG_CV=1"; do
  echo "== $e"; env $e timeout 300 python tools/determinism_probe.py --case c2 --configs 1,0 --runs 3
done
