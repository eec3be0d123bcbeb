for e in "IG_DBG_SYNC=none" "IG_DBG_SYNC=app_after_fs" "IG_DBG_SYNC=gemm_after_fs"; do
  echo "== $e"; env $e timeout 300 python tools/determinism_probe.py --case c2 --configs 1,0 --runs 3
done
