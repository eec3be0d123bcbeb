for e in "IG_DBG_SYNC=none" "IG_DBG_SYNC=att_after_sp" "IG_DBG_SYNC=att_after_fs" "IG_DBG_SYNC=plan_after_c" "IG_DBG_SYNC=fs_after_c"; do
  echo "== $e"; env $e timeout 300 python tools/determinism_probe.py --case c2 --configs 1 --runs 3
done
