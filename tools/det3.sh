# determinism of the current code under switches: PDL off, double-buffered qkv, LN without PDL
for e in "IG_PDL=1" "IG_PDL=0" "IG_QKV_DB=1" "IG_LN_PDL=0"; do
  echo "== $e"; env $e timeout 300 python tools/determinism_probe.py --case c2 --configs 1 --runs 3
done
