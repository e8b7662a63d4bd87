# Ax timings of library variants (dirs under paper_1905_03748_b200/_lib):
#   bash tools/ab_fwd_variants.sh OUT.jsonl variant...
out=$1; shift
for v in "$@"; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so python tools/ab_fwd.py "$v" /tmp/ab_$v.npy >> $out
done
python - "$@" <<'PY' >> $out
import sys, json, numpy as np
ref = np.load(f"/tmp/ab_{sys.argv[1]}.npy")
for v in sys.argv[2:]:
    b = np.load(f"/tmp/ab_{v}.npy")
    print(json.dumps({"variant": v, "relL2_vs_" + sys.argv[1]: float(np.linalg.norm((ref - b).ravel()) / np.linalg.norm(ref.ravel()))}))
PY
rm -f /tmp/ab_*.npy
