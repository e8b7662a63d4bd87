# Ax kernel variants at config 2: bash tools/ab_occ.sh variant... (dirs under _lib)
for v in "$@"; do
 for ml in 0 1; do
  CS_LIB_PATH=$PWD/paper_1905_03748_b200/_lib/$v/libconesplit_b200.so CS_FWD_MLAYER=$ml python tools/ab_fwd.py "$v-ml$ml" /tmp/ab_$v-ml$ml.npy
 done
done
python - "$@" <<'PY'
import sys, numpy as np
ref = np.load("/tmp/ab_.-ml0.npy")
for v in sys.argv[1:]:
    b = np.load(f"/tmp/ab_{v}-ml1.npy")
    print(v, "ml1 vs production relL2", float(np.linalg.norm((ref - b).ravel()) / np.linalg.norm(ref.ravel())))
PY
rm -f /tmp/ab_*.npy
