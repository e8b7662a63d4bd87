# A/B of the z-layered (production) and main-axis-layered Ax kernels at
# config 2: timings, outputs compared, GPU tests under CS_FWD_MLAYER=1, and
# an ncu instruction / texture summary of one 90-view launch of each.
mkdir -p gpurun_out/ab
for i in 1 2; do
CS_FWD_MLAYER=0 python tools/ab_fwd.py zlayer gpurun_out/ab/z.npy
CS_FWD_MLAYER=1 python tools/ab_fwd.py mlayer gpurun_out/ab/m.npy
done
python - <<'PY'
import numpy as np
for suf in ("", "_slab"):
    a = np.load(f"gpurun_out/ab/z{suf}.npy"); b = np.load(f"gpurun_out/ab/m{suf}.npy")
    print(suf, "relL2 m vs z", float(np.linalg.norm((a-b).ravel())/np.linalg.norm(a.ravel())))
PY
rm -f gpurun_out/ab/*.npy
[ "$1" = "tests" ] && CS_FWD_MLAYER=1 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
M=gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_elapsed
CS_FWD_MLAYER=1 PROF_A=90 ncu -k regex:"fwd_|fill_" --metrics $M --clock-control none -c 4 --csv --log-file gpurun_out/ab/ml.csv python tools/ab_fwd.py m /tmp/m.npy > /dev/null 2>&1
CS_FWD_MLAYER=0 PROF_A=90 ncu -k regex:"fwd_|fill_" --metrics $M --clock-control none -c 1 --csv --log-file gpurun_out/ab/z.csv python tools/ab_fwd.py z /tmp/z.npy > /dev/null 2>&1
python - <<'PY'
import csv
for f in ("gpurun_out/ab/ml.csv", "gpurun_out/ab/z.csv"):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]
    for r in rows[1:]:
        print(r[h.index("ID")], r[h.index("Kernel Name")][:32], r[h.index("Metric Name")], r[h.index("Metric Value")])
PY
