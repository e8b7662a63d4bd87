"""Per-source-line totals from an ncu report (cuda,sass source page):
instructions executed and warp-stall samples, top lines first.

    python tools/ncu_lines.py report.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                          "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    fname = func = None
    hdr = None
    agg = {}
    cur = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or (want and want not in (func or "")):
            continue
        if not r[0]:
            continue  # SASS rows: the line row above already sums them
        cur = (fname, int(r[0]), r[1][:70])
        try:
            ie = float(r[hdr["Instructions Executed"]] or 0)
            st = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (KeyError, ValueError):
            continue
        a = agg.setdefault(cur, [0.0, 0.0])
        a[0] += ie
        a[1] += st
    tot_i = sum(v[0] for v in agg.values()) or 1
    tot_s = sum(v[1] for v in agg.values()) or 1
    print(f"total warp-inst {tot_i:.3e}  stall samples {tot_s:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100*v[0]/tot_i:5.1f}% inst {100*v[1]/tot_s:5.1f}% stall  "
              f"{k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
