"""Summarise ncu --set full reports into profiles/: a markdown table per
kernel (time, DRAM bytes, L1/L2 hit rates, pipe utilisation, limiter) and
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py).

    python tools/ncu_summary.py TAG report1.ncu-rep [report2 ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1/TEX hit %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX thru %"),
    ("l1tex__tex_writeback_active.avg.pct_of_peak_sustained_elapsed",
     "TEX writeback %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 thru %"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 RED requests"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp insts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
     "ATOMS wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
     "ATOMS bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
]
# kernel-name fragment -> bench key.  One Ax call on main-axis layers is
# fill_xlayers + fwd_mlayer<.., 0> + fill_ylayers + fwd_mlayer<.., 1>: the
# fills count in its DRAM traffic, only the projector in its pipe limits.
KEYS = {"fwd_mlayer": "fwd_mlayer_kernel", "fill_xlayers": "fwd_mlayer_kernel",
        "fill_ylayers": "fwd_mlayer_kernel",
        "fwd_interp": "fwd_interp_kernel",
        "staged_kernel<1": "bwd_matched_kernel",
        "transpose_add": "bwd_matched_kernel",
        "bwd_fdk": "bwd_fdk_kernel", "fdk_staged": "bwd_fdk_kernel",
        "fwd_siddon": "fwd_siddon_kernel",
        "tv_march2_kernel<1": "tv_gd_fused_kernel",
        "tv_march2_kernel<0": "tv_grad_kernel",
        "tv_march2_tma_kernel<1": "tv_gd_fused_kernel",
        "tv_march2_tma_kernel<0": "tv_grad_kernel",
        "rof_march2": "rof_iter_kernel"}


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
             "Tbyte": 1e12}
    return float(v) * scale.get(unit, 1)


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    rows_out = []
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        traffic = json.load(open(traffic_path))
    except (OSError, ValueError):
        traffic = {}
    sums = {}
    for rep in reps:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        hdr, units, data = rows[0], rows[1], rows[2:]
        idx = {h: i for i, h in enumerate(hdr)}
        for r in data:
            name = r[idx["Kernel Name"]]
            rec = {"kernel": name.split("(")[0], "report": os.path.basename(rep)}
            for m, label in METRICS:
                if m in idx:
                    rec[label] = (r[idx[m]], units[idx[m]])
            rows_out.append(rec)
            for k, key in KEYS.items():
                if k in name and "dram read" in rec:
                    try:
                        rd = to_bytes(*rec["dram read"])
                        wr = to_bytes(*rec["dram write"])
                    except ValueError:
                        continue
                    if rd == rd and wr == wr:  # skip failed (nan) captures
                        # one C-ABI call may be several kernels (staged
                        # matched = x-major + y-major views): sum them
                        sums[key] = sums.get(key, 0.0) + rd + wr
    traffic.update(sums)
    # pipe limiters per kernel key (bench.py reports them beside the HBM
    # roofline of the dominant kernel)
    lim_path = os.path.join(ROOT, "profiles", "ncu_limits.json")
    try:
        limits = json.load(open(lim_path))
    except (OSError, ValueError):
        limits = {}
    for rec in rows_out:
        for k, key in KEYS.items():
            if (k not in rec["kernel"] or k.startswith("fill_")
                    or k == "transpose_add"):
                continue
            ent = {}
            for label in ("TEX writeback %", "issue active %", "L1/TEX thru %",
                          "dram %"):
                if label in rec:
                    try:
                        v = float(rec[label][0])
                    except ValueError:
                        continue
                    if v == v:
                        ent[label] = v
            if ent:
                ent["report"] = f"profiles/ncu_{tag}.md"
                limits[key] = ent
    with open(lim_path, "w") as f:
        json.dump(limits, f, indent=1)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md = [f"# ncu --set full summary ({tag})", "",
          "Captured with `ncu --set full --clock-control none --import-source on`"
          " on one B200 (tools/prof_c2.py replays bench.py's launches).", ""]
    for rec in rows_out:
        md.append(f"## {rec['kernel']}  ({rec['report']})")
        md.append("")
        md.append("| metric | value |")
        md.append("|---|---|")
        for _, label in METRICS:
            if label in rec:
                v, u = rec[label]
                md.append(f"| {label} | {v} {u} |")
        md.append("")
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
