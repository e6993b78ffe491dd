"""Compact per-launch summary of an ncu --set full capture exported with
``ncu -i REP --page raw --csv``: duration, grid, registers, occupancy, FP64
pipe and issue activity, DRAM bytes and the fraction of the measured HBM peak
(MEASURED_PEAKS.json).

  python tools/ncu_summary.py RAW.csv [--label text] > profiles/rNN_ncu_full_<what>.csv
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COLS = [
    ("us", "gpu__time_duration.sum"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("regs", "launch__registers_per_thread"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("occ_limit_regs", "launch__occupancy_limit_registers"),
    ("occ_limit_smem", "launch__occupancy_limit_shared_mem"),
    ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("l1tex_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("dram_read_MB", "dram__bytes_read.sum"),
    ("dram_write_MB", "dram__bytes_write.sum"),
]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3,
         "us": 1.0, "ns": 1e-3, "ms": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    w = csv.writer(sys.stdout)
    if a.label:
        print(f"# {a.label}; HBM peak {peak:.1f} GB/s (MEASURED_PEAKS.json)")
    w.writerow(["kernel"] + [c for c, _ in COLS] + ["dram_GBps", "frac_hbm"])
    for r in rows[2:]:
        out, vals = [r[col["Kernel Name"]].split("(")[0]], {}
        for name, m in COLS:
            if m not in col or not r[col[m]]:
                out.append("")
                continue
            v = float(r[col[m]].replace(",", ""))
            v *= SCALE.get(units[col[m]], 1.0)
            vals[name] = v
            out.append(f"{v:.4g}")
        if "us" in vals and "dram_read_MB" in vals:
            gbs = (vals["dram_read_MB"] + vals.get("dram_write_MB", 0.0)) * 1e-3 / (vals["us"] * 1e-6)
            out += [f"{gbs:.1f}", f"{gbs / peak:.3f}"]
        w.writerow(out)


if __name__ == "__main__":
    main()
