"""Summarise an ncu --csv launch list by kernel: time share, and -- when the
capture has dram__bytes_read.sum / dram__bytes_write.sum -- the DRAM bytes
each kernel moved, its achieved GB/s and the fraction of the measured HBM
peak (MEASURED_PEAKS.json), plus the same for the whole step.

  python tools/launch_summary.py launches.csv [--by-grid]
"""
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1.0, "B": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def main(path, by_grid=False):
    data = load(path)
    t = collections.defaultdict(float)
    b = collections.defaultdict(float)
    cnt = collections.Counter()
    have_bytes = False
    for d in data:
        name = re.sub(r"\(.*", "", d["Kernel Name"])
        if by_grid:
            name += " " + d["Grid Size"]
        m, unit = d["Metric Name"], d["Metric Unit"]
        v = float(d["Metric Value"].replace(",", ""))
        if m == "gpu__time_duration.sum":
            t[name] += v * TIME[unit]
            cnt[name] += 1
        elif m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b[name] += v * BYTES[unit]
            have_bytes = True
    T = sum(t.values())
    pk = peak_gbs()
    head = f"total {T:.1f} us over {sum(cnt.values())} launches"
    if have_bytes:
        B = sum(b.values())
        head += f"; DRAM {B / 1e9:.3f} GB -> {B / T / 1e3:.0f} GB/s = {B / T / 1e3 / pk:.2f} of {pk:.0f} GB/s (whole step)"
    print(head)
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        line = f"{k:62s} {cnt[k]:6d} {v:10.1f} us {100 * v / T:5.1f}%  avg {v / cnt[k]:8.2f} us"
        if have_bytes:
            gbs = b[k] / v / 1e3 if v > 0 else 0.0
            line += f"  {gbs:6.0f} GB/s {gbs / pk:5.2f}"
        print(line)


if __name__ == "__main__":
    main(sys.argv[1], by_grid="--by-grid" in sys.argv[2:])
