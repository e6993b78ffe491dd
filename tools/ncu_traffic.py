"""DRAM traffic per launch of the bench's roofline kernel, from an ncu
--set full capture:  python tools/ncu_traffic.py REP.ncu-rep CONFIG KERNEL

Reads dram__bytes_read.sum + dram__bytes_write.sum and gpu__time_duration.sum
of every captured launch whose name contains KERNEL, keeps the launches with
the largest grid (level 0 of the multigrid hierarchy), and records their mean
in profiles/r01_ncu_traffic.json under CONFIG (bench.py reports it as
roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")
METRICS = "launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def _num(s):
    return float(s.replace(",", ""))


def main(rep, config, kernel):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", METRICS],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1.0, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "ns": 1e-3, "ms": 1e3,
             "msecond": 1e3}
    recs = []
    for r in rows[2:]:
        if kernel not in r[col["Kernel Name"]]:
            continue
        g = _num(r[col["launch__grid_size"]])
        rd = _num(r[col["dram__bytes_read.sum"]]) * scale[units[col["dram__bytes_read.sum"]]]
        wr = _num(r[col["dram__bytes_write.sum"]]) * scale[units[col["dram__bytes_write.sum"]]]
        us = _num(r[col["gpu__time_duration.sum"]]) * scale[units[col["gpu__time_duration.sum"]]]
        recs.append((g, rd + wr, us, r[col["Kernel Name"]]))
    if not recs:
        raise SystemExit(f"no launch of {kernel} in {rep}")
    gmax = max(r[0] for r in recs)
    top = [r for r in recs if r[0] == gmax]
    entry = {"kernel": top[0][3], "grid": int(gmax), "launches": len(top),
             "dram_bytes_per_launch": sum(r[1] for r in top) / len(top),
             "ncu_us_per_launch": sum(r[2] for r in top) / len(top),
             "source": os.path.relpath(rep, ROOT)}
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data[config] = entry
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)
    print(config, json.dumps(entry))


if __name__ == "__main__":
    main(*sys.argv[1:4])
