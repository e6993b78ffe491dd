"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import re
import sys


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


def main(path, by_grid=False):
    data = load(path)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", d["Kernel Name"])
        if by_grid:
            name += " " + d["Grid Size"]
        unit = d["Metric Unit"]
        v = float(d["Metric Value"].replace(",", ""))
        v = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    print(f"total {T:.1f} us over {sum(cnt.values())} launches")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:70s} {cnt[k]:6d} {v:10.1f} us {100 * v / T:5.1f}%  avg {v / cnt[k]:7.2f} us")


if __name__ == "__main__":
    main(sys.argv[1], by_grid=len(sys.argv) > 2)
