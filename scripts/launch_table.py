"""Per-kernel totals from an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]).

usage: python scripts/launch_table.py launches.csv [top]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = collections.defaultdict(dict)
    name = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name[r[ii]] = r[ki]
    agg = collections.OrderedDict()
    for i, m in per.items():
        k = name[i][:70]
        a = agg.setdefault(k, [0.0, 0, 0.0])
        a[0] += m.get("gpu__time_duration.sum", 0.0)
        a[1] += 1
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[0] for a in agg.values())
    print(f"total {tot:.1f} us over {len(per)} launches")
    for k, (t, n, b) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{t:9.1f} us {n:3d}x {b / 1e6:9.1f} MB  {k}")


if __name__ == "__main__":
    main()
