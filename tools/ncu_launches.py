"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes) per kernel name.
    python tools/ncu_launches.py launches.csv [--order]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
data = collections.OrderedDict()
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    d = data.setdefault(r[ii], {"k": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
if "--order" in sys.argv:
    for i, d in data.items():
        t = d.get("gpu__time_duration.sum", 0) / 1e3
        b = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
        print(f"{i:>4} {t:9.1f} us {b:9.1f} MB  {d['k'][:110]}")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for d in data.values():
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    b = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    a = agg[d["k"][:110]]
    a[0] += 1
    a[1] += t
    a[2] += b
    tot += t
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:4d} x {t / c:8.1f} us = {t:9.1f} us ({100 * t / tot:4.1f}%)  {b / c:8.1f} MB/launch  {b / t:6.2f} GB/ms  {n}")
print(f"total {tot:.1f} us")
