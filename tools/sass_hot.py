"""Hot SASS regions from `ncu -i rep --page source --csv --print-source sass` output.
    python tools/sass_hot.py sass.csv [min_samples] [window_bits]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
iv = lambda x: int(x) if x.strip().isdigit() else 0  # noqa: E731
seen, d2 = set(), []
for r in rows[2:]:
    if len(r) <= ei or not r[0].startswith("0x") or r[0] in seen:
        continue
    seen.add(r[0])
    d2.append(r)
tot = sum(iv(r[si]) for r in d2)
print("samples", tot)
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
wb = int(sys.argv[3]) if len(sys.argv) > 3 else 9
g = collections.OrderedDict()
for r in d2:
    k = int(r[0], 16) >> wb
    e = g.setdefault(k, [0, 0, "", ""])
    e[0] += iv(r[si])
    e[1] = max(e[1], iv(r[ei]))
    if iv(r[si]) > (iv(e[3].split("|")[0]) if e[3] else -1):
        e[3] = f"{iv(r[si])}|{r[1].strip()[:60]}"
for k, (s, e, _, top) in g.items():
    if s >= mn:
        print(f"{hex(k << wb)[-5:]} {s:6d} ({100 * s / tot:4.1f}%) exec {e:8d}  top: {top}")
