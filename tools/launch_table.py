"""Summarise an ncu --csv launch list (gpu__time_duration.sum and optional
dram bytes): per kernel name, launches, total/mean us, DRAM MB; optionally
only the last `--last K` launches."""
import argparse
import collections
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--skip", type=int, default=0, help="skip the first N launches")
ap.add_argument("--seq", action="store_true", help="print the launch sequence")
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ii = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                  hdr.index("ID"))
L = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    d = L.setdefault(int(r[ii]), {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
seq = [v for k, v in sorted(L.items())][a.skip:]
agg = collections.OrderedDict()
for d in seq:
    nm = d["name"].split("(")[0].replace("fga::<unnamed>::", "")[:60]
    g = agg.setdefault(nm, [0, 0.0, 0.0])
    g[0] += 1
    g[1] += d.get("gpu__time_duration.sum", 0.0) / 1e3
    g[2] += (d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)) / 1e6
tot = sum(g[1] for g in agg.values())
if a.seq:
    for d in seq:
        print(f'{d["name"].split("(")[0][-50:]:50s} {d.get("gpu__time_duration.sum", 0)/1e3:9.1f} us')
print(f"{'kernel':60s} {'n':>4s} {'total us':>10s} {'share':>6s} {'DRAM MB':>9s}")
for nm, (n, t, b) in agg.items():
    print(f"{nm:60s} {n:4d} {t:10.1f} {100*t/tot:5.1f}% {b:9.1f}")
print(f"total {tot:.1f} us")
