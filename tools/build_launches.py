"""Per-launch table of the LAST build in an ncu launch list (tools/prof_build.py
runs 2 builds): name, us, DRAM read/write MB, and the build total."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
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
seq = [v for _, v in sorted(L.items())]
starts = [j for j, d in enumerate(seq) if "k_bbox_partial" in d["name"]]
last = seq[starts[-1]:]
tot = rb = wb = 0.0
agg = collections.OrderedDict()
for d in last:
    nm = d["name"].split("(")[0].replace("fga::<unnamed>::", "").split("<")[0][-34:]
    t = d["gpu__time_duration.sum"] / 1e3
    r = d.get("dram__bytes_read.sum", 0) / 1e6
    w = d.get("dram__bytes_write.sum", 0) / 1e6
    g = agg.setdefault(nm, [0, 0.0, 0.0, 0.0])
    g[0] += 1; g[1] += t; g[2] += r; g[3] += w
    tot += t; rb += r; wb += w
for nm, (c, t, r, w) in agg.items():
    print(f"{nm:36s} x{c:<3d} {t:9.1f} us  R {r:8.1f} MB  W {w:8.1f} MB")
print(f"{'build total':36s}      {tot:9.1f} us  R {rb:8.1f} MB  W {wb:8.1f} MB")
