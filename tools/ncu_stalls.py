"""Stall reasons per SASS range of an ncu report: python tools/ncu_stalls.py rep lo hi [top]"""
import collections, csv, io, subprocess, sys
rep, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: hdr.index(c) for c in cols}
iSrc, iI = hdr.index("Source"), hdr.index("Instructions Executed")
agg = collections.Counter()
per = []
for k in range(lo, min(hi, len(data))):
    r = data[k]
    tot = 0
    for c in cols:
        v = int(r[idx[c]] or 0)
        agg[c] += v
        if c != "stall_barrier":
            tot += v
    per.append((tot, k, r[iSrc][:70], r[iI], {c: int(r[idx[c]] or 0) for c in cols if int(r[idx[c]] or 0)}))
S = sum(agg.values())
print(" ".join(f"{c[6:]}:{100*v/S:.1f}%" for c, v in agg.most_common(10)))
for tot, k, src, ins, d in sorted(per, reverse=True)[:top]:
    print(f"{k:5d} {tot:6d} {ins:>9} {src:70s} {dict(sorted(d.items(), key=lambda x:-x[1])[:3])}")
