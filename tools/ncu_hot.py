"""Hot SASS windows of one kernel in an ncu report (stall samples), for reading here.
    python tools/ncu_hot.py <report.ncu-rep> [windows] [window_size]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nwin = int(sys.argv[2]) if len(sys.argv) > 2 else 6
ws = int(sys.argv[3]) if len(sys.argv) > 3 else 24
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iS, iI = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
iSrc, iA = hdr.index("Source"), hdr.index("Address")
tot = sum(int(r[iS] or 0) for r in data)
totI = sum(int(r[iI] or 0) for r in data)
print(f"samples {tot}  warp-instructions {totI}  sass lines {len(data)}")
op, opi = collections.Counter(), collections.Counter()
for r in data:
    f = r[iSrc].split()
    o = (f[1] if f and f[0].startswith("@") else (f[0] if f else "")).split(".")[0]
    op[o] += int(r[iS] or 0)
    opi[o] += int(r[iI] or 0)
print(" ".join(f"{o}:{100*v/tot:.1f}%s/{100*opi[o]/totI:.1f}%i" for o, v in op.most_common(14)))
win = sorted(((sum(int(r[iS] or 0) for r in data[k:k + ws]), k) for k in range(0, len(data), ws // 2)),
             reverse=True)
seen = set()
for s, k in win:
    if len(seen) >= nwin or any(abs(k - j) < ws for j in seen):
        continue
    seen.add(k)
    print(f"---- @{k} {100*s/tot:.1f}%")
    for r in data[k:k + ws]:
        print(f"   {r[iA][-5:]} {r[iS]:>6} {r[iI]:>9}  {r[iSrc][:86]}")
