"""Instructions executed and stall samples per CUDA source line of one kernel
in an ncu report (needs -lineinfo), for reading here.
    python tools/ncu_lines.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
path = None
line = None
src = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Function Name", "Line No"):
        continue
    if len(r) < 8:
        continue
    if r[0]:
        line = (path, r[0])
        src[line] = r[1].strip()[:80]
    try:
        ie = int(r[7] or 0)
        ss = int(r[4] or 0)
    except ValueError:
        continue
    a = agg.setdefault(line, [0, 0])
    a[0] += ie
    a[1] += ss
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"warp-instructions {ti}  samples {ts}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/ti:5.1f}%i {100*v[1]/ts:5.1f}%s {k[0]}:{k[1]:>5} {src.get(k, '')}")
