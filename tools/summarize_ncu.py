"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

    python tools/summarize_ncu.py <launches.csv> <full.ncu-rep> <out.md> [traffic.json]

launches.csv: `ncu --metrics gpu__time_duration.sum --csv --log-file` of the
bench command (cold-cache, serialised: compare SHARES, not absolutes).
full.ncu-rep: `ncu --set full` capture of the hot kernels.
"""
import csv
import json
import re
import subprocess
import sys
from collections import OrderedDict

UNITS = {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
         "s": 1e9, "second": 1e9}


def kname(s):
    s = re.sub(r"\(.*", "", s).replace("void ", "")
    return s.replace("fga::<unnamed>::", "").replace("fga::", "")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h, data = rows[0], rows[1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    tot = 0.0
    for r in data:
        try:
            v = float(r[iv].replace(",", "")) * UNITS.get(r[iu], 1)
        except ValueError:
            continue
        k = kname(r[ik])[:70]
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + v)
        tot += v
    return agg, tot


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        item = {"kernel": kname(d.get("Kernel Name", "?"))}
        for m, label in METRICS:
            if m in d and d[m] not in ("", "-nan", "nan"):
                item[label] = f"{d[m]} {u.get(m, '')}".strip()
        res.append(item)
    return res


def main():
    lpath, fpath, out = sys.argv[1:4]
    agg, tot = launches(lpath)
    lines = ["# ncu summary", "", f"Launch list: `{lpath}` (gpu__time_duration.sum, cold-cache, "
             "serialised).", "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if t / tot < 0.0005:
            continue
        lines.append(f"| `{k}` | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
    lines += ["", f"Total {tot / 1e6:.1f} ms.", "", f"## Full captures (`{fpath}`)", ""]
    for item in full(fpath):
        lines.append(f"### `{item.pop('kernel')}`")
        for k, v in item.items():
            lines.append(f"- {k}: {v}")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
