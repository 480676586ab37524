"""Key metrics of one kernel from an `ncu --page raw --csv` export.
    python tools/ncu_metrics.py gpurun_out/bh_raw.csv [--json]"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2]
get = dict(zip(hdr, vals))
unit = dict(zip(hdr, units))
want = {
    "kernel": "Kernel Name",
    "duration_ns": "gpu__time_duration.sum",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts_sectors": "lts__t_sectors.sum",
    "lts_sectors_srcunit_tex": "lts__t_sectors_srcunit_tex.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fp32_pipe_pct": "sm__pipe_fp32_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__pipe_lsu_cycles_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
}
out = {}
for k, name in want.items():
    if name in get:
        v = get[name].replace(",", "")
        try:
            v = float(v)
            u = unit.get(name, "")
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "msecond": 1e6,
                     "usecond": 1e3, "nsecond": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}.get(u)
            if scale:
                v *= scale
        except ValueError:
            pass
        out[k] = v
if "--json" in sys.argv:
    print(json.dumps(out, indent=1))
else:
    for k, v in out.items():
        print(f"{k:26s} {v}")
