"""Small driver for ncu: one 1M x 1M session, a few iterations of the BH or
direct force pass (plus the energy kernel).  Not a benchmark (numbers printed
under a profiler are never reported)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth
from paper_2009_14005_b200.engine import Session

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="bh", choices=["bh", "direct", "gpe", "all"])
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
ap.add_argument("--shard", default="0/1", help="r/N: template shard r of N (per-GPU work of N GPUs)")
a = ap.parse_args()
if a.mode == "all":
    for m in ("bh", "direct", "gpe"):
        os.system(f"{sys.executable} {__file__} --mode {m} --n {a.n} --iters {a.iters}")
    sys.exit(0)
x, y = synth.configs2_pair(a.n)  # bench.py's configs[2] workload
theta = 0.0 if a.mode == "direct" else 0.5
p = fga.default_params().replace(theta=theta, G=66.7 * (2000.0 / a.n) ** 0.5, conv_tol=1e-300,
                                 max_iters=a.iters + 2)
sr, sn = (int(v) for v in a.shard.split("/"))
s = Session(x, y, p, fga.RegisterOptions(compute_gpe=False, precision=a.precision), stream=0,
            shard_rank=sr, shard_count=sn)
if a.mode == "gpe":
    for _ in range(a.iters):
        s.gpe()
        print("gpe", s.take_gpe())
elif sn > 1:
    for _ in range(a.iters):  # (a shard alone: no collective, the update uses its partial sums)
        s.forces()
        s.update()
else:
    s.iterate(a.iters)
r = s.finish()
torch.cuda.synchronize()
print("ok", r.iterations, r.interactions, getattr(r, "visits_per_iter", None))
