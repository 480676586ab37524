"""configs[3] (200k partial overlap, kNN-16 masses, G 2, theta 0.5):
register() loop time (FGA_LIB_PATH / FGA_* select the paths).  usage: python tools/c4_timing2.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth

x, y, gt = synth.configs3_pair()
p = fga.default_params().replace(theta=0.5, G=2.0)
o = fga.RegisterOptions(mass_field="knn", knn_k=16, record_iterations=True)
fga.register(x, y, params=p, options=o)
for _ in range(2):
    t0 = time.perf_counter()
    r = fga.register(x, y, params=p, options=o)
    w = time.perf_counter() - t0
    print(f"wall {w*1e3:.1f} ms, iterations {r.iterations}, loop {r.timings_ms['loop']:.2f} ms "
          f"({r.timings_ms['loop']/r.iterations:.3f} ms/iter); interactions/iter "
          f"{np.mean(r.interactions):.4g}", flush=True)
