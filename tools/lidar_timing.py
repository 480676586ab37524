"""configs[1] (100k LiDAR-shaped pair, G 0.2, theta 0.5): register() loop time
and per-iteration interactions (FGA_* env variables select the paths).
usage: python tools/lidar_timing.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth

x, y, gt = synth.configs1_pair()
p = fga.default_params().replace(theta=0.5, G=0.2)
fga.register(x, y, params=p)
for _ in range(2):
    t0 = time.perf_counter()
    r = fga.register(x, y, params=p, options=fga.RegisterOptions(record_iterations=True))
    w = time.perf_counter() - t0
    it = r.iterations
    print(f"wall {w*1e3:.1f} ms, iterations {it}, loop {r.timings_ms['loop']:.2f} ms "
          f"({r.timings_ms['loop']/it:.3f} ms/iter), setup {r.timings_ms['setup']:.2f}, gpe "
          f"{r.timings_ms['gpe']:.2f}; interactions/iter {np.mean(r.interactions):.4g}", flush=True)
