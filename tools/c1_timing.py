"""configs[0]-shaped registrations (2k blob, theta 0.5): wall time per
register() call on the GPU path (design tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth

p = fga.default_params().replace(theta=0.5)
pairs = []
for s in range(20):
    rng = synth.rng_from_seed(s)
    x = synth.blob(2000, rng)
    pairs.append((x, synth.misalign(x, synth.random_rigid(rng, np.deg2rad(60), 0.1))))
fga.register(*pairs[0], params=p)
walls, its, tms = [], [], []
for x, y in pairs:
    t0 = time.perf_counter()
    r = fga.register(x, y, params=p)
    walls.append(time.perf_counter() - t0)
    its.append(r.iterations)
    tms.append(r.timings_ms)
print(f"C1 register(): median {1e3*np.median(walls):.2f} ms, iterations median {np.median(its)}, "
      f"per-iteration {1e3*np.median(np.array(walls)/np.array(its)):.3f} ms")
print("timings_ms (first):", tms[0])
t0 = time.perf_counter()
br = fga.register_batch(pairs, params=p)
print(f"batched 20 pairs: {1e3*(time.perf_counter()-t0):.2f} ms")
