"""configs[3] registrations (200k partial overlap): wall and setup per call,
kNN-16 and NIV masses, repeated (design tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth

rng = synth.rng_from_seed(4)
x, y0 = synth.partial_overlap(200_000, rng)
gt = synth.random_rigid(rng, np.deg2rad(60), 0.1)
y = synth.misalign(y0, gt)
p = fga.default_params().replace(theta=0.5, G=2.0)
for name, o in [("knn16", fga.RegisterOptions(mass_field="knn", knn_k=16)),
                ("niv", fga.RegisterOptions())] * 3:
    t0 = time.perf_counter()
    r = fga.register(x, y, params=p, options=o)
    print(name, f"wall {time.perf_counter() - t0:.4f}", {k: round(v, 2) for k, v in r.timings_ms.items()},
          r.iterations)
