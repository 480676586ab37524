"""1M x 1M FP32 energy pass (Session.gpe) wall time, 3 reps (design tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth
from paper_2009_14005_b200.engine import Session

rng = synth.rng_from_seed(3)
x = synth.blob(1_000_000, rng)
y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(60), 0.1))
s = Session(x, y, fga.default_params().replace(theta=0.5), fga.RegisterOptions(compute_gpe=False))
s.gpe()
s.take_gpe()
for _ in range(3):
    t = time.perf_counter()
    s.gpe()
    v = s.take_gpe()
    print(f"gpe {time.perf_counter() - t:.4f} s  {v!r}")
