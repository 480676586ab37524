"""bh_forces operator (fga_tree_forces) on a 1M-point tree and 1M queries,
host numpy in/out, fp32 and fp64, 3 reps each (design tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import bhtree, synth

rng = synth.rng_from_seed(3)
x = synth.blob(1_000_000, rng)
y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(60), 0.1))
xn, yn, _ = fga.normalize_pair(x, y, -5.0, 5.0)
tree = bhtree.build(xn, np.full(len(x), 0.01), 20)
p = fga.default_params().replace(theta=0.5)
qm = np.full(len(y), 0.05)
for prec in ("fp32", "fp64"):
    bhtree.bh_forces(tree, yn.points, qm, p, precision=prec)
    for _ in range(3):
        t = time.perf_counter()
        bhtree.bh_forces(tree, yn.points, qm, p, precision=prec)
        print(prec, f"{time.perf_counter() - t:.4f} s")
