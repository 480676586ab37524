import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth
from oracle import oracle as orc
rng = synth.rng_from_seed(12)
x = synth.blob(800, rng)
y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(20), 0.05))
for prec in ("fp32", "fp64"):
    res2 = fga.register(x, y, options=fga.RegisterOptions(normalize=False, record_iterations=True, precision=prec))
    ref2 = orc.register(x.points, y.points, normalize=False)
    err = np.abs(res2.trajectory - np.array(ref2.trajectory)).max(axis=(1, 2))
    print(prec, res2.iterations, ref2.iterations, "per-iter traj err", err)
