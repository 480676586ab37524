"""configs[3] (200k partial overlap, kNN-16 masses): register() outcome vs G
(design tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth

rng = synth.rng_from_seed(4)
x, y0 = synth.partial_overlap(200_000, rng)
gt = synth.random_rigid(rng, np.deg2rad(60), 0.1)
y = synth.misalign(y0, gt)
print("gt angle deg", np.rad2deg(np.arccos((np.trace(gt.rotation) - 1) / 2)))
for mf in ["knn", "niv"]:
    for G in [66.7 * (2000.0 / 200_000) ** 0.5, 2.0, 1.0, 0.5, 0.2, 0.05]:
        p = fga.default_params().replace(theta=0.5, G=G)
        o = fga.RegisterOptions(mass_field=mf, knn_k=16)
        r = fga.register(x, y, params=p, options=o)
        err = fga.angular_deviation(gt.rotation, r.transform.rotation)
        terr = np.linalg.norm(r.transform.translation - gt.translation)
        print(f"{mf} G={G:8.3f} it={r.iterations:3d} conv={r.converged} rot_err={err:8.3f} deg "
              f"t_err={terr:.4f}")
