"""configs[1] (100k LiDAR-shaped pair): register() outcome vs G (design tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
rng = synth.rng_from_seed(2)
x = synth.lidar_scan(n, rng)
gt = synth.random_rigid(rng, np.deg2rad(10), 1.0)
y = synth.misalign(x, gt)
print("extent", np.ptp(x.points, 0), "gt angle deg", np.rad2deg(np.arccos((np.trace(gt.rotation) - 1) / 2)),
      "t", gt.translation)
for G in [66.7, 66.7 * (2000.0 / n) ** 0.5, 2.0, 1.0, 0.5, 0.2]:
    for theta in [0.5]:
        p = fga.default_params().replace(theta=theta, G=G)
        r = fga.register(x, y, params=p)
        err = fga.angular_deviation(gt.rotation, r.transform.rotation)
        terr = np.linalg.norm(r.transform.translation - gt.translation)
        print(f"G={G:8.3f} theta={theta} it={r.iterations:3d} conv={r.converged} "
              f"rot_err={err:8.3f} deg t_err={terr:.3f}")
