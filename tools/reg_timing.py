import sys, time; sys.path.insert(0, '.')
import numpy as np
import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth
rng = synth.rng_from_seed(3); x = synth.blob(1000000, rng)
y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(60), 0.1))
p = fga.default_params().replace(theta=0.5, G=66.7 * (2000 / 1e6) ** 0.5)
fga.register(x, y, params=p)
for _ in range(2):
    t0 = time.perf_counter(); r = fga.register(x, y, params=p); w = time.perf_counter() - t0
    print(round(w, 4), r.iterations, r.gpe_initial, r.gpe_final, r.timings_ms)
