"""configs[0] (2k x 2k blob pair) register() wall time and its phases, next to
the batched kernel on the same pair (P = 1).  usage: python tools/c0_timing.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth

pairs = []
for s in range(20):
    rng = synth.rng_from_seed(s)
    x = synth.blob(2000, rng)
    pairs.append((x, synth.misalign(x, synth.random_rigid(rng, np.deg2rad(60), 0.1))))
p = fga.default_params().replace(theta=0.5)
fga.register(*pairs[0], params=p)
fga.register_batch([pairs[0]], params=p)
for name, fn in (("register", lambda a, b: fga.register(a, b, params=p)),
                 ("batch1", lambda a, b: fga.register_batch([(a, b)], params=p).results[0])):
    w, its = [], []
    for x, y in pairs:
        t0 = time.perf_counter()
        r = fn(x, y)
        w.append(time.perf_counter() - t0)
        its.append(r.iterations)
    print(name, "median ms %.3f" % (1e3 * np.median(w)), "iters", its[:6],
          getattr(r, "timings_ms", None), flush=True)
