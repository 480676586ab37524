"""Time fga_register_batch on config-5-shaped pairs (not the bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth

P = int(sys.argv[1]) if len(sys.argv) > 1 else 512
pairs = []
for p in range(P):
    rng = synth.rng_from_seed(100000 + p)
    x = synth.blob(4096, rng) if p % 2 == 0 else synth.bumped_box(4096, rng)
    pairs.append((x, synth.misalign(x, synth.random_rigid(rng, np.deg2rad(60), 0.1))))
fga.register_batch(pairs[:16])
t0 = time.perf_counter()
br = fga.register_batch(pairs)
dt = time.perf_counter() - t0
its = np.array([r.iterations for r in br.results if r is not None])
print(f"{P} pairs in {dt:.3f} s -> {P/dt:.1f} pairs/s; iterations min/median/max "
      f"{its.min()}/{np.median(its)}/{its.max()}; interactions/s {br.interactions.sum()/dt:.3e}; "
      f"errors {sum(e is not None for e in br.errors)}")
t0 = time.perf_counter()
for x, y in pairs[:32]:
    fga.register(x, y)
d1 = time.perf_counter() - t0
print(f"single-pair path: {32/d1:.1f} pairs/s")
