"""kNN (fga_knn_masses) timing on configs[3]-shaped data and a uniform blob
(design tool, not the bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2009_14005_b200 import masses, synth

rng = synth.rng_from_seed(4)
x, _ = synth.partial_overlap(200_000, rng)
u = synth.blob(1_000_000, synth.rng_from_seed(3))
for name, c in (("c4_200k", x), ("blob_1M", u)):
    masses.knn_masses(c, 16)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        masses.knn_masses(c, 16)
        ts.append(time.perf_counter() - t0)
    print(f"{name}: knn_masses k=16 median {1e3*np.median(ts):.2f} ms")
