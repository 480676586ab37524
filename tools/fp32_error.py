"""Error anatomy of the FP32 BH sum at configs[2] (1M): per-variant max
relative error on sampled queries vs the fp64 reference sum (see
tools/fp32_error.c).  Usage: python tools/fp32_error.py [n] [sample]"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402
from paper_2009_14005_b200 import synth  # noqa: E402

so = "/tmp/fp32err_%s.so" % os.environ.get("H5T", "float")
subprocess.run(["gcc", "-O2", "-DH5T=" + os.environ.get("H5T", "float"), "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC", "-o", so,
                os.path.join(ROOT, "tools", "fp32_error.c"), "-lm"], check=True)
L = ctypes.CDLL(so)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
x, y = synth.configs2_pair(n)
xn, yn, mx, my, _ = orc.setup(x.points, y.points)
t = orc.tree_build(xn, mx, 20)
idx = np.sort(np.random.default_rng(0).choice(len(yn), S, replace=False))
q = np.ascontiguousarray(yn[idx])
qm = np.ascontiguousarray(my[idx])
G = 66.7 * (2000.0 / n) ** 0.5
vp = ctypes.c_void_p
L.fp32_error.argtypes = [vp] * 6 + [ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, vp, ctypes.c_int64, vp]
P = lambda a: a.ctypes.data
# mirrored preorder index (csrc/tree.cu tree_upload_host): depth + nn - skip
nn = t.node_count
depth, skip = t.depth, np.empty(nn, np.int64)
for x_ in range(nn - 1, -1, -1):
    ch = t.children[x_][t.children[x_] >= 0]
    skip[x_] = x_ + 1 if len(ch) == 0 else skip[ch[-1]]
mir = np.ascontiguousarray(depth + nn - skip)
folds = [int(v) for v in os.environ.get("FOLDS", "0,8192,2048,512,-64").split(",")]
for fold in folds:
    out = np.zeros((S, 6, 3))
    L.fp32_error(P(t.children), P(t.com), P(t.mass), P(t.length), P(q), P(qm), S, 0.5, G, 0.04,
                 P(mir), fold, P(out))
    ref = out[:, 0]
    nr = np.linalg.norm(ref, axis=1)
    names = ["fp64", "fp32 coords+sum", "dx from fp64, fp32 sum", "fp32 terms, fp64 sum",
             "fp32 + approx rsqrt bias", f"fold {fold}"]
    for v, name in enumerate(names):
        if v == 0 or (fold != folds[0] and v < 5):
            continue
        rel = np.linalg.norm(out[:, v] - ref, axis=1) / nr
        print(f"{name:28s} max {rel.max():.2e}  p99 {np.quantile(rel, 0.99):.2e}  "
              f"median {np.median(rel):.2e}  >1e-5: {(rel > 1e-5).sum()}")
