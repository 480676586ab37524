"""The bench's e2e leg alone (fga_tree_forces from pinned host buffers on the
configs[2] initial state), wall clock per call; under ncu it gives the
call's launch list.  usage: python tools/e2e_timing.py [calls]
E2E_SHARDS=N: also time each rank's slice of an N-way run (bench.py run_e2e)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import _native as N
from paper_2009_14005_b200 import bhtree, synth

K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
x, y = synth.configs2_pair(1_000_000, 3)
xn, yn, ctx = fga.normalize_pair(x, y, -5.0, 5.0)
p = fga.default_params().replace(theta=0.5, G=66.7 * (2000.0 / 1e6) ** 0.5)
sx = fga.niv_masses(xn, 16, ctx, 20)
sy = fga.niv_masses(yn, 16, ctx, 20)
mx = np.minimum(16.0 * np.sqrt(len(sx) / 2000) * sx / sx.sum(), 0.022)
my = np.maximum(0.1 * sy / sy.max(), max(1e-6, p.dt * p.eta))
c = N.context(0)
bhtree.build(xn, mx, 20)
M = len(yn)


def pinned(shape, dtype):
    return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()


L = N.lib()
with_acc = os.environ.get("E2E_ACC", "1") == "1"


def morton_order(p, bits=10):
    """host-side spatial partition order (30-bit Morton key of the points)"""
    lo, ext = p.min(0), np.ptp(p, 0).max()
    g = np.clip(((p - lo) / ext * ((1 << bits) - 1)).astype(np.uint64), 0, (1 << bits) - 1)
    key = np.zeros(len(p), np.uint64)
    for b in range(bits):
        for a in range(3):
            key |= ((g[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + 2 - a)
    return np.argsort(key, kind="stable")


PART = os.environ.get("E2E_PART", "slice")  # slice | morton
perm = morton_order(yn.points) if PART == "morton" else np.arange(M)


def run(lo, hi, label):
    m = hi - lo
    sel = perm[lo:hi]
    q = pinned((m, 3), torch.float64)
    q[:] = yn.points[sel]
    qm = pinned((m,), torch.float64)
    qm[:] = my[sel]
    f = pinned((m, 3), torch.float64)
    vis = pinned((m,), torch.int64)
    acc = pinned((m,), torch.int64)
    ts = []
    for k in range(K + 2):
        t0 = time.perf_counter()
        N.check(L.fga_tree_forces(c.handle, N.ptr(q), N.ptr(qm), m, 0.5, float(p.G), 0.04,
                                  N.PREC_FP32, N.ptr(f), N.ptr(vis),
                                  N.ptr(acc) if with_acc else None))
        ts.append(time.perf_counter() - t0)
    print("%s e2e call ms median %.3f min %.3f" % (label, 1e3 * np.median(ts[2:]),
                                                   1e3 * min(ts[2:])), flush=True)
    return np.median(ts[2:])


S = int(os.environ.get("E2E_SHARDS", "0"))
only = os.environ.get("E2E_SHARD_ONLY")  # one shard (e.g. under ncu)
if only is None:
    run(0, M, "full")
if S > 1:
    ranks = [int(only)] if only is not None else range(S)
    t = [run(M * r // S, M * (r + 1) // S, "shard %d/%d" % (r, S)) for r in ranks]
    print("max over %d shards %.3f ms" % (S, 1e3 * max(t)))
