"""Split passes of small template shards (forces.cu k_bh_split): after a
first pass that records every warp's node trace, each warp's traversal runs
as FGA_SPLIT_PARTS warps over fold-chunk-aligned node ranges.  Every fp32
chunk sum is the unsplit pass's, so the trajectory equals the unsplit run's
to fp64 regrouping and the accepted interactions are identical; both agree
with the oracle.  GPU only (the unsplit run is a subprocess with FGA_SPLIT=0)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth
rng = synth.rng_from_seed(41)
x = synth.blob(40000, rng)
y = synth.misalign(synth.blob(20000, synth.rng_from_seed(42)), synth.random_rigid(rng, 0.5, 0.05))
p = fga.default_params().replace(theta=0.5, G=66.7 * (2000 / 40000) ** 0.5, max_iters=12,
                                 conv_tol=1e-300)
r = fga.register(x, y, params=p, options=fga.RegisterOptions(record_iterations=True))
print(json.dumps({"traj": r.trajectory.tolist(), "inter": r.interactions.tolist(),
                  "it": r.iterations}))
""" % ROOT


def _run(split):
    env = dict(os.environ, FGA_SPLIT="1" if split else "0", FGA_SPLIT_LOG="1")
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert ("[fga] split pass" in out.stderr) == split  # the split passes did run
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_split_passes_match_unsplit_and_oracle(orc):
    a, b = _run(True), _run(False)
    assert a["it"] == b["it"] == 12
    assert a["inter"] == b["inter"]
    ta, tb = np.array(a["traj"]), np.array(b["traj"])
    # fold-chunk-aligned parts: the fp32 chunk sums are the unsplit ones and
    # their fp64 regrouping is exact here (24-bit terms), so the runs agree
    assert np.abs(ta - tb).max() < 1e-10
    from paper_2009_14005_b200 import synth
    rng = synth.rng_from_seed(41)
    x = synth.blob(40000, rng)
    y = synth.misalign(synth.blob(20000, synth.rng_from_seed(42)),
                       synth.random_rigid(rng, 0.5, 0.05))
    ref = orc.register(x.points, y.points, theta=0.5, G=66.7 * (2000 / 40000) ** 0.5,
                       max_iters=12, conv_tol=1e-300)
    assert np.abs(ta - np.array(ref.trajectory)).max() < 1e-5


LPT_SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth
rng = synth.rng_from_seed(43)
x = synth.blob(150000, rng)
y = synth.misalign(synth.blob(150000, synth.rng_from_seed(44)), synth.random_rigid(rng, 0.5, 0.05))
p = fga.default_params().replace(theta=0.5, G=66.7 * (2000 / 150000) ** 0.5, max_iters=6,
                                 conv_tol=1e-300)
r = fga.register(x, y, params=p, options=fga.RegisterOptions(record_iterations=True))
print(json.dumps({"traj": r.trajectory.tolist(), "inter": r.interactions.tolist()}))
""" % ROOT


def test_heaviest_first_order_changes_nothing():
    """Multi-wave passes launch their blocks heaviest first after the first
    pass (k_bh_iterate with `order`): the partial-sum slots are unchanged,
    so the run equals the in-order one bit for bit (FGA_LPT=0)."""
    outs = []
    for lpt in ("1", "0"):
        env = dict(os.environ, FGA_LPT=lpt)
        out = subprocess.run([sys.executable, "-c", LPT_SCRIPT], env=env, capture_output=True,
                             text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(json.loads(out.stdout.strip().splitlines()[-1]))
    assert outs[0]["inter"] == outs[1]["inter"]
    assert np.array_equal(np.array(outs[0]["traj"]), np.array(outs[1]["traj"]))


SWEEP_SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2009_14005_b200 as fga
from paper_2009_14005_b200 import synth
out = {}
for n, m in ((3000, 1500), (60000, 20000), (60000, 140000), (120000, 280000)):
    rng = synth.rng_from_seed(n + m)
    x = synth.blob(n, rng)
    y = synth.misalign(synth.blob(m, synth.rng_from_seed(m)), synth.random_rigid(rng, 0.4, 0.05))
    p = fga.default_params().replace(theta=0.5, G=66.7 * (2000 / n) ** 0.5, max_iters=5,
                                     conv_tol=1e-300)
    r = fga.register(x, y, params=p, options=fga.RegisterOptions(record_iterations=True))
    out["%%d_%%d" %% (n, m)] = {"traj": r.trajectory.tolist(), "inter": r.interactions.tolist()}
print(json.dumps(out))
""" % ROOT


def test_pass_schedules_agree_across_sizes():
    """Every pass schedule (shared-memory small tree, split passes, heaviest-
    first order, plain) gives the same accepted interactions and the same
    trajectory to fp64 regrouping, across template sizes that select them."""
    runs = []
    for env in ({}, {"FGA_SPLIT": "0", "FGA_LPT": "0"}):
        e = dict(os.environ, **env)
        out = subprocess.run([sys.executable, "-c", SWEEP_SCRIPT], env=e, capture_output=True,
                             text=True, timeout=900)
        assert out.returncode == 0, out.stderr[-2000:]
        runs.append(json.loads(out.stdout.strip().splitlines()[-1]))
    for k in runs[0]:
        assert runs[0][k]["inter"] == runs[1][k]["inter"], k
        d = np.abs(np.array(runs[0][k]["traj"]) - np.array(runs[1][k]["traj"])).max()
        assert d < 1e-10, (k, d)


OP_SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
import ctypes
import numpy as np
import torch
from paper_2009_14005_b200 import PointCloud, bhtree, synth
from paper_2009_14005_b200 import _native as N
rng = synth.rng_from_seed(7)
x = synth.blob(200000, rng)
mx = rng.uniform(0.005, 0.02, len(x))
bhtree.build(PointCloud(x.points), mx, 20)
c = N.context(0)
L = N.lib()
out = {}
for m, pinned in ((3000, False), (25000, True), (3000, True)):
    q = np.ascontiguousarray(synth.blob(m, synth.rng_from_seed(m)).points)
    qm = synth.rng_from_seed(m + 1).uniform(0.02, 0.1, m)
    runs = []
    for call in range(3):
        if pinned:
            f = torch.zeros((m, 3), dtype=torch.float64, pin_memory=True).numpy()
            vis = torch.zeros(m, dtype=torch.int64, pin_memory=True).numpy()
        else:
            f, vis = np.zeros((m, 3)), np.zeros(m, np.int64)
        acc = np.zeros(m, np.int64)
        t = N._i64(-1)
        N.check(L.fga_tree_forces(c.handle, N.ptr(q), N.ptr(qm), m, 0.5, 1.0, 0.04, 0,
                                  N.ptr(f), N.ptr(vis), N.ptr(acc)))
        N.check(L.fga_last_interactions(c.handle, ctypes.byref(t)))
        runs.append((f.copy(), vis.copy(), acc.copy(), t.value))
    (f0, v0, a0, t0) = runs[0]
    out[f"{m}-{pinned}"] = {
        "vis_equal": all(np.array_equal(v0, r[1]) for r in runs),
        "acc_equal": all(np.array_equal(a0, r[2]) for r in runs),
        "total_equal": all(t0 == r[3] == int(a0.sum()) for r in runs),
        "frel": max(float(np.abs(r[0] - f0).max() / np.abs(f0).max()) for r in runs),
        "f0": f0[:64].tolist(), "v0": v0[:64].tolist(), "acc_sum": int(a0.sum())}
print(json.dumps(out))
""" % ROOT


def _run_op(split):
    env = dict(os.environ, FGA_SPLIT="1" if split else "0", FGA_SPLIT_LOG="1")
    out = subprocess.run([sys.executable, "-c", OP_SCRIPT], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1]), out.stderr


def test_operator_split_passes_match_unsplit(orc):
    """One-wave fga_tree_forces calls (an N-way rank's slice of the queries):
    the first call over a tree / query count / theta records the warps'
    traces, later calls run as split passes.  Visits, accepted counts and the
    interaction total are identical to the unsplit calls; forces agree to
    fp64 regrouping; pageable and pinned (zero-copy) outputs; a new query
    count records a new trace."""
    a, err = _run_op(True)
    b, err0 = _run_op(False)
    assert "operator trace: 3000 queries" in err and "-> split" in err
    assert err.count("operator trace:") == 3  # 3000, 25000, then 3000 again
    assert "operator trace" not in err0
    for k in a:
        assert a[k]["vis_equal"] and a[k]["acc_equal"] and a[k]["total_equal"], k
        assert a[k]["frel"] < 1e-12, (k, a[k]["frel"])
        assert b[k]["frel"] == 0.0
        assert a[k]["v0"] == b[k]["v0"] and a[k]["acc_sum"] == b[k]["acc_sum"]
        assert np.abs(np.array(a[k]["f0"]) - np.array(b[k]["f0"])).max() <= 1e-12 * np.abs(
            np.array(b[k]["f0"])).max()
    # and the oracle's visits on the first queries
    from paper_2009_14005_b200 import synth
    rng = synth.rng_from_seed(7)
    x = synth.blob(200000, rng)
    mx = rng.uniform(0.005, 0.02, len(x))
    tree = orc.tree_build(x.points, mx, 20)
    q = np.ascontiguousarray(synth.blob(3000, synth.rng_from_seed(3000)).points)
    qm = synth.rng_from_seed(3001).uniform(0.02, 0.1, 3000)
    of, ovis, oacc = orc.bh_forces(tree, q[:64], qm[:64], 0.5, 1.0, 0.2, 1)
    assert np.array_equal(np.array(a["3000-False"]["v0"]), ovis)
    np.testing.assert_allclose(np.array(a["3000-False"]["f0"]), of, rtol=1e-5,
                               atol=1e-5 * np.abs(of).max())


@pytest.mark.parametrize("case", ["forces", "two_d"])
def test_operator_split_calls_match_reference_golden(golden, case):
    """Repeated FP32 bh_forces calls over the same tree and query count: the
    first records the warps' traces, the later ones run as split passes
    (>= 8 warps, one wave).  Every call reproduces the REFERENCE's visits
    (golden vectors from the reference itself) and its forces within 1e-5;
    the split calls equal the first to 1e-12.  D=3 (500 queries) and D=2
    (the 150 golden queries tiled to 450)."""
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import bhtree
    g = golden(case)
    theta = 0.5 if case == "two_d" else 0.3
    q, qm = g["q"], g["qm"]
    ref_f, ref_v = g[f"bh/theta{theta}/forces"], g[f"bh/theta{theta}/visits"]
    if case == "two_d":
        q, qm = np.tile(q, (3, 1)), np.tile(qm, 3)
        ref_f, ref_v = np.tile(ref_f, (3, 1)), np.tile(ref_v, 3)
    t = bhtree.build(fga.PointCloud(g["x"]), g["xm"], 20)
    p = fga.default_params().replace(theta=theta)
    runs = [bhtree.bh_forces(t, q, qm, p, count_visits=True, precision="fp32")
            for _ in range(3)]
    for f, v in runs:
        assert np.array_equal(v, ref_v)
        rel = np.linalg.norm(f - ref_f, axis=1) / np.linalg.norm(ref_f, axis=1)
        assert rel.max() < 1e-5
        assert np.abs(f - runs[0][0]).max() <= 1e-12 * np.abs(runs[0][0]).max()
