"""Batched registration (BASELINE configs[4], csrc/batched.cu): one persistent
kernel runs register() for many pairs.  Each pair must equal the single-pair
device path (same algorithm; only the warp grouping of the template and the
moment summation order differ) and the oracle.  GPU only."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pairs(k=6):
    from paper_2009_14005_b200 import synth
    out = []
    for p in range(k):
        rng = synth.rng_from_seed(100000 + p)
        n = 4096 if p % 3 == 0 else 2000 + 300 * p
        x = synth.blob(n, rng) if p % 2 == 0 else synth.bumped_box(n, rng)
        gt = synth.random_rigid(rng, np.deg2rad(60), 0.1)
        y = synth.misalign(x, gt)
        if p == 4:  # unequal sizes
            from paper_2009_14005_b200 import PointCloud
            y = PointCloud(y.points[: n - 500])
        out.append((x, y))
    return out


def test_batch_matches_single_pair_path(orc):
    import paper_2009_14005_b200 as fga
    pairs = _pairs()
    p = fga.default_params()
    br = fga.register_batch(pairs, params=p, options=fga.RegisterOptions(record_iterations=True))
    assert all(e is None for e in br.errors)
    for (x, y), r in zip(pairs, br.results):
        s = fga.register(x, y, params=p, options=fga.RegisterOptions(record_iterations=True))
        assert r.iterations == s.iterations and r.converged == s.converged
        assert np.abs(r.transform.rotation - s.transform.rotation).max() < 1e-8
        assert np.abs(r.transform.translation - s.transform.translation).max() < 1e-8
        d1 = np.array([q.transform_delta for q in r.records])
        d2 = np.array([q.transform_delta for q in s.records])
        # per-iteration deltas (squared transform steps): the single-pair path
        # sums the FP32 force in fp64 chunks (split into node-range parts for
        # small templates), the batched kernel in its own order
        assert np.allclose(d1, d2, rtol=1e-5, atol=1e-14)
        assert abs(r.gpe_initial - s.gpe_initial) <= 1e-6 * abs(s.gpe_initial)
        assert abs(r.gpe_final - s.gpe_final) <= 1e-6 * abs(s.gpe_final)
    for (x, y), r in list(zip(pairs, br.results))[:2]:
        o = orc.register(x.points, y.points, theta=p.theta)
        assert r.iterations == o.iterations and r.converged == o.converged
        assert np.abs(r.transform.rotation - o.R_orig).max() < 1e-4


def test_batch_reports_per_pair_failures():
    import paper_2009_14005_b200 as fga
    pairs = _pairs(3)
    bad = (fga.PointCloud(np.ones((10, 3))), fga.PointCloud(np.ones((10, 3))))
    br = fga.register_batch([pairs[0], bad, pairs[1]])
    assert br.results[1] is None and isinstance(br.errors[1], fga.DegenerateExtent)
    assert br.results[0] is not None and br.results[2] is not None
    single = fga.register(*pairs[1])
    assert br.results[2].iterations == single.iterations


def test_wide_batch_matches_single_pair_path(orc):
    """>= one pair per SM selects the wide mode (per-pair setup / finish in
    the persistent kernel, one wide launch per iteration over all active
    pairs' chunks).  Every pair equals register() of that pair, a sample
    equals the oracle, and a rerun is bitwise identical."""
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import synth
    P = 160  # > 148 SMs
    pairs = [synth.fragment_pair(p, n=1000 + 37 * (p % 7)) for p in range(P)]
    pairs[5] = (fga.PointCloud(np.ones((10, 3))), fga.PointCloud(np.ones((10, 3))))
    p = fga.default_params()
    br = fga.register_batch(pairs, params=p)
    assert isinstance(br.errors[5], fga.DegenerateExtent) and br.results[5] is None
    again = fga.register_batch(pairs, params=p)
    for k in range(0, P, 9):
        if k == 5:
            continue
        r = br.results[k]
        s = fga.register(*pairs[k], params=p)
        assert r.iterations == s.iterations and r.converged == s.converged
        if s.converged:  # (a non-converging run amplifies summation-order differences)
            assert np.abs(r.transform.rotation - s.transform.rotation).max() < 1e-7
        assert np.array_equal(again.results[k].transform.rotation, r.transform.rotation)
    for k in (0, 17, 33):
        x, y = pairs[k]
        o = orc.register(x.points, y.points, theta=p.theta)
        assert br.results[k].iterations == o.iterations
        assert np.abs(br.results[k].transform.rotation - o.R_orig).max() < 1e-4
