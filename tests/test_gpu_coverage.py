"""Coverage of valid reference inputs beyond the fast paths' limits
(VERDICT r01 "missing" 3 and 5).  GPU only.

* max_depth > 21 (core.py:143-144 accepts any max_depth >= 1): up to 42
  levels the tree is built with 128-bit keys and equals the reference's
  (bhtree.py:89: duplicates chain down to max_depth, points closer than
  2^-21 of the box split further); beyond 42 levels it is built with 42 and
  equals the reference's when no level-42 cell holds two points, and for a
  registration also when such cells hold only exact duplicates (the
  reference's single-child chain below them has the duplicates' com and mass
  at every node, so only visit counts differ); anything else raises
  DeviceError.
* register_batch runs every pair the batched kernel cannot take (> 8192
  points, fp64, kNN masses, max_depth > 21, D = 2) through register(), so
  each pair gets register()'s result.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _tree_equal(t, o):
    assert t.node_count == o.node_count
    for k in ("children", "occupancy", "depth", "bbox_min", "bbox_max", "length"):
        assert np.array_equal(getattr(t, k), getattr(o, k)), k
    assert np.allclose(t.mass, o.mass, rtol=1e-12, atol=0)
    assert np.abs(t.com - o.com).max() <= 1e-12 * max(np.abs(o.com).max(), 1.0)


@pytest.mark.parametrize("depth", [22, 25, 33, 42])
def test_tree_deep_equals_reference(orc, depth):
    """Duplicates (chained to max_depth) and near-duplicates closer than
    2^-21 of the box: the 128-bit-key build against the oracle."""
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import bhtree, synth
    rng = np.random.default_rng(depth)
    x = synth.blob(20_000, synth.rng_from_seed(31)).points * 4
    near = x[:300] + rng.normal(scale=1e-9, size=(300, 3))   # << 2^-21 of the box
    nearer = x[300:340] + rng.normal(scale=1e-12, size=(40, 3))
    xs = np.vstack([x, x[:25], near, nearer])                # 25 exact duplicates
    m = rng.uniform(0.001, 0.02, size=len(xs))
    t = bhtree.build(fga.PointCloud(xs), m, depth)
    o = orc.tree_build(xs, m, depth)
    assert t.depth_cap == depth and int(o.depth.max()) == depth
    _tree_equal(t, o)


def test_tree_depth_25_plain_blob(orc):
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import bhtree, synth
    x = synth.blob(20_000, synth.rng_from_seed(31)).points * 4
    m = np.random.default_rng(1).uniform(0.001, 0.02, size=len(x))
    _tree_equal(bhtree.build(fga.PointCloud(x), m, 25), orc.tree_build(x, m, 25))


def test_tree_beyond_42_levels(orc):
    """max_depth 50: exact duplicates reach the 42-level cap -> the exported
    tree would lack the reference's chain below it -> DeviceError; without
    them the tree is the reference's."""
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import bhtree, synth
    x = synth.blob(5000, synth.rng_from_seed(33)).points
    m = np.full(len(x), 0.01)
    _tree_equal(bhtree.build(fga.PointCloud(x), m, 50), orc.tree_build(x, m, 50))
    with pytest.raises(fga.DeviceError):
        bhtree.build(fga.PointCloud(np.vstack([x, x[:1]])), np.append(m, 0.01), 50)


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-9), ("fp32", 1e-5)])
def test_register_deep_with_near_duplicates(orc, precision, tol):
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import synth
    rng = synth.rng_from_seed(32)
    base = synth.blob(3000, rng).points
    g = np.random.default_rng(5)
    x = fga.PointCloud(np.vstack([base, base[:40],                            # duplicates
                                  base[40:90] + g.normal(scale=1e-9, size=(50, 3))]))
    y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(30), 0.1))
    p = fga.default_params().replace(theta=0.5, max_depth=30)
    res = fga.register(x, y, params=p, options=fga.RegisterOptions(record_iterations=True,
                                                                   precision=precision))
    ref = orc.register(x.points, y.points, theta=0.5, max_depth=30)
    assert res.iterations == ref.iterations and res.converged == ref.converged
    assert np.abs(res.trajectory - np.array(ref.trajectory)).max() < tol


def test_register_beyond_42_levels(orc):
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import synth
    rng = synth.rng_from_seed(34)
    base = synth.blob(3000, rng).points
    x = fga.PointCloud(np.vstack([base, base[:40]]))  # exact duplicates: exact at any depth
    y = synth.misalign(x, synth.random_rigid(rng, np.deg2rad(30), 0.1))
    p = fga.default_params().replace(theta=0.5, max_depth=60)
    res = fga.register(x, y, params=p, options=fga.RegisterOptions(record_iterations=True,
                                                                   precision="fp64"))
    ref = orc.register(x.points, y.points, theta=0.5, max_depth=60)
    assert res.iterations == ref.iterations
    assert np.abs(res.trajectory - np.array(ref.trajectory)).max() < 1e-9
    # distinct points closer than 2^-42 of the box at max_depth > 42: loud error
    xn = fga.PointCloud(np.vstack([base, base[:1] * (1 + 1e-15) + 1e-15]))
    with pytest.raises(fga.DeviceError):
        fga.register(xn, y, params=p)


def _pair(k, n):
    from paper_2009_14005_b200 import synth
    return synth.fragment_pair(500 + k, n=n)


def test_register_batch_routes_unsupported_pairs_through_register():
    import paper_2009_14005_b200 as fga
    pairs = [_pair(0, 2000), _pair(1, 9000), _pair(2, 3000)]  # the 9000-point pair: register()
    p = fga.default_params()
    br = fga.register_batch(pairs, params=p)
    assert all(e is None for e in br.errors)
    for (x, y), r in zip(pairs, br.results):
        s = fga.register(x, y, params=p)
        assert r.iterations == s.iterations
        assert np.abs(r.transform.rotation - s.transform.rotation).max() < 1e-8
    big = br.results[1]
    s = fga.register(*pairs[1], params=p)
    assert np.array_equal(big.transform.rotation, s.transform.rotation)  # the same call
    # options the kernel does not implement: every pair through register()
    for opts, prm in ((fga.RegisterOptions(precision="fp64"), p),
                      (fga.RegisterOptions(mass_field="knn"), p),
                      (fga.RegisterOptions(), p.replace(max_depth=24))):
        br = fga.register_batch(pairs[:2], params=prm, options=opts)
        for (x, y), r in zip(pairs[:2], br.results):
            s = fga.register(x, y, params=prm, options=opts)
            assert np.array_equal(r.transform.rotation, s.transform.rotation)
            assert r.iterations == s.iterations
