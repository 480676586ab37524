"""kNN smooth-particle masses (BASELINE configs[3]; an opt-in extension, not a
reference feature -- parity is against scipy.spatial.cKDTree, the stand-in
oracle named in SURVEY §8(a9)/(c)).  Neighbour sets must be exact up to
distance ties.  GPU only."""

import numpy as np
import pytest
from scipy.spatial import cKDTree

pytestmark = pytest.mark.gpu


def _check_knn(pts, k):
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import masses
    idx, d2 = masses.knn(fga.PointCloud(pts), k)
    dist, ref = cKDTree(pts).query(pts, k + 1)
    # drop self (index i) from the reference lists
    rd = np.empty((len(pts), k))
    ri = np.empty((len(pts), k), np.int64)
    for i in range(len(pts)):
        keep = ref[i] != i
        rd[i] = dist[i][keep][:k]
        ri[i] = ref[i][keep][:k]
    assert np.allclose(np.sqrt(d2), rd, rtol=1e-12, atol=1e-12)
    # index sets equal wherever the k-th distance is not tied with the (k+1)-th
    dk1, _ = cKDTree(pts).query(pts, k + 2)
    for i in range(len(pts)):
        if np.isclose(dk1[i][-1], rd[i][-1], rtol=1e-12, atol=0) or rd[i][-1] == 0:
            continue
        assert set(idx[i]) == set(ri[i]), i
    return idx, d2


@pytest.mark.parametrize("kind", ["blob", "uniform", "overlap_outliers", "far_offset"])
def test_knn_exact_vs_ckdtree(kind):
    from paper_2009_14005_b200 import synth
    rng = synth.rng_from_seed(7)
    if kind == "blob":
        pts = synth.blob(20000, rng).points
    elif kind == "uniform":
        pts = rng.uniform(-5, 5, size=(20000, 3))
    elif kind == "far_offset":  # tiny spacing far from the origin: fp32 prefilter at its limit
        pts = synth.blob(20000, rng).points * 0.01 + np.array([500.0, -300.0, 750.0])
    else:
        x, _ = synth.partial_overlap(20000, rng)
        pts = x.points
    _check_knn(pts, 16)


def test_knn_duplicates_and_small_k():
    rng = np.random.default_rng(3)
    base = rng.uniform(-1, 1, size=(300, 3))
    pts = np.vstack([base, base[:50], rng.uniform(-1, 1, size=(200, 3))])
    idx, d2 = _check_knn(pts, 4)
    assert (d2[:50, 0] == 0).all()  # each duplicated point finds its twin at distance 0


def test_knn_masses_and_registration(orc):
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import masses, synth
    rng = synth.rng_from_seed(4)
    x, y = synth.partial_overlap(6000, rng)
    y = synth.misalign(y, synth.random_rigid(rng, np.deg2rad(30), 0.05))
    k = 16
    m = masses.knn_masses(x, k)
    dist, _ = cKDTree(x.points).query(x.points, k + 1)
    ref_m = np.maximum((4.0 / 3.0) * np.pi * dist[:, -1] ** 3 / k, 1e-6)
    assert np.allclose(m, ref_m, rtol=1e-12)
    # register(mass_field="knn") == oracle register with the same masses as
    # external weights (kNN computed in the normalized frame, like NIV)
    xn, yn, _ = orc.normalize_pair(x.points, y.points, -5.0, 5.0)

    def kw(p):
        d, _ = cKDTree(p).query(p, k + 1)
        return np.maximum((4.0 / 3.0) * np.pi * d[:, -1] ** 3 / k, 1e-6)

    ref = orc.register(x.points, y.points, theta=0.5, x_weights=kw(xn), y_weights=kw(yn))
    res = fga.register(x, y, params=fga.default_params().replace(theta=0.5),
                       options=fga.RegisterOptions(mass_field="knn", knn_k=k,
                                                   record_iterations=True))
    assert res.iterations == ref.iterations and res.converged == ref.converged
    assert np.abs(res.trajectory - np.array(ref.trajectory)).max() < 1e-5
