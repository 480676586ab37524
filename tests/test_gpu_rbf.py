"""Landmark RBF mass field and SPM (masses.py:55-82, :119-125,
registration.py:74-83) on the device: the reference's own RBF tests
(test_masses.py:27-70) plus golden values and a landmark registration
(test_registration.py:98-110).  GPU only."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    import paper_2009_14005_b200 as fga
    return fga


def test_rbf_reference_unit_tests(F):
    from paper_2009_14005_b200.synth import axis_angle, rng_from_seed
    cloud = F.PointCloud(rng_from_seed(0).normal(size=(10, 3)))
    assert np.array_equal(F.rbf_masses(cloud, [], 0.03), np.ones(10))
    two = F.PointCloud(np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]]))
    assert abs(F.rbf_masses(two, [0], 0.03)[0] - 1.0) < 1e-12
    s = 0.03
    v = F.rbf_masses(F.PointCloud(np.array([[0.0, 0, 0], [s, 0, 0]])), [0], s)
    assert abs(v[1] - np.exp(-1.0)) < 1e-12
    far = F.rbf_masses(F.PointCloud(np.array([[0.0, 0, 0], [100.0, 0, 0]])), [0], 0.03)
    assert far[1] == 1e-6
    rng = rng_from_seed(1)
    pts = rng.uniform(-5, 5, size=(60, 3))
    base = F.rbf_masses(F.PointCloud(pts), [3, 17, 40], 2.0)
    rot = axis_angle(rng.normal(size=3), 1.3)
    moved = F.rbf_masses(F.PointCloud(pts @ rot.T + np.array([1.0, -2.0, 0.5])), [3, 17, 40], 2.0)
    assert np.max(np.abs(base - moved)) < 1e-9
    with pytest.raises(F.SingularCollocation):
        F.rbf_masses(F.PointCloud(np.array([[0.0, 0, 0], [0.0, 0, 0], [1.0, 0, 0]])), [0, 1], 0.03)
    with pytest.raises(F.InvalidParam):
        F.rbf_masses(F.PointCloud(np.zeros((1, 3))), [0], 0.0)


def test_rbf_golden(golden, F):
    g = golden("rbf")
    for j in range(3):
        v = F.rbf_masses(F.PointCloud(g["rbf/pts"]), list(g[f"rbf/{j}/anchors"]),
                         float(g[f"rbf/{j}/sigma"]))
        assert np.allclose(v, g[f"rbf/{j}/values"], rtol=1e-9, atol=1e-15)


def test_landmark_registration_matches_reference(golden, F):
    g = golden("rbf")
    idx = [int(i) for i in g["lm/idx"]]
    lm = F.LandmarkSet(tuple((i, i) for i in idx))
    r = F.register(F.PointCloud(g["lm/x"]), F.PointCloud(g["lm/y"]), landmarks=lm,
                   params=F.default_params().replace(sigma=12.0),
                   options=F.RegisterOptions(record_iterations=True))
    assert r.iterations == int(g["lm/iterations"])
    assert np.allclose([q.transform_delta for q in r.records], g["lm/deltas"], rtol=1e-3,
                       atol=1e-12)
    assert np.abs(r.transform.rotation - g["lm/R"]).max() < 1e-4
    assert np.abs(r.transform.translation - g["lm/t"]).max() < 1e-4
    with pytest.raises(F.InvalidParam):
        F.register(F.PointCloud(g["lm/x"]), F.PointCloud(g["lm/y"]),
                   landmarks=F.LandmarkSet(((0, 10_000),)))


@pytest.mark.parametrize("m,sigma", [(65, 0.6), (200, 0.5), (501, 0.4)])
def test_rbf_many_landmarks_vs_oracle(F, orc, m, sigma):
    """More than 64 landmarks (the reference is unbounded): the parallel
    Jacobi collocation solve (rbf.cu k_rbf_solve_large) against the oracle's
    numpy restatement of masses.py:55-82."""
    rng = np.random.default_rng(m)
    pts = rng.uniform(-5, 5, size=(20000, 3))
    anchors = sorted(rng.choice(len(pts), m, replace=False).tolist())
    v = F.rbf_masses(F.PointCloud(pts), anchors, sigma)
    ref = orc.rbf_masses(pts, anchors, sigma)
    assert np.allclose(v, ref, rtol=1e-8, atol=1e-14)


def test_rbf_many_landmarks_singular(F):
    """An ill-conditioned collocation (wide kernel over many close anchors)
    raises SingularCollocation like the reference (cond > 1e12)."""
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1, 1, size=(5000, 3))
    with pytest.raises(F.SingularCollocation):
        F.rbf_masses(F.PointCloud(pts), list(range(100)), 5.0)
