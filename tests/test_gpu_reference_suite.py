"""The reference's own hot-path tests (pkg/tests/test_bhtree.py,
test_dynamics.py, test_masses.py, test_registration.py, test_acceptance.py
criteria 1-9), re-run against the B200 package (D=3; the device path
implements D=3 only).  Same inputs, seeds and thresholds as the reference.
GPU only."""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import bhtree, dynamics, procrustes, synth
    fga.bhtree, fga.dynamics, fga.procrustes, fga.synth = bhtree, dynamics, procrustes, synth
    return fga


# ------------------------------------------------------------ test_bhtree.py
def test_single_point_tree(F):
    t = F.bhtree.build(F.PointCloud(np.array([[1.0, 2.0, 3.0]])), np.array([0.7]), 20)
    assert t.node_count == 1 and t.mass[0] == 0.7 and t.realized_depth == 0
    assert np.allclose(t.com[0], [1.0, 2.0, 3.0])


def test_empty_cloud_rejected(F):
    with pytest.raises(F.EmptyCloud):
        F.bhtree.build(F.PointCloud(np.zeros((0, 3))), np.zeros(0), 20)


def test_one_point_per_octant(F):
    pts = np.array([[a, b, c] for a in (-0.5, 0.5) for b in (-0.5, 0.5) for c in (-0.5, 0.5)])
    t = F.bhtree.build(F.PointCloud(pts), np.ones(8), 20)
    assert t.node_count == 9 and t.node_count <= t.node_count_bound() and t.realized_depth == 1


def test_duplicates_terminate_at_depth_cap(F):
    pts = np.array([[0.25, 0.25, 0.25], [0.25, 0.25, 0.25], [0.9, 0.9, 0.9]])
    t = F.bhtree.build(F.PointCloud(pts), np.ones(3), 6)
    assert t.realized_depth == 6
    leaves = [i for i in range(t.node_count) if (t.children[i] < 0).all() and t.occupancy[i] == 2]
    assert leaves and t.depth[leaves[0]] == 6


def test_node_aggregates_conserved(F):
    rng = F.synth.rng_from_seed(0)
    pts = rng.uniform(-5, 5, size=(300, 3))
    m = rng.uniform(0.01, 1.0, size=300)
    t = F.bhtree.build(F.PointCloud(pts), m, 20)
    assert abs(t.mass[0] - m.sum()) < 1e-9 * m.sum()
    for node in range(t.node_count):
        kids = t.children[node][t.children[node] >= 0]
        if len(kids) == 0:
            continue
        mk = t.mass[kids].sum()
        assert abs(mk - t.mass[node]) < 1e-9 * t.mass[node]
        ck = (t.com[kids] * t.mass[kids, None]).sum(0) / mk
        assert np.linalg.norm(ck - t.com[node]) < 1e-9


def test_cell_length_is_bbox_diagonal(F):
    rng = F.synth.rng_from_seed(1)
    t = F.bhtree.build(F.PointCloud(rng.uniform(-5, 5, size=(50, 3))), np.ones(50), 20)
    diag = np.linalg.norm(t.bbox_max - t.bbox_min, axis=1)
    assert np.abs(t.length - diag).max() < 1e-12


def test_far_cluster_is_summarized(F):
    p = F.default_params().replace(G=1.0, theta=0.6)
    pts = np.array([[10.0, 0.0, 0.0], [10.1, 0.0, 0.1]])
    masses = np.array([1.0, 2.0])
    t = F.bhtree.build(F.PointCloud(pts), masses, 20)
    f, v = F.bhtree.bh_forces(t, np.zeros(3), [1.0], p, count_visits=True)
    assert v[0] == 1
    com = (pts * masses[:, None]).sum(0) / masses.sum()
    d2 = (com**2).sum() + p.epsilon**2
    assert np.allclose(f[0], -p.G * masses.sum() * (np.zeros(3) - com) / d2**1.5, atol=1e-12)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_force_error_monotone_in_theta(F, precision):
    rng = F.synth.rng_from_seed(4)
    pts = rng.uniform(-5, 5, size=(1500, 3))
    masses = rng.uniform(0.001, 0.05, size=1500)
    cloud = F.PointCloud(pts)
    t = F.bhtree.build(cloud, masses, 20)
    q = rng.uniform(-5, 5, size=(120, 3))
    p = F.default_params()
    exact = F.bhtree.direct_forces(cloud, masses, q, np.full(120, 0.05), p, precision="fp64")
    norms = np.linalg.norm(exact, axis=1)
    errs = []
    for theta in (0.0, 0.3, 0.6, 0.9):
        approx = F.bhtree.bh_forces(t, q, np.full(120, 0.05), p.replace(theta=theta),
                                    precision=precision)
        errs.append((np.linalg.norm(approx - exact, axis=1) / norms).mean())
    for lo, hi in zip(errs, errs[1:]):
        assert hi >= lo - (1e-15 if precision == "fp64" else 1e-6)


def test_batch_matches_single_queries(F):
    rng = F.synth.rng_from_seed(5)
    t = F.bhtree.build(F.PointCloud(rng.uniform(-5, 5, size=(100, 3))), np.ones(100), 20)
    q = rng.uniform(-5, 5, size=(7, 3))
    p = F.default_params()
    batch = F.bhtree.bh_forces(t, q, np.full(7, 0.1), p)
    for i in range(7):
        assert np.array_equal(batch[i], F.bhtree.bh_force(t, q[i], 0.1, p))


# ------------------------------------------------------ criterion 1 (exact)
def test_criterion_01_exact_force_oracle(F):
    """theta=0 tree force == brute force to 1e-12 over 100 random configs
    (test_acceptance.py:33-57; D=3 configs, fp64 device paths)."""
    rng = F.synth.rng_from_seed(11)
    p = F.default_params().replace(theta=0.0)
    worst = 0.0
    t0 = time.perf_counter()
    for _ in range(100):
        n = int(np.exp(rng.uniform(np.log(10), np.log(2000))))
        pts = rng.uniform(-5, 5, size=(n, 3))
        masses = rng.uniform(0.001, 0.05, size=n)
        cloud = F.PointCloud(pts)
        tree = F.bhtree.build(cloud, masses, 20)
        q = rng.uniform(-5, 5, size=3)
        qm = rng.uniform(0.01, 0.2)
        exact = F.bhtree.brute_force(cloud, masses, q, qm, p)
        gated = F.bhtree.bh_force(tree, q, qm, p)
        worst = max(worst, np.linalg.norm(gated - exact) / np.linalg.norm(exact))
    assert worst < 1e-12
    assert time.perf_counter() - t0 < 10.0


def test_criterion_02_node_count_bound(F):
    rng = F.synth.rng_from_seed(12)
    for _ in range(25):
        n = int(np.exp(rng.uniform(np.log(10), np.log(10000))))
        t = F.bhtree.build(F.PointCloud(rng.uniform(-5, 5, size=(n, 3))), np.ones(n), 20)
        assert t.node_count <= t.node_count_bound()


def test_criterion_03_rigid_projection_exactness(F):
    rng = F.synth.rng_from_seed(13)
    worst = 0.0
    for k in range(300):
        y = rng.normal(size=(rng.integers(4, 50), 3))
        if k % 10 == 9:
            tf, _ = F.procrustes.solve_rigid(y, y * np.array([1.0, 1.0, -1.0]))
            assert abs(np.linalg.det(tf.rotation) - 1.0) < 1e-9
            continue
        r0 = F.synth.axis_angle(rng.normal(size=3), rng.uniform(0, np.pi))
        t0 = rng.normal(size=3)
        tf, _ = F.procrustes.solve_rigid(y, y @ r0.T + t0)
        worst = max(worst, np.linalg.norm(tf.rotation - r0), np.linalg.norm(tf.translation - t0))
        assert abs(np.linalg.det(tf.rotation) - 1.0) < 1e-9
    assert worst < 1e-9


# --------------------------------------------------- criteria 4 and 7 (C1)
@pytest.fixture(scope="module")
def clean_runs(F):
    runs = []
    t0 = time.perf_counter()
    for s in range(20):
        rng = F.synth.rng_from_seed(s)
        x = F.synth.blob(2000, rng)
        gt = F.synth.random_rigid(rng, np.deg2rad(60), 0.1)
        y = F.synth.misalign(x, gt)
        r = F.register(x, y)
        runs.append((r, F.rmse(y, r.transform, gt)))
    return runs, time.perf_counter() - t0


def test_criterion_04_clean_recovery(clean_runs):
    runs, elapsed = clean_runs
    errs = [e for _, e in runs]
    assert sum(e < 0.01 for e in errs) >= 19
    assert all(r.converged and r.iterations <= 100 for r, _ in runs)
    assert elapsed < 60.0


def test_criterion_07_potential_energy_descent(clean_runs):
    runs, _ = clean_runs
    conv = [r for r, _ in runs if r.converged]
    assert conv and all(r.gpe_final < r.gpe_initial for r in conv)


def test_criterion_05_noise_robustness(F):
    ok = 0
    for s in range(20):
        rng = F.synth.rng_from_seed(1000 + s)
        x = F.synth.add_uniform_noise(F.synth.blob(2000, rng), 0.4, rng)
        gt = F.synth.random_rigid(rng, np.deg2rad(60), 0.1)
        y = F.synth.misalign(x, gt)
        ok += F.rmse(y, F.register(x, y).transform, gt) < 0.01
    assert ok / 20 >= 0.6


def test_criterion_06_landmark_lift(F):
    """test_acceptance.py:163-178: 3 landmark correspondences lift success on
    near-symmetric boxes under large Euler rotations."""
    p = F.default_params().replace(sigma=12.0)
    plain_ok = lm_ok = 0
    for s in range(20):
        rng = F.synth.rng_from_seed(2000 + s)
        x = F.synth.bumped_box(2000, rng)
        gt = F.synth.random_rigid(rng, 3 * np.pi / 4, 0.1, euler=True)
        y = F.synth.misalign(x, gt)
        idx = rng.choice(2000, size=3, replace=False)
        lm = F.LandmarkSet(tuple((int(i), int(i)) for i in idx))
        plain_ok += F.rmse(y, F.register(x, y).transform, gt) < 0.01
        lm_ok += F.rmse(y, F.register(x, y, landmarks=lm, params=p).transform, gt) < 0.01
    assert lm_ok > plain_ok


def test_criterion_08_frame_consistency(F):
    worst = 0.0
    for s in range(20):
        rng = F.synth.rng_from_seed(500 + s)
        x0 = F.synth.blob(800, rng)
        mu = x0.points.mean(axis=0)
        rot = F.synth.random_rotation(rng, np.deg2rad(30))
        y0 = F.PointCloud((x0.points - mu) @ rot.T + mu)
        xn, yn, _ = F.normalize_pair(x0, y0, -5.0, 5.0)
        a = F.register(xn, yn)
        b = F.register(xn, yn, options=F.RegisterOptions(normalize=False))
        d = a.transform.apply(yn.points) - b.transform.apply(yn.points)
        worst = max(worst, float(np.sqrt((d**2).sum(axis=1).mean())))
    assert worst < 1e-6


def test_criterion_09_quasilinear_scaling(F):
    rng = F.synth.rng_from_seed(42)
    q = rng.uniform(-5, 5, size=(256, 3))
    qm = np.full(256, 0.05)
    p = F.default_params()
    visits_mean = []
    for n in (8000, 16000, 32000, 64000):
        t = F.bhtree.build(F.PointCloud(rng.uniform(-5, 5, size=(n, 3))), np.full(n, 16.0 / n),
                           p.max_depth)
        _, v = F.bhtree.bh_forces(t, q, qm, p, count_visits=True)
        visits_mean.append(v.mean())
    assert visits_mean[-1] / visits_mean[0] < 4.0


# ---------------------------------------------------------- test_dynamics.py
def test_step_hand_example(F):
    st = F.dynamics.SwarmState.at_rest(np.zeros((1, 3)), np.array([1.0]))
    v, d = F.dynamics.step(st, np.array([[1.0, 0.0, 0.0]]), F.default_params())
    assert np.allclose(v, [[0.1, 0, 0]], atol=1e-15) and np.allclose(d, [[0.01, 0, 0]], atol=1e-15)


def test_total_force_matches_brute_at_rest(F):
    rng = F.synth.rng_from_seed(0)
    pts = rng.uniform(-5, 5, size=(200, 3))
    masses = rng.uniform(0.01, 0.1, size=200)
    cloud = F.PointCloud(pts)
    t = F.bhtree.build(cloud, masses, 20)
    q = rng.uniform(-5, 5, size=(6, 3))
    p0 = F.default_params().replace(theta=0.0)
    f = F.dynamics.total_force(F.dynamics.SwarmState.at_rest(q, np.full(6, 0.05)), t, p0)
    for i in range(6):
        fb = F.bhtree.brute_force(cloud, masses, q[i], 0.05, p0)
        assert np.linalg.norm(f[i] - fb) < 1e-12 * max(np.linalg.norm(fb), 1.0)


def test_total_force_dissipation_only(F):
    t = F.bhtree.build(F.PointCloud(np.array([[100.0, 100.0, 100.0]])), np.ones(1), 20)
    st = F.dynamics.SwarmState(np.zeros((1, 3)), np.array([[1.0, 0, 0]]), np.array([1.0]))
    f = F.dynamics.total_force(st, t, F.default_params().replace(G=1e-300))
    assert np.allclose(f, [[-0.2, 0, 0]], atol=1e-12)


def test_gpe_hand_values(F):
    p = F.default_params().replace(G=1.0)
    ref = F.PointCloud(np.zeros((1, 3)))
    at0 = F.dynamics.SwarmState.at_rest(np.zeros((1, 3)), np.ones(1))
    assert abs(F.dynamics.gpe(at0, ref, np.ones(1), p) + 5.0) < 1e-12
    at1 = F.dynamics.SwarmState.at_rest(np.array([[1.0, 0, 0]]), np.ones(1))
    assert abs(F.dynamics.gpe(at1, ref, np.ones(1), p) + 1.0 / 1.2) < 1e-12


# ------------------------------------------------------------ test_masses.py
def _ctx(F):
    from paper_2009_14005_b200.normalize import NormalizationContext
    z = np.zeros(3)
    return NormalizationContext(mean_x=z, mean_y=z, l=-5.0, r=5.0, a=-5.0, b=5.0)


def test_niv_two_cell_count_ratio(F):
    rho, depth = 16, 20
    edge = 10.0 / rho
    crowded = np.tile(np.array([[-5 + 0.3 * edge] * 3]), (10, 1))
    crowded = crowded + np.linspace(0, 0.1 * edge, 10)[:, None]
    lone = np.array([[-5 + 5.5 * edge, -5 + 0.3 * edge, -5 + 0.3 * edge]])
    v = F.niv_masses(F.PointCloud(np.vstack([crowded, lone])), rho, _ctx(F), depth)
    assert np.allclose(v[:10], v[0]) and abs(v[0] / v[10] - 0.1) < 1e-12


def test_niv_single_cell_closed_form(F):
    rho, depth, n = 16, 20, 4
    edge = 10.0 / rho
    ball = 4.0 / 3.0 * np.pi * (10.0 / (2 * depth * rho)) ** 3
    pts = np.full((n, 3), -5 + 0.2 * edge) + np.linspace(0, 0.1 * edge, n)[:, None]
    v = F.niv_masses(F.PointCloud(pts), rho, _ctx(F), depth)
    assert np.allclose(v, edge**3 * edge**3 / (n * ball), rtol=1e-12)


def test_niv_uniform_lattice_equal_values(F):
    rho = 4
    c = -5 + (np.arange(rho) + 0.5) * (10.0 / rho)
    pts = np.stack(np.meshgrid(c, c, c, indexing="ij"), axis=-1).reshape(-1, 3)
    v = F.niv_masses(F.PointCloud(pts), rho, _ctx(F), 20)
    assert np.allclose(v, v[0])


def test_niv_uniform_cube_low_variation_interior(F):
    rng = F.synth.rng_from_seed(2)
    rho = 4
    pts = rng.uniform(-5, 5, size=(200000, 3))
    v = F.niv_masses(F.PointCloud(pts), rho, _ctx(F), 20)
    idx = np.clip(np.floor((pts + 5) / (10.0 / rho)).astype(int), 0, rho - 1)
    interior = np.all((idx >= 1) & (idx <= rho - 2), axis=1)
    assert v[interior].std() / v[interior].mean() < 0.05


def test_niv_denser_cells_get_smaller_values(F):
    rng = F.synth.rng_from_seed(3)
    pts = np.vstack([rng.uniform(-5, -2, size=(20, 3)), rng.uniform(2, 2.2, size=(200, 3))])
    v = F.niv_masses(F.PointCloud(pts), 16, _ctx(F), 20)
    assert v[:20].mean() > v[20:].mean()


def test_niv_rejects_bad_rho(F):
    with pytest.raises(F.InvalidParam):
        F.niv_masses(F.PointCloud(np.zeros((1, 3))), 1, _ctx(F), 20)


# ------------------------------------------------------ test_registration.py
def test_recovers_synthetic_misalignment(F):
    rng = F.synth.rng_from_seed(11)
    x = F.synth.blob(1000, rng)
    gt = F.synth.random_rigid(rng, np.deg2rad(30), 0.1)
    y = F.synth.misalign(x, gt)
    r = F.register(x, y)
    assert r.converged and F.rmse(y, r.transform, gt) < 0.01


def test_result_shape_and_trace(F):
    rng = F.synth.rng_from_seed(12)
    x = F.synth.blob(600, rng)
    y = F.synth.misalign(x, F.synth.random_rigid(rng, np.deg2rad(20), 0.05))
    r = F.register(x, y, options=F.RegisterOptions(trace_gpe=True, record_iterations=True))
    assert len(r.gpe_trace) == r.iterations == len(r.records)
    assert all(rec.transform_delta >= 0 for rec in r.records)
    R = r.transform.rotation
    assert np.linalg.norm(R.T @ R - np.eye(3)) < 1e-9 and abs(np.linalg.det(R) - 1) < 1e-9


def test_theta_accuracy_close_to_exact(F):
    gated, exact = [], []
    for s in range(3):
        rng = F.synth.rng_from_seed(100 + s)
        x = F.synth.blob(1500, rng)
        gt = F.synth.random_rigid(rng, np.deg2rad(45), 0.1)
        y = F.synth.misalign(x, gt)
        gated.append(F.rmse(y, F.register(x, y).transform, gt))
        e = F.register(x, y, params=F.default_params().replace(theta=0.0))
        exact.append(F.rmse(y, e.transform, gt))
    assert np.mean(gated) < 2.0 * np.mean(exact)


def test_sequence_odometry(F):
    rng = F.synth.rng_from_seed(30)
    base = F.synth.blob(1000, rng)
    frames = [base]
    for _ in range(3):
        frames.append(F.synth.misalign(frames[-1], F.synth.random_rigid(rng, np.deg2rad(10), 0.05)))
    seq = F.register_sequence(frames)
    assert len(seq.pairwise) == 3 and len(seq.trajectory) == 4 and not any(seq.failed)
