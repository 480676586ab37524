"""Operator-level parity of the CUDA path (libfga via the package API) against
the reference's golden vectors and the CPU oracle.  GPU only."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TREE_CASES = ["octant", "dups_cap6", "uniform300", "grid1200", "dups400", "blob2000",
              "uniform_cap3"]


@pytest.fixture(scope="module")
def fga():
    import paper_2009_14005_b200 as f
    return f


@pytest.mark.parametrize("case", TREE_CASES)
def test_tree_build_matches_reference(golden, fga, case):
    """bhtree.build topology bit-exact (bhtree.py:56-122)."""
    from paper_2009_14005_b200 import bhtree
    g = golden("trees")
    t = bhtree.build(fga.PointCloud(g[f"{case}/pts"]), g[f"{case}/masses"],
                     int(g[f"{case}/max_depth"]))
    for k in ("children", "occupancy", "depth", "bbox_min", "bbox_max"):
        assert np.array_equal(getattr(t, k), g[f"{case}/{k}"]), k
    assert np.allclose(t.length, g[f"{case}/length"], rtol=2.5e-16, atol=0)
    ref_mass = g[f"{case}/mass"]
    assert np.allclose(t.mass, ref_mass, rtol=1e-12, atol=0)
    scale = np.abs(g[f"{case}/com"]).max()
    assert np.abs(t.com - g[f"{case}/com"]).max() <= 1e-12 * max(scale, 1.0)


def _split_plane_points(rng, n, lo, hi, L=20):
    """Points exactly on fp64 split planes of the midpoint recursion
    (bhtree.py:89-104) and one ulp either side, inside a box pinned by two
    corner points: the cases where the device's fast key path must defer to
    the exact replay."""
    pts = np.empty((n, 3))
    for k in range(3):
        for i in range(n):
            a, b = lo, hi
            c = a
            for _ in range(int(rng.integers(1, L + 1))):
                c = a + (b - a) / 2.0
                if rng.integers(0, 2):
                    a = c
                else:
                    b = c
            pts[i, k] = [c, np.nextafter(c, -np.inf), np.nextafter(c, np.inf)][rng.integers(0, 3)]
    return np.vstack([[lo] * 3, [hi] * 3, np.clip(pts, lo, hi)])


@pytest.mark.parametrize("kind,n", [("uniform", 50000), ("blob", 200000), ("grid", 27000),
                                    ("dups", 20000), ("planes_dyadic", 6000),
                                    ("planes_odd", 6000), ("dups200", 20000), ("dense", 30000)])
def test_tree_build_matches_oracle_large(orc, fga, kind, n):
    from paper_2009_14005_b200 import bhtree
    rng = np.random.default_rng(n)
    if kind == "uniform":
        p = rng.uniform(-5, 5, size=(n, 3))
    elif kind == "blob":
        from paper_2009_14005_b200 import synth
        p = synth.blob(n, rng).points * 8.0
    elif kind == "grid":
        g = np.arange(30, dtype=np.float64) * 0.25
        p = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
        p = p[rng.permutation(len(p))]
    elif kind == "planes_dyadic":
        p = _split_plane_points(rng, n, -3.0, 5.0)
    elif kind == "planes_odd":
        p = _split_plane_points(rng, n, -1.3, 2.9000000000000004)
    elif kind == "dups200":  # runs of > 64 equal keys: the full-sort fallback
        base = rng.uniform(-1, 1, size=(n // 200, 3))
        p = base[rng.integers(0, len(base), size=n)]
    elif kind == "dense":  # clusters far below the top-32-bit cell size: run fix-ups
        c = rng.uniform(-4, 4, size=(40, 3))
        p = np.vstack([c, c[rng.integers(0, 40, size=n - 40)] +
                       rng.normal(size=(n - 40, 3)) * 2e-4])
    else:
        base = rng.uniform(-1, 1, size=(n // 50, 3))
        p = base[rng.integers(0, len(base), size=n)]
    m = rng.uniform(0.001, 0.02, size=len(p))
    t = bhtree.build(fga.PointCloud(p), m, 20)
    o = orc.tree_build(p, m, 20)
    assert t.node_count == o.node_count
    for k in ("children", "occupancy", "depth", "bbox_min", "bbox_max"):
        assert np.array_equal(getattr(t, k), getattr(o, k)), k
    assert np.allclose(t.mass, o.mass, rtol=1e-12, atol=0)
    assert np.abs(t.com - o.com).max() <= 1e-12 * max(np.abs(o.com).max(), 1.0)


def _boundary_case(kind, rng):
    """Inputs around the device build's 128-point blocks (csrc/tree.cu
    k_subtrees / k_crossing): sizes next to block multiples, duplicate runs
    and depth-cap leaves spanning several blocks, shallow depth caps, a flat
    axis."""
    L = 20
    if kind.startswith("n"):
        p = rng.uniform(-2, 3, size=(int(kind[1:]), 3))
    elif kind == "dup_runs":  # 5 distinct points x 300: depth-cap leaves over 3 blocks
        p = np.repeat(rng.uniform(-1, 1, size=(5, 3)), 300, axis=0)[rng.permutation(1500)]
    elif kind == "dup_plus_uniform":
        p = np.vstack([np.repeat(rng.uniform(-1, 1, size=(1, 3)), 600, axis=0),
                       rng.uniform(-1, 1, size=(900, 3))])
    elif kind.startswith("cap"):
        L = int(kind[3:])
        p = rng.uniform(-1, 1, size=(3000, 3))
    elif kind == "close_pairs":  # ~10-node single-child chains: > 4 nodes per point in a block
        c = rng.uniform(-1, 1, size=(1000, 3))
        d = rng.normal(size=(1000, 3))
        p = np.vstack([c, c + 2e-5 * d / np.linalg.norm(d, axis=1, keepdims=True)])
        p = p[np.argsort(p[:, 0])]
    elif kind == "flat_z":
        p = np.column_stack([rng.uniform(-1, 1, size=(3000, 2)), np.full(3000, 0.25)])
    else:  # one tight cluster inside a sparse cloud: deep chains across blocks
        p = np.vstack([rng.uniform(-1, 1, size=(700, 3)),
                       0.3 + rng.normal(size=(700, 3)) * 1e-9])
    return p, L


@pytest.mark.parametrize("kind", ["n1", "n2", "n127", "n128", "n129", "n255", "n257", "n1000",
                                  "n4097", "dup_runs", "dup_plus_uniform", "cap1", "cap2",
                                  "cap3", "flat_z", "tight_cluster", "close_pairs"])
def test_tree_build_block_boundaries(orc, fga, kind):
    from paper_2009_14005_b200 import bhtree
    import zlib
    rng = np.random.default_rng(zlib.crc32(kind.encode()))
    p, L = _boundary_case(kind, rng)
    m = rng.uniform(0.001, 0.02, size=len(p))
    t = bhtree.build(fga.PointCloud(p), m, L)
    o = orc.tree_build(p, m, L)
    assert t.node_count == o.node_count
    for k in ("children", "occupancy", "depth", "bbox_min", "bbox_max"):
        assert np.array_equal(getattr(t, k), getattr(o, k)), k
    assert np.allclose(t.length, o.length, rtol=2.5e-16, atol=0)
    assert np.allclose(t.mass, o.mass, rtol=1e-12, atol=0)
    assert np.abs(t.com - o.com).max() <= 1e-12 * max(np.abs(o.com).max(), 1.0)


@pytest.mark.parametrize("theta", [0.0, 0.3, 0.5, 0.6, 0.9])
def test_bh_forces_fp64_bit_exact_on_reference_tree(golden, orc, fga, theta):
    """fga_tree_forces(fp64) on the reference's own tree: same visits, same
    forces bit for bit (same node order and per-term arithmetic)."""
    from paper_2009_14005_b200 import bhtree
    g = golden("forces")
    otree = orc.tree_build(g["x"], g["xm"], 20)  # == reference tree (pinned by oracle tests)
    t = bhtree.BHTree(3, 20, otree.children, otree.com, otree.mass, otree.length,
                      otree.occupancy, otree.depth, otree.bbox_min, otree.bbox_max)
    p = fga.default_params().replace(theta=theta)
    f, v = bhtree.bh_forces(t, g["q"], g["qm"], p, count_visits=True, precision="fp64")
    assert np.array_equal(v, g[f"bh/theta{theta}/visits"])
    assert np.array_equal(f, g[f"bh/theta{theta}/forces"])


@pytest.mark.parametrize("theta", [0.0, 0.5, 0.9])
def test_bh_forces_fp32_exact_visits(golden, orc, fga, theta):
    """FP32 traversal: identical accepted set (guard-band MAC), forces within
    1e-5 relative of the reference."""
    from paper_2009_14005_b200 import bhtree
    g = golden("forces")
    t = bhtree.build(fga.PointCloud(g["x"]), g["xm"], 20)
    p = fga.default_params().replace(theta=theta)
    f, v = bhtree.bh_forces(t, g["q"], g["qm"], p, count_visits=True, precision="fp32")
    assert np.array_equal(v, g[f"bh/theta{theta}/visits"])
    ref = g[f"bh/theta{theta}/forces"]
    rel = np.linalg.norm(f - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() < 1e-5


def test_bh_forces_large_vs_oracle(orc, fga):
    from paper_2009_14005_b200 import bhtree, synth
    rng = synth.rng_from_seed(5)
    x = synth.blob(100000, rng).points * 6
    m = rng.uniform(0.0001, 0.001, size=len(x))
    q = synth.blob(4096, rng).points * 6.3 + 0.1
    qm = rng.uniform(0.02, 0.1, size=len(q))
    t = bhtree.build(fga.PointCloud(x), m, 20)
    ot = orc.tree_build(x, m, 20)
    p = fga.default_params().replace(theta=0.5)
    of, ov, oa = orc.bh_forces(ot, q, qm, 0.5, p.G, p.epsilon)
    for prec, tol in (("fp32", 1e-5), ("fp64", 1e-12)):
        f, v, a = bhtree.bh_forces(t, q, qm, p, precision=prec, return_accepted=True)
        assert np.array_equal(v, ov) and np.array_equal(a, oa), prec
        rel = np.linalg.norm(f - of, axis=1) / np.linalg.norm(of, axis=1)
        assert rel.max() < tol, (prec, rel.max())


def test_brute_force_hand_values(fga):
    """test_bhtree.py:89-98 known answers."""
    from paper_2009_14005_b200 import bhtree
    p = fga.default_params().replace(G=1.0)
    ref = fga.PointCloud(np.array([[1.0, 0.0, 0.0]]))
    f = bhtree.brute_force(ref, np.ones(1), np.zeros(3), 1.0, p)
    assert np.allclose(f, [1.0 / 1.04**1.5, 0, 0], atol=1e-12)
    f0 = bhtree.brute_force(ref, np.ones(1), np.zeros(3), 1.0, p.replace(epsilon=0.0))
    assert np.allclose(f0, [1.0, 0, 0], atol=1e-12)
    coinc = fga.PointCloud(np.array([[0.5, 0.5, 0.5]]))
    assert np.allclose(bhtree.brute_force(coinc, np.ones(1), np.array([0.5, 0.5, 0.5]), 1.0, p),
                       0.0)
    # epsilon = 0 and coincident: the reference skips the term (no NaN)
    z = bhtree.direct_forces(coinc, np.ones(1), np.array([[0.5, 0.5, 0.5]]), [1.0],
                             p.replace(epsilon=0.0), precision="fp32")
    assert np.all(np.isfinite(z)) and np.allclose(z, 0.0)


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("fp64", 1e-13)])
def test_direct_forces_vs_reference(golden, fga, prec, tol):
    """Tiled direct sum vs bhtree.brute_force (bhtree.py:155-164)."""
    from paper_2009_14005_b200 import bhtree
    g = golden("forces")
    f = bhtree.direct_forces(fga.PointCloud(g["x"]), g["xm"], g["q"], g["qm"],
                             fga.default_params(), precision=prec)
    ref = g["brute/forces"]
    rel = np.linalg.norm(f - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert rel.max() < tol


def test_direct_forces_large_vs_oracle(orc, fga):
    from paper_2009_14005_b200 import bhtree, synth
    rng = synth.rng_from_seed(8)
    x = synth.blob(300000, rng).points * 6
    m = rng.uniform(0.0001, 0.001, size=len(x))
    q = synth.blob(1000, rng).points * 6
    qm = rng.uniform(0.02, 0.1, size=len(q))
    p = fga.default_params()
    of = orc.brute_forces(x, m, q, qm, p.G, p.epsilon)
    f = bhtree.direct_forces(fga.PointCloud(x), m, q, qm, p, precision="fp32")
    rel = np.linalg.norm(f - of, axis=1) / np.linalg.norm(of, axis=1)
    assert rel.max() < 1e-5, rel.max()


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-6), ("fp64", 1e-13)])
def test_gpe_vs_reference(golden, fga, prec, tol):
    from paper_2009_14005_b200 import dynamics
    g = golden("forces")
    st = dynamics.SwarmState.at_rest(g["q"], g["qm"])
    e = dynamics.gpe(st, fga.PointCloud(g["x"]), g["xm"], fga.default_params(), precision=prec)
    ref = float(g["gpe/value"])
    assert abs(e - ref) <= tol * abs(ref)
    one = dynamics.gpe(dynamics.SwarmState.at_rest(np.zeros((1, 3)), np.ones(1)),
                       fga.PointCloud(np.array([[1.0, 0, 0]])), np.ones(1),
                       fga.default_params().replace(G=1.0, epsilon=0.0), precision=prec)
    assert abs(one - float(g["gpe/hand1"])) < 1e-6


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-6), ("fp64", 1e-13)])
def test_gpe_split_reference_segments(orc, fga, prec, tol):
    """40k x 50k: few query blocks, so the energy kernels split the reference
    points over blockIdx.y (forces.cu gpe_shape).  Same value as the oracle
    and bitwise the same on a rerun."""
    from paper_2009_14005_b200 import dynamics
    rng = np.random.default_rng(11)
    x = rng.uniform(-5, 5, size=(50000, 3))
    xm = rng.uniform(0.001, 0.02, size=50000)
    y = rng.normal(size=(40000, 3)) * 2.0
    ym = rng.uniform(0.02, 0.1, size=40000)
    prm = fga.default_params()
    st = dynamics.SwarmState.at_rest(y, ym)
    e1 = dynamics.gpe(st, fga.PointCloud(x), xm, prm, precision=prec)
    e2 = dynamics.gpe(st, fga.PointCloud(x), xm, prm, precision=prec)
    assert e1 == e2
    ref = orc.gpe(y, ym, x, xm, prm.G, prm.epsilon)
    assert abs(e1 - ref) <= tol * abs(ref)


@pytest.mark.parametrize("seed", [1, 2])
def test_normalize_and_niv_bit_exact(golden, fga, seed):
    g = golden("masses")
    k = f"s{seed}/"
    xn, yn, ctx = fga.normalize_pair(fga.PointCloud(g[k + "x"]), fga.PointCloud(g[k + "y"]),
                                     -5.0, 5.0)
    assert np.array_equal(xn.points, g[k + "xn"]) and np.array_equal(yn.points, g[k + "yn"])
    c = g[k + "ctx"]
    assert np.array_equal(np.r_[ctx.mean_x, ctx.mean_y, ctx.l, ctx.r, ctx.a, ctx.b], c)
    assert np.array_equal(fga.niv_masses(xn, 16, ctx, 20), g[k + "niv_x"])
    assert np.array_equal(fga.niv_masses(yn, 16, ctx, 20), g[k + "niv_y"])


def test_solve_rigid_vs_reference(golden, fga):
    from paper_2009_14005_b200 import procrustes
    g = golden("rigid")
    for i in range(len(g["y"])):
        tf, _ = procrustes.solve_rigid(g["y"][i], g["yd"][i])
        assert np.abs(tf.rotation - g["R"][i]).max() < 1e-9
        assert np.abs(tf.translation - g["t"][i]).max() < 1e-9


def test_solve_rigid_construct_and_recover(fga):
    """test_acceptance.py:77-104 style: 200 random rigid motions incl.
    reflections in the data, recovered to 1e-9 with det = +1."""
    from paper_2009_14005_b200 import procrustes, synth
    rng = synth.rng_from_seed(13)
    worst = 0.0
    for _ in range(200):
        y = rng.normal(size=(50, 3))
        gt = synth.random_rigid(rng, np.pi, 3.0)
        tf, _ = procrustes.solve_rigid(y, gt.apply(y))
        worst = max(worst, np.abs(tf.rotation - gt.rotation).max(),
                    np.abs(tf.translation - gt.translation).max())
        assert abs(np.linalg.det(tf.rotation) - 1) < 1e-9
    assert worst < 1e-9
    # planar + reflection guard
    y = rng.normal(size=(40, 3))
    y[:, 2] = 0
    tf, _ = procrustes.solve_rigid(y, y * np.array([1.0, 1.0, -1.0]))
    assert abs(np.linalg.det(tf.rotation) - 1) < 1e-9
