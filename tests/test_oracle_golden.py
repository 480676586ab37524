"""Pins the CPU oracle (oracle/) against golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

TREE_CASES = ["octant", "dups_cap6", "uniform300", "grid1200", "dups400", "blob2000",
              "uniform_cap3"]


@pytest.mark.parametrize("case", TREE_CASES)
def test_oracle_tree_matches_reference(golden, orc, case):
    g = golden("trees")
    t = orc.tree_build(g[f"{case}/pts"], g[f"{case}/masses"], int(g[f"{case}/max_depth"]))
    for k in ("children", "occupancy", "depth", "bbox_min", "bbox_max", "mass", "com"):
        assert np.array_equal(getattr(t, k), g[f"{case}/{k}"]), k
    # length: numpy norm goes through BLAS ddot; allow 1 ulp
    assert np.allclose(t.length, g[f"{case}/length"], rtol=2.5e-16, atol=0)


@pytest.mark.parametrize("theta", [0.0, 0.3, 0.5, 0.6, 0.9])
def test_oracle_bh_forces_match_reference(golden, orc, theta):
    g = golden("forces")
    t = orc.tree_build(g["x"], g["xm"], 20)
    f, v, a = orc.bh_forces(t, g["q"], g["qm"], theta, 66.7, 0.2)
    assert np.array_equal(v, g[f"bh/theta{theta}/visits"])
    assert np.array_equal(f, g[f"bh/theta{theta}/forces"])
    assert np.all(a <= v) and np.all(a >= 1)


def test_oracle_bh_eps0(golden, orc):
    g = golden("forces")
    t = orc.tree_build(g["x"], g["xm"], 20)
    f, v, _ = orc.bh_forces(t, g["q"], g["qm"], 0.5, 66.7, 0.0)
    assert np.array_equal(v, g["bh/eps0/visits"])
    assert np.array_equal(f, g["bh/eps0/forces"])


def test_oracle_brute_and_gpe(golden, orc):
    g = golden("forces")
    bf = orc.brute_forces(g["x"], g["xm"], g["q"], g["qm"], 66.7, 0.2)
    # numpy's float64 ``**1.5`` dispatches to a SIMD pow (SVML on AVX-512 hosts)
    # that differs from libm pow in the last ulp: compare to 1e-14 relative.
    ref = g["brute/forces"]
    err = np.linalg.norm(bf - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert err.max() < 1e-14
    assert orc.gpe(g["q"], g["qm"], g["x"], g["xm"], 66.7, 0.2) == float(g["gpe/value"])
    assert orc.gpe(g["q"], g["qm"], g["x"], g["xm"], 66.7, 0.2, nthreads=1) == float(g["gpe/value"])
    assert orc.gpe(np.zeros((1, 3)), np.ones(1), np.array([[1.0, 0, 0]]), np.ones(1), 1.0,
                   0.0) == float(g["gpe/hand1"]) == -1.0


@pytest.mark.parametrize("seed", [1, 2])
def test_oracle_normalize_and_masses(golden, orc, seed):
    g = golden("masses")
    k = f"s{seed}/"
    xn, yn, ctx = orc.normalize_pair(g[k + "x"], g[k + "y"], -5.0, 5.0)
    assert np.array_equal(xn, g[k + "xn"]) and np.array_equal(yn, g[k + "yn"])
    c = g[k + "ctx"]
    assert np.array_equal(np.r_[ctx.mean_x, ctx.mean_y, ctx.l, ctx.r, ctx.a, ctx.b], c)
    nx = orc.niv_masses(xn, 16, -5.0, 5.0, 20)
    ny = orc.niv_masses(yn, 16, -5.0, 5.0, 20)
    assert np.array_equal(nx, g[k + "niv_x"]) and np.array_equal(ny, g[k + "niv_y"])
    mx, my = orc.rescale(nx, ny, 0.1, 0.2)
    assert np.array_equal(mx, g[k + "mass_x"]) and np.array_equal(my, g[k + "mass_y"])


def test_oracle_pairwise_sum_matches_numpy(orc):
    rng = np.random.default_rng(3)
    for n in (1, 7, 8, 9, 127, 128, 129, 1000, 65537):
        a = rng.normal(size=n) * 1e3
        assert orc.pairwise_sum(a) == a.sum()


def test_oracle_solve_rigid(golden, orc):
    g = golden("rigid")
    for i in range(len(g["y"])):
        R, t = orc.solve_rigid(g["y"][i], g["yd"][i])
        assert np.array_equal(R, g["R"][i]) and np.array_equal(t, g["t"][i])


@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_register_trajectory(golden, orc, seed):
    g = golden("register")
    k = f"s{seed}/"
    r = orc.register(g[k + "x"], g[k + "y"], theta=0.5)
    assert r.iterations == int(g[k + "iterations"])
    assert r.converged == bool(g[k + "converged"])
    assert np.array_equal(np.array(r.deltas), g[k + "deltas"])
    assert np.array_equal(np.array(r.trajectory), g[k + "traj"])
    assert np.array_equal(r.R_orig, g[k + "R"])
    assert np.array_equal(r.t_orig, g[k + "t"])
    assert r.gpe_initial == float(g[k + "gpe_initial"])
    assert r.gpe_final == float(g[k + "gpe_final"])


def test_oracle_two_d_matches_reference(golden, orc):
    """D = 2 (quadtree, 2-D NIV, 2-D Kabsch, registration) bit-exact."""
    g = golden("two_d")
    t = orc.tree_build(g["x"], g["xm"], 20)
    for k in ("children", "occupancy", "depth", "bbox_min", "bbox_max", "mass", "com"):
        assert np.array_equal(getattr(t, k), g[f"tree/{k}"]), k
    for theta in (0.0, 0.5):
        f, v, _ = orc.bh_forces(t, g["q"], g["qm"], theta, 66.7, 0.2)
        assert np.array_equal(v, g[f"bh/theta{theta}/visits"])
        assert np.array_equal(f, g[f"bh/theta{theta}/forces"])
    assert orc.gpe(g["q"], g["qm"], g["x"], g["xm"], 66.7, 0.2) == float(g["gpe"])
    xn, yn, ctx = orc.normalize_pair(g["norm/x"], g["norm/y"], -5.0, 5.0)
    assert np.array_equal(xn, g["norm/xn"]) and np.array_equal(yn, g["norm/yn"])
    assert np.array_equal(orc.niv_masses(xn, 16, -5.0, 5.0, 20), g["norm/niv_x"])
    for i in range(len(g["rigid/y"])):
        R, tt = orc.solve_rigid(g["rigid/y"][i], g["rigid/yd"][i])
        assert np.array_equal(R, g["rigid/R"][i]) and np.array_equal(tt, g["rigid/t"][i])
    r = orc.register(g["reg/x"], g["reg/y"])
    assert r.iterations == int(g["reg/iterations"])
    assert np.array_equal(np.array(r.deltas), g["reg/deltas"])
    assert np.array_equal(r.t_orig, g["reg/t"]) and np.array_equal(r.R_orig, g["reg/R"])


def test_oracle_rbf_and_landmark_registration(golden, orc):
    g = golden("rbf")
    for j in range(3):
        v = orc.rbf_masses(g["rbf/pts"], list(g[f"rbf/{j}/anchors"]), float(g[f"rbf/{j}/sigma"]))
        assert np.array_equal(v, g[f"rbf/{j}/values"])
    idx = [int(i) for i in g["lm/idx"]]
    r = orc.register(g["lm/x"], g["lm/y"], landmarks=(idx, idx), sigma=12.0)
    assert r.iterations == int(g["lm/iterations"])
    assert np.array_equal(np.array(r.deltas), g["lm/deltas"])
    assert np.array_equal(r.R_orig, g["lm/R"]) and np.array_equal(r.t_orig, g["lm/t"])
