"""D = 2 on the device path (carried as z = const through the 3-D kernels,
2-D NIV lattice and 2-D Kabsch): parity with the reference's own 2-D
outputs (tests/golden/two_d.npz).  GPU only."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    import paper_2009_14005_b200 as fga
    from paper_2009_14005_b200 import bhtree, dynamics, procrustes
    fga.bhtree, fga.dynamics, fga.procrustes = bhtree, dynamics, procrustes
    return fga


def test_two_d_tree_and_forces(golden, F):
    g = golden("two_d")
    t = F.bhtree.build(F.PointCloud(g["x"]), g["xm"], 20)
    for k in ("children", "occupancy", "depth", "bbox_min", "bbox_max"):
        assert np.array_equal(getattr(t, k), g[f"tree/{k}"]), k
    assert np.allclose(t.mass, g["tree/mass"], rtol=1e-12, atol=0)
    assert np.abs(t.com - g["tree/com"]).max() < 1e-12 * 5
    p = F.default_params()
    for theta in (0.0, 0.5):
        for prec, tol in (("fp64", 1e-12), ("fp32", 1e-5)):
            f, v = F.bhtree.bh_forces(t, g["q"], g["qm"], p.replace(theta=theta),
                                      count_visits=True, precision=prec)
            assert np.array_equal(v, g[f"bh/theta{theta}/visits"]), (theta, prec)
            ref = g[f"bh/theta{theta}/forces"]
            rel = np.linalg.norm(f - ref, axis=1) / np.linalg.norm(ref, axis=1)
            assert f.shape == ref.shape and rel.max() < tol, (theta, prec)
    bf = F.bhtree.direct_forces(F.PointCloud(g["x"]), g["xm"], g["q"], g["qm"], p,
                                precision="fp64")
    assert np.abs(bf - g["brute"]).max() < 1e-12 * np.abs(g["brute"]).max()
    e = F.dynamics.gpe(F.dynamics.SwarmState.at_rest(g["q"], g["qm"]), F.PointCloud(g["x"]),
                       g["xm"], p)
    assert abs(e - float(g["gpe"])) < 1e-12 * abs(float(g["gpe"]))


def test_two_d_reference_tree_bit_exact(golden, F):
    g = golden("two_d")
    t = F.bhtree.BHTree(2, 20, g["tree/children"], g["tree/com"], g["tree/mass"],
                        g["tree/length"], g["tree/occupancy"], g["tree/depth"],
                        g["tree/bbox_min"], g["tree/bbox_max"])
    f, v = F.bhtree.bh_forces(t, g["q"], g["qm"], F.default_params().replace(theta=0.5),
                              count_visits=True)
    assert np.array_equal(v, g["bh/theta0.5/visits"])
    assert np.array_equal(f, g["bh/theta0.5/forces"])


def test_two_d_normalize_niv_rigid(golden, F):
    g = golden("two_d")
    xn, yn, ctx = F.normalize_pair(F.PointCloud(g["norm/x"]), F.PointCloud(g["norm/y"]), -5.0, 5.0)
    assert np.array_equal(xn.points, g["norm/xn"]) and np.array_equal(yn.points, g["norm/yn"])
    assert np.array_equal(F.niv_masses(xn, 16, ctx, 20), g["norm/niv_x"])
    for i in range(len(g["rigid/y"])):
        tf, _ = F.procrustes.solve_rigid(g["rigid/y"][i], g["rigid/yd"][i])
        assert tf.rotation.shape == (2, 2)
        assert np.abs(tf.rotation - g["rigid/R"][i]).max() < 1e-9
        assert np.abs(tf.translation - g["rigid/t"][i]).max() < 1e-9


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_two_d_registration(golden, F, precision):
    """test_registration.py:113-125 case, compared with the reference run."""
    g = golden("two_d")
    r = F.register(F.PointCloud(g["reg/x"]), F.PointCloud(g["reg/y"]),
                   options=F.RegisterOptions(record_iterations=True, precision=precision))
    assert r.transform.rotation.shape == (2, 2)
    assert abs(np.linalg.det(r.transform.rotation) - 1.0) < 1e-9
    assert r.iterations == int(g["reg/iterations"]) and r.converged == bool(g["reg/converged"])
    assert np.allclose([q.transform_delta for q in r.records], g["reg/deltas"], rtol=1e-3,
                       atol=1e-12)
    assert np.abs(r.transform.rotation - g["reg/R"]).max() < 1e-4
    assert np.abs(r.transform.translation - g["reg/t"]).max() < 1e-4
    assert abs(r.gpe_initial - float(g["reg/gpe_initial"])) < 1e-6 * abs(float(g["reg/gpe_initial"]))
