"""The register() setup chain on the device -- normalize_pair
(normalize.py:36-60), NIV masses (masses.py:85-116) and the rescale
(registration.py:85-87, numpy's pairwise sx.sum()) -- is bit-exact: the
session's mass fields equal the reference's golden vectors and the oracle's.
GPU only."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fga():
    import paper_2009_14005_b200 as f
    return f


@pytest.mark.parametrize("seed", [1, 2])
def test_session_masses_match_reference_golden(golden, fga, seed):
    from paper_2009_14005_b200.engine import Session
    g = golden("masses")
    k = f"s{seed}/"
    s = Session(fga.PointCloud(g[k + "x"]), fga.PointCloud(g[k + "y"]), fga.default_params())
    mx, my = s.masses()
    s.finish()
    assert np.array_equal(mx, g[k + "mass_x"])
    assert np.array_equal(my, g[k + "mass_y"])


@pytest.mark.parametrize("n", [129, 4097, 200_003])
def test_session_masses_match_oracle(orc, fga, n):
    from paper_2009_14005_b200 import synth
    from paper_2009_14005_b200.engine import Session
    rng = synth.rng_from_seed(n)
    x = synth.blob(n, rng)
    y = synth.misalign(synth.blob(n - 7, rng), synth.random_rigid(rng, np.deg2rad(30), 0.1))
    p = fga.default_params()
    s = Session(x, y, p, fga.RegisterOptions(compute_gpe=False))
    mx, my = s.masses()
    s.finish()
    xn, yn, _ = orc.normalize_pair(x.points, y.points, *p.norm_range)
    sx = orc.niv_masses(xn, p.rho, *p.norm_range, p.max_depth)
    sy = orc.niv_masses(yn, p.rho, *p.norm_range, p.max_depth)
    ex, ey = orc.rescale(sx, sy, p.dt, p.eta)
    assert np.array_equal(mx, ex)
    assert np.array_equal(my, ey)
