"""INTEGRATION.md's Level-1 drop-in, executed: the replacement
``gravreg/_kernels.py`` module printed there is written to a temp dir,
imported, and called the way the reference calls its numba kernels
(bhtree.py:139-144, dynamics.py:52-60) -- the reference's own tree arrays in,
forces and visits out bit-identical to ``bh_forces_kernel`` (_kernels.py:7-50),
energy equal to ``gpe_kernel`` (_kernels.py:53-67).  Also checks that the
shim keeps an unchanged tree resident instead of re-uploading it every call
(fga_tree_generation).  GPU only."""

import ctypes
import importlib.util
import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"## Level 1.*?```python\n(.*?)```", text, re.S).group(1)
    assert "def bh_forces_kernel" in block and "def gpe_kernel" in block
    d = tmp_path_factory.mktemp("gravreg_b200")
    path = d / "_kernels.py"
    path.write_text(block)
    os.environ["FGA_LIB"] = os.path.join(ROOT, "paper_2009_14005_b200", "_lib", "libfga.so")
    spec = importlib.util.spec_from_file_location("gravreg_kernels_b200", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod._lib.fga_tree_generation.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
    return mod


def _generation(shim):
    g = ctypes.c_int64(0)
    assert shim._lib.fga_tree_generation(shim._ctx, ctypes.byref(g)) == 0
    return g.value


def _ref_tree(orc, g):
    # the oracle's tree == the reference's build (pinned by test_oracle_golden)
    return orc.tree_build(g["x"], g["xm"], 20)


@pytest.mark.parametrize("theta", [0.0, 0.5, 0.9])
def test_shim_bh_forces_kernel_bit_exact(golden, orc, shim, theta):
    g = golden("forces")
    t = _ref_tree(orc, g)
    stack_cap = 8 * (20 + 2)  # bhtree.py:138
    q = np.ascontiguousarray(g["q"])
    qm = np.ascontiguousarray(g["qm"])
    f, v = shim.bh_forces_kernel(t.children, t.com, t.mass, t.length, q, qm, theta, 66.7,
                                 0.2**2, stack_cap)
    assert np.array_equal(v, g[f"bh/theta{theta}/visits"])
    assert np.array_equal(f, g[f"bh/theta{theta}/forces"])


def test_shim_gpe_kernel(golden, shim):
    g = golden("forces")
    e = shim.gpe_kernel(np.ascontiguousarray(g["q"]), np.ascontiguousarray(g["qm"]),
                        np.ascontiguousarray(g["x"]), np.ascontiguousarray(g["xm"]), 66.7, 0.2)
    ref = float(g["gpe/value"])
    assert abs(e - ref) <= 1e-13 * abs(ref)


def test_shim_keeps_the_tree_resident(golden, orc, shim):
    """Per-iteration calls with the same BHTree arrays upload once; a
    different tree (or a rebuild at the same addresses) re-uploads."""
    g = golden("forces")
    a = _ref_tree(orc, g)
    rng = np.random.default_rng(2)
    xb = rng.uniform(-4, 4, size=(3000, 3))
    b = orc.tree_build(xb, np.full(3000, 0.01), 20)
    q = np.ascontiguousarray(g["q"])
    qm = np.ascontiguousarray(g["qm"])

    def call(t):
        return shim.bh_forces_kernel(t.children, t.com, t.mass, t.length, q, qm, 0.5, 66.7,
                                     0.2**2, 176)  # float(eps) ** 2, as bhtree.py:142 passes it

    fa, va = call(a)
    g0 = _generation(shim)
    for _ in range(3):
        f, v = call(a)
        assert np.array_equal(f, fa) and np.array_equal(v, va)
    assert _generation(shim) == g0  # no re-upload
    fb, vb = call(b)
    assert _generation(shim) == g0 + 1
    ob, ovb, _ = orc.bh_forces(b, q, qm, 0.5, 66.7, 0.2)
    assert np.array_equal(vb, ovb) and np.array_equal(fb, ob)
    # the same buffers refilled with another tree's values (same node count)
    c_com = a.com.copy()
    c_com[:, 0] += 0.25
    a.com[:] = c_com
    f2, v2 = call(a)
    assert _generation(shim) == g0 + 2
    a2 = _ref_tree(orc, g)
    a2.com[:] = c_com
    o2, ov2, _ = orc.bh_forces(a2, q, qm, 0.5, 66.7, 0.2)
    assert np.array_equal(v2, ov2) and np.array_equal(f2, o2)
