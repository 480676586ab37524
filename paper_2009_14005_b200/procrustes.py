"""Closed-form rigid projection (mirrors gravreg/procrustes.py).

``solve_rigid`` runs on the device: deterministic fp64 reductions for the
means and the 3x3 cross-covariance, a one-sided Jacobi SVD in fp64 and the
reference's reflection guard R = U diag(1, 1, sign det(U V^T)) V^T
(procrustes.py:12-49).  Inside ``register`` the same device code runs fused
into the per-iteration update kernel.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .core import RigidTransform


def _solve(y, y_d):
    y = N.f64(y)
    y_d = N.f64(y_d)
    d = y.shape[1]
    R = np.empty((d, d))
    t = np.empty(d)
    deg = N._i32(0)
    c = N.context()
    N.check(N.lib().fga_solve_rigid(c.handle, N.ptr(y), N.ptr(y_d), len(y), y.shape[1], N.ptr(R),
                                    N.ptr(t), N.ctypes.byref(deg)))
    return R, t, bool(deg.value)


def solve_rotation(y, y_d):
    """(rotation, degenerate) mapping centred y onto centred y_d
    (procrustes.py:12-35)."""
    R, _, deg = _solve(y, y_d)
    return R, deg


def solve_translation(y, y_d, rotation):
    """t = mean(y_d) - R mean(y) (procrustes.py:38-42)."""
    y = np.asarray(y, dtype=np.float64)
    y_d = np.asarray(y_d, dtype=np.float64)
    return y_d.mean(axis=0) - rotation @ y.mean(axis=0)


def solve_rigid(y, y_d):
    """(RigidTransform, degenerate) (procrustes.py:45-49)."""
    R, t, deg = _solve(y, y_d)
    return RigidTransform(R, t), deg
