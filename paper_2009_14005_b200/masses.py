"""Per-point mass fields (mirrors gravreg/masses.py).

``niv_masses`` -- the normalized-intrinsic-volume lattice histogram that is the
default (SPM) mass field on the registration path -- runs on the device
(libfga ``fga_niv_masses``, bit-identical to masses.py:85-116).
``external_masses`` and ``spm`` are the reference's O(N) validation /
element-wise glue (masses.py:119-135).  The RBF landmark field
(masses.py:55-82) runs on the device too (``rbf_masses`` -> libfga
``fga_rbf_masses``, csrc/rbf.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import PointCloud
from .errors import InvalidParam, LengthMismatch, NonFiniteWeight
from .normalize import NormalizationContext

MASS_FLOOR = 1e-6


@dataclass(frozen=True)
class LandmarkSet:
    """One-to-one prior correspondences (template_index, reference_index)
    (masses.py:19-48)."""

    pairs: tuple[tuple[int, int], ...]

    def __post_init__(self):
        pairs = tuple((int(t), int(r)) for t, r in self.pairs)
        tpl = [t for t, _ in pairs]
        ref = [r for _, r in pairs]
        if len(set(tpl)) != len(tpl) or len(set(ref)) != len(ref):
            raise InvalidParam("pairs", "duplicate landmark index")
        if min(tpl + ref, default=0) < 0:
            raise InvalidParam("pairs", "negative index")
        object.__setattr__(self, "pairs", pairs)

    def __len__(self):
        return len(self.pairs)

    def template_indices(self):
        return [t for t, _ in self.pairs]

    def reference_indices(self):
        return [r for _, r in self.pairs]

    def check_bounds(self, n_template, n_reference):
        if any(i >= n_template for i in self.template_indices()):
            raise InvalidParam("pairs", "template index out of range")
        if any(i >= n_reference for i in self.reference_indices()):
            raise InvalidParam("pairs", "reference index out of range")


def niv_masses(cloud: PointCloud, rho: int, ctx: NormalizationContext, max_depth: int):
    """NIV measure over a rho^D lattice on [ctx.a, ctx.b]^D: points in denser
    cells get smaller values (masses.py:85-116), computed on the device."""
    if rho < 2:
        raise InvalidParam("rho", rho)
    out = np.empty(len(cloud))
    c = N.context()
    N.check(N.lib().fga_niv_masses(c.handle, N.ptr(cloud.points), len(cloud), cloud.dim, int(rho),
                                   float(ctx.a), float(ctx.b), int(max_depth), N.ptr(out)))
    return out


def knn(cloud: PointCloud, k: int = 16):
    """Exact k nearest OTHER points of every point on the device (grid
    bucketing, fp64 distances, ties by index): (idx (n,k) int64, d2 (n,k))."""
    n = len(cloud)
    idx = np.empty((n, k), np.int64)
    d2 = np.empty((n, k))
    c = N.context()
    N.check(N.lib().fga_knn(c.handle, N.ptr(cloud.points), n, cloud.dim, int(k), N.ptr(idx),
                            N.ptr(d2)))
    return idx, d2


def knn_masses(cloud: PointCloud, k: int = 16):
    """kNN smooth-particle masses (BASELINE configs[3]; not a reference
    feature): (4/3) pi r_k^3 / k, floored at MASS_FLOOR.  Use through
    RegisterOptions(mass_field="knn") or as x/y_weights."""
    out = np.empty(len(cloud))
    c = N.context()
    N.check(N.lib().fga_knn_masses(c.handle, N.ptr(cloud.points), len(cloud), cloud.dim, int(k),
                                   N.ptr(out)))
    return out


def rbf_masses(cloud: PointCloud, anchors, sigma: float):
    """Gaussian RBF field through the anchors, forced to 1.0 at every anchor
    (masses.py:55-82), on the device; SingularCollocation when the kernel
    matrix condition exceeds 1e12.  No anchors -> uniform 1.0."""
    if sigma <= 0:
        raise InvalidParam("sigma", sigma)
    a = np.ascontiguousarray(list(anchors), dtype=np.int64)
    out = np.empty(len(cloud))
    c = N.context()
    N.check(N.lib().fga_rbf_masses(c.handle, N.ptr(cloud.points), len(cloud), cloud.dim,
                                   N.ptr(a) if len(a) else None, len(a), float(sigma), N.ptr(out)))
    return out


def spm(niv, rbf):
    """Hadamard product of two mass fields (masses.py:119-125)."""
    niv = np.asarray(niv, dtype=np.float64)
    rbf = np.asarray(rbf, dtype=np.float64)
    if niv.shape != rbf.shape:
        raise LengthMismatch(f"{niv.shape} vs {rbf.shape}")
    return niv * rbf


def check_weights(cloud_len: int, weights) -> np.ndarray:
    """external_masses' validation (masses.py:128-134) without the floor."""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    if w.shape != (cloud_len,):
        raise LengthMismatch(f"weights {w.shape} vs points {cloud_len}")
    if not np.isfinite(w).all():
        raise NonFiniteWeight("weights must be finite")
    return w


def external_masses(cloud: PointCloud, weights):
    """Adopt per-point feature weights as masses, floored (masses.py:128-135)."""
    return np.maximum(check_weights(len(cloud), weights), MASS_FLOOR)
