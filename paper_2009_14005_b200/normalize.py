"""Joint normalization into [a, b]^D (mirrors gravreg/normalize.py).

``normalize_pair`` runs on the device (libfga ``fga_normalize_pair``) and is
bit-identical to the reference's numpy arithmetic (normalize.py:47-58): the
column means are summed in numpy's row order and every element-wise step
rounds in the reference's operation order.  ``denormalize_translation`` is the
3x3 host-side closing step (normalize.py:63-84).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import PointCloud, RigidTransform
from .errors import EmptyCloud


@dataclass(frozen=True)
class NormalizationContext:
    mean_x: np.ndarray
    mean_y: np.ndarray
    l: float
    r: float
    a: float
    b: float

    @property
    def scale(self):
        """Original -> normalized distance factor."""
        return (self.b - self.a) / (self.r - self.l)

    @classmethod
    def identity(cls, dim):
        z = np.zeros(dim)
        return cls(mean_x=z, mean_y=z.copy(), l=0.0, r=1.0, a=0.0, b=1.0)

    @classmethod
    def from_array(cls, ctx10):
        c = np.asarray(ctx10, dtype=np.float64)
        return cls(mean_x=c[0:3].copy(), mean_y=c[3:6].copy(), l=float(c[6]), r=float(c[7]),
                   a=float(c[8]), b=float(c[9]))


def normalize_pair(x: PointCloud, y: PointCloud, a: float, b: float):
    """(x_norm, y_norm, context); DegenerateExtent when both clouds collapse
    onto their centroids (normalize.py:36-60)."""
    x.require_nonempty()
    y.require_nonempty()
    if x.dim != y.dim:
        raise EmptyCloud(f"dimension mismatch: {x.dim} vs {y.dim}")
    xn = np.empty_like(x.points)
    yn = np.empty_like(y.points)
    ctx = np.empty(10)
    c = N.context()
    N.check(N.lib().fga_normalize_pair(c.handle, N.ptr(x.points), len(x), N.ptr(y.points), len(y),
                                       x.dim, float(a), float(b), N.ptr(xn), N.ptr(yn),
                                       N.ptr(ctx)))
    return PointCloud(xn), PointCloud(yn), NormalizationContext.from_array(ctx)


def denormalize_translation(t_norm: RigidTransform, ctx: NormalizationContext):
    """Express a normalized-frame transform in the original frame: rotation
    unchanged; translation inverts the affine map around R and restores the
    centroid offset (normalize.py:73-84)."""
    R = t_norm.rotation
    ones = np.ones(t_norm.dim)
    undo = (ctx.r - ctx.l) / (ctx.b - ctx.a)
    t = (-R @ (ctx.mean_y + ctx.l * ones) + undo * (R @ (ctx.a * ones) + t_norm.translation
                                                    - ctx.a * ones)
         + ctx.mean_x + ctx.l * ones)
    return RigidTransform(R, t)
