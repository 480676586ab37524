"""Barnes-Hut 2^D tree: device build and gated force evaluation (mirrors
gravreg/bhtree.py).

* ``build`` runs the GPU octree build (libfga ``fga_tree_build``: exact fp64
  split keys, radix sort, closed-form preorder emission, bottom-up mass/COM)
  and exports the reference's flat arrays -- topology bit-identical to
  bhtree.py:56-122.
* ``bh_forces`` evaluates the stackless warp-coherent traversal on the device
  (``fga_tree_forces``) against the tree held by the context; a tree built
  elsewhere (e.g. by the reference) is uploaded first (``fga_tree_upload``).
  ``precision="fp64"`` (the default here, as the reference computes in fp64)
  reproduces the reference's visit order and per-term arithmetic exactly;
  ``"fp32"`` is the fast path the registration loop uses.
* ``brute_force`` is the exact O(N) sum (bhtree.py:155-164) on the device's
  tiled direct-sum kernel.
"""

from __future__ import annotations

import itertools

import numpy as np

from . import _native as N
from .core import PointCloud
from .errors import EmptyCloud, LengthMismatch

_tokens = itertools.count(1)


class BHTree:
    """Immutable spatial tree (same arrays as bhtree.py:14-45):
    children (n, 2^D) int64 (-1 absent), com (n, D), mass, length (bbox
    diagonal), occupancy, depth, bbox_min/max."""

    def __init__(self, dim, depth_cap, children, com, mass, length, occupancy, depth, bbox_min,
                 bbox_max):
        self.dim = dim
        self.depth_cap = depth_cap
        self.children = children
        self.com = com
        self.mass = mass
        self.length = length
        self.occupancy = occupancy
        self.depth = depth
        self.bbox_min = bbox_min
        self.bbox_max = bbox_max
        self._token = next(_tokens)

    @property
    def node_count(self):
        return len(self.mass)

    @property
    def realized_depth(self):
        return int(self.depth.max())

    def node_count_bound(self):
        """Theorem 1: N + sum_{d=1}^{d0-1} (2^D)^d + 1 (bhtree.py:47-53)."""
        n = int(self.occupancy[0])
        d0 = self.realized_depth
        k = 2**self.dim
        return n + sum(k**d for d in range(1, d0)) + 1


def build(reference: PointCloud, masses, max_depth: int) -> BHTree:
    """GPU build of the reference's midpoint-split tree (bhtree.py:56-122)."""
    reference.require_nonempty()
    masses = N.f64(masses)
    pts = reference.points
    if masses.shape != (len(pts),):
        raise LengthMismatch(f"masses {masses.shape} vs points {len(pts)}")
    c = N.context()
    nn = N._i64(0)
    N.check(N.lib().fga_tree_build(c.handle, N.ptr(pts), N.ptr(masses), len(pts), reference.dim,
                                   int(max_depth), N.ctypes.byref(nn)))
    n = int(nn.value)
    d = reference.dim
    t = BHTree(d, int(max_depth), np.empty((n, 2**d), np.int64), np.empty((n, d)), np.empty(n),
               np.empty(n), np.empty(n, np.int64), np.empty(n, np.int64), np.empty((n, d)),
               np.empty((n, d)))
    N.check(N.lib().fga_tree_export(c.handle, N.ptr(t.children), N.ptr(t.com), N.ptr(t.mass),
                                    N.ptr(t.length), N.ptr(t.occupancy), N.ptr(t.depth),
                                    N.ptr(t.bbox_min), N.ptr(t.bbox_max)))
    c.tree_token = (t._token, c.tree_generation())
    return t


def _ensure_on_device(tree: BHTree, c: N.Context):
    """Upload ``tree`` unless it is still the context's tree.  The check is on
    (tree token, the context's tree generation): register(), sessions and
    other builds on this thread's context replace its tree and bump the
    generation, so a stale device copy is never reused."""
    if not hasattr(tree, "_token"):
        tree._token = next(_tokens)
    if getattr(c, "tree_token", None) == (tree._token, c.tree_generation()):
        return
    children = np.ascontiguousarray(tree.children, dtype=np.int64)
    com = N.f64(tree.com)
    N.check(N.lib().fga_tree_upload(c.handle, N.ptr(children), N.ptr(com), N.ptr(N.f64(tree.mass)),
                                    N.ptr(N.f64(tree.length)), len(tree.mass), children.shape[1],
                                    tree.dim))
    c.tree_token = (tree._token, c.tree_generation())


def bh_forces(tree, queries, query_masses, params, count_visits=False, precision="fp64",
              return_accepted=False):
    """Gated gravitational forces on a batch of queries (bhtree.py:125-147).

    Returns (M, D) forces, plus (M,) visits with ``count_visits``; with
    ``return_accepted`` also the accepted (leaf + cell) interactions."""
    q = N.f64(queries)
    if q.ndim == 1:
        q = q[None, :]
    qm = np.ascontiguousarray(np.broadcast_to(N.f64(query_masses), (len(q),)))
    c = N.context()
    _ensure_on_device(tree, c)
    m = len(q)
    f = np.zeros((m, q.shape[1]))
    visits = np.zeros(m, np.int64)
    acc = np.zeros(m, np.int64)
    prec = N.PREC_FP64 if precision == "fp64" else N.PREC_FP32
    N.check(N.lib().fga_tree_forces(c.handle, N.ptr(q), N.ptr(qm), m, float(params.theta),
                                    float(params.G), float(params.epsilon) ** 2, prec, N.ptr(f),
                                    N.ptr(visits), N.ptr(acc)))
    if return_accepted:
        return f, visits, acc
    if count_visits:
        return f, visits
    return f


def bh_force(tree, query, query_mass, params, precision="fp64"):
    """Force on a single query (bhtree.py:150-152)."""
    return bh_forces(tree, np.asarray(query)[None, :], [query_mass], params,
                     precision=precision)[0]


def direct_forces(reference: PointCloud, ref_masses, queries, query_masses, params,
                  precision="fp32"):
    """Exact O(NM) softened sum for every query row (the batched form of
    brute_force) on the tiled direct-sum kernel."""
    reference.require_nonempty()
    rm = N.f64(ref_masses)
    q = N.f64(queries)
    if q.ndim == 1:
        q = q[None, :]
    qm = np.ascontiguousarray(np.broadcast_to(N.f64(query_masses), (len(q),)))
    out = np.zeros_like(q)
    c = N.context()
    prec = N.PREC_FP64 if precision == "fp64" else N.PREC_FP32
    N.check(N.lib().fga_direct_forces(c.handle, N.ptr(reference.points), N.ptr(rm), len(reference),
                                      N.ptr(q), N.ptr(qm), len(q), reference.dim,
                                      float(params.G), float(params.epsilon), prec, N.ptr(out)))
    return out


def brute_force(reference: PointCloud, ref_masses, query, query_mass, params):
    """Exact O(N) sum for one query (bhtree.py:155-164), fp64 on the device."""
    if len(reference) == 0:
        raise EmptyCloud("registration requires a non-empty cloud")
    return direct_forces(reference, ref_masses, np.asarray(query, dtype=np.float64)[None, :],
                         [query_mass], params, precision="fp64")[0]
