"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference's (gravreg 0.1.0, /root/reference/pkg) hot-path
algorithm, used as the checker by tests/, __graft_entry__.smoke() and as the CPU
baseline by bench.py (cpu_baseline / --impl reference).  The product package
``paper_2009_14005_b200`` never imports this module.

Heavy loops live in ``fga_oracle.c`` (plain C, OpenMP over independent queries,
built by ``oracle/Makefile`` into ``oracle/_build/liboracle.so``); everything
O(N) is numpy written to round exactly like the reference.  Each function cites
the reference file:line it restates.  The oracle is pinned against golden
vectors produced by the reference itself: see tests/golden/make_golden.py and
tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

# registration.py:41-54 constants
FIELD_MASS = 16.0
FIELD_MASS_POINTS = 2000
REFERENCE_POINT_CAP = 0.022
TEMPLATE_PEAK_MASS = 0.1
MASS_FLOOR = 1e-6  # masses.py:16


def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "fga_oracle.c"))
    ):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build_lib()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        dbl = ctypes.c_double
        L.orc_pairwise_sum.argtypes = [P, i64]
        L.orc_pairwise_sum.restype = dbl
        L.orc_tree_build.argtypes = [P, P, i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(P)]
        L.orc_tree_build.restype = i64
        L.orc_tree_copy.argtypes = [P] * 9
        L.orc_tree_copy.restype = None
        L.orc_tree_free.argtypes = [P]
        L.orc_tree_free.restype = None
        L.orc_bh_forces.argtypes = [P, P, P, P, i64, ctypes.c_int, P, P, i64, ctypes.c_int,
                                    dbl, dbl, dbl, i64, P, P, P, ctypes.c_int]
        L.orc_bh_forces.restype = ctypes.c_int
        L.orc_brute_forces_out.argtypes = [P, P, i64, P, P, i64, ctypes.c_int, dbl, dbl, P,
                                           ctypes.c_int]
        L.orc_brute_forces_out.restype = None
        L.orc_gpe.argtypes = [P, P, i64, P, P, i64, ctypes.c_int, dbl, dbl, ctypes.c_int]
        L.orc_gpe.restype = dbl
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def max_threads() -> int:
    return int(lib().orc_max_threads())


def pairwise_sum(a) -> float:
    a = _f64(a)
    return float(lib().orc_pairwise_sum(_p(a), len(a)))


# ---------------------------------------------------------------------------
# normalize.py:36-60 / :63-84
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class NormCtx:
    mean_x: np.ndarray
    mean_y: np.ndarray
    l: float
    r: float
    a: float
    b: float


def normalize_pair(x, y, a, b):
    """normalize.py:47-58: own means, joint scalar l/r, shared scale."""
    x = _f64(x)
    y = _f64(y)
    mean_x = x.mean(axis=0)
    mean_y = y.mean(axis=0)
    cx = x - mean_x
    cy = y - mean_y
    l = min(cx.min(), cy.min())
    r = max(cx.max(), cy.max())
    if r <= l:
        raise ValueError("DegenerateExtent")
    s = (b - a) / (r - l)
    return (cx - l) * s + a, (cy - l) * s + a, NormCtx(mean_x, mean_y, float(l), float(r), a, b)


def denormalize_translation(R, t, ctx: NormCtx):
    """normalize.py:73-84."""
    d = len(t)
    ones = np.ones(d)
    inv_scale = (ctx.r - ctx.l) / (ctx.b - ctx.a)
    return (-R @ (ctx.mean_y + ctx.l * ones) + inv_scale * (R @ (ctx.a * ones) + t - ctx.a * ones)
            + ctx.mean_x + ctx.l * ones)


# ---------------------------------------------------------------------------
# masses.py:85-116, registration.py:64-88
# ---------------------------------------------------------------------------
def niv_masses(pts, rho, a, b, max_depth):
    """masses.py:85-116 (rho^D lattice histogram NIV measure)."""
    pts = _f64(pts)
    n, d = pts.shape
    extent = b - a
    cell_edge = extent / rho
    cell_vol = cell_edge**d
    r_ball = extent / (2.0 * max_depth * rho)
    ball_vol = np.pi * r_ball**2 if d == 2 else (4.0 / 3.0) * np.pi * r_ball**3
    idx = np.floor((pts - a) / cell_edge).astype(np.int64)
    np.clip(idx, 0, rho - 1, out=idx)
    flat = idx[:, 0]
    for k in range(1, d):
        flat = flat * rho + idx[:, k]
    counts = np.bincount(flat, minlength=rho**d)
    total_vol = np.count_nonzero(counts) * cell_vol
    union = np.minimum(counts * ball_vol, cell_vol)
    with np.errstate(divide="ignore"):
        cell_value = np.where(counts > 0, total_vol * cell_vol / np.where(union > 0, union, 1.0), 0.0)
    return np.maximum(cell_value[flat], MASS_FLOOR)


def rbf_masses(pts, anchors, sigma):
    """masses.py:55-82 (Gaussian RBF collocation through the anchors)."""
    pts = _f64(pts)
    anchors = list(anchors)
    if sigma <= 0:
        raise ValueError("InvalidParam sigma")
    if not anchors:
        return np.ones(len(pts))
    centers = pts[anchors]
    dmat = np.linalg.norm(centers[:, None, :] - centers[None, :, :], axis=-1)
    K = np.exp(-(dmat * dmat) / (sigma * sigma))
    cond = np.linalg.cond(K)
    if not np.isfinite(cond) or cond > 1e12:
        raise ValueError("SingularCollocation")
    lam = np.linalg.solve(K, np.ones(len(centers)))
    deval = np.linalg.norm(pts[:, None, :] - centers[None, :, :], axis=-1)
    values = np.exp(-(deval * deval) / (sigma * sigma)) @ lam
    return np.maximum(values, MASS_FLOOR)


def external_masses(w, n):
    """masses.py:128-135."""
    w = _f64(w)
    if w.shape != (n,):
        raise ValueError("LengthMismatch")
    if not np.all(np.isfinite(w)):
        raise ValueError("NonFiniteWeight")
    return np.maximum(w, MASS_FLOOR)


def rescale(sx, sy, dt, eta):
    """registration.py:85-87."""
    budget = FIELD_MASS * np.sqrt(len(sx) / FIELD_MASS_POINTS)
    sx = np.minimum(budget * sx / sx.sum(), REFERENCE_POINT_CAP)
    sy = np.maximum(TEMPLATE_PEAK_MASS * sy / sy.max(), max(MASS_FLOOR, dt * eta))
    return sx, sy


# ---------------------------------------------------------------------------
# bhtree.py:56-122 (C)
# ---------------------------------------------------------------------------
@dataclass
class Tree:
    dim: int
    depth_cap: int
    children: np.ndarray
    com: np.ndarray
    mass: np.ndarray
    length: np.ndarray
    occupancy: np.ndarray
    depth: np.ndarray
    bbox_min: np.ndarray
    bbox_max: np.ndarray

    @property
    def node_count(self):
        return len(self.mass)


def tree_build(pts, masses, max_depth=20) -> Tree:
    pts = _f64(pts)
    masses = _f64(masses)
    n, d = pts.shape
    handle = ctypes.c_void_p()
    nn = lib().orc_tree_build(_p(pts), _p(masses), n, d, max_depth, ctypes.byref(handle))
    if nn <= 0:
        raise RuntimeError(f"orc_tree_build failed: {nn}")
    nc = 1 << d
    t = Tree(d, max_depth, np.empty((nn, nc), np.int64), np.empty((nn, d)), np.empty(nn),
             np.empty(nn), np.empty(nn, np.int64), np.empty(nn, np.int64), np.empty((nn, d)),
             np.empty((nn, d)))
    lib().orc_tree_copy(handle, _p(t.children), _p(t.com), _p(t.mass), _p(t.length),
                        _p(t.occupancy), _p(t.depth), _p(t.bbox_min), _p(t.bbox_max))
    lib().orc_tree_free(handle)
    return t


# ---------------------------------------------------------------------------
# _kernels.py:7-50 / bhtree.py:125-147 (C)
# ---------------------------------------------------------------------------
def bh_forces(tree: Tree, queries, qmasses, theta, G, eps, nthreads=0):
    """Returns (forces, visits, accepted) -- accepted = leaf+cell interactions."""
    q = _f64(queries)
    if q.ndim == 1:
        q = q[None, :]
    qm = np.ascontiguousarray(np.broadcast_to(_f64(qmasses), (len(q),)))
    m, d = q.shape
    f = np.zeros((m, d))
    visits = np.zeros(m, np.int64)
    acc = np.zeros(m, np.int64)
    stack_cap = (2**tree.dim) * (tree.depth_cap + 2)
    err = lib().orc_bh_forces(_p(tree.children), _p(tree.com), _p(tree.mass), _p(tree.length),
                              tree.node_count, tree.children.shape[1], _p(q), _p(qm), m, d,
                              float(theta), float(G), float(eps) ** 2, stack_cap, _p(f),
                              _p(visits), _p(acc), int(nthreads))
    if err:
        raise RuntimeError(f"orc_bh_forces failed: {err}")
    return f, visits, acc


def brute_forces(ref, rmass, queries, qmasses, G, eps, nthreads=0):
    """bhtree.py:155-164 applied to every query row."""
    ref = _f64(ref)
    rmass = _f64(rmass)
    q = _f64(queries)
    qm = np.ascontiguousarray(np.broadcast_to(_f64(qmasses), (len(q),)))
    out = np.zeros_like(q)
    lib().orc_brute_forces_out(_p(ref), _p(rmass), len(ref), _p(q), _p(qm), len(q), q.shape[1],
                               float(G), float(eps), _p(out), int(nthreads))
    return out


def gpe(pos_y, mass_y, pos_x, mass_x, G, eps, nthreads=0):
    """_kernels.py:53-67 (bit-identical to the serial reference)."""
    pos_y, mass_y, pos_x, mass_x = map(_f64, (pos_y, mass_y, pos_x, mass_x))
    return float(lib().orc_gpe(_p(pos_y), _p(mass_y), len(pos_y), _p(pos_x), _p(mass_x),
                               len(pos_x), pos_y.shape[1], float(G), float(eps), int(nthreads)))


# ---------------------------------------------------------------------------
# dynamics.py:37-47, procrustes.py:12-49
# ---------------------------------------------------------------------------
def step(pos, vel, mass, grav, dt, eta):
    forces = grav - eta * vel  # dynamics.py:40
    new_v = vel + dt * forces / mass[:, None]  # :45
    return new_v, dt * new_v  # :46


def solve_rigid(y, y_d):
    """procrustes.py:12-42 (numpy/LAPACK, identical operations)."""
    yc = y - y.mean(axis=0)
    yd_c = y_d - y_d.mean(axis=0)
    cov = yd_c.T @ yc
    u, s, vt = np.linalg.svd(cov)
    d = cov.shape[0]
    sign = np.sign(np.linalg.det(u @ vt))
    if sign == 0:
        sign = 1.0
    diag = np.ones(d)
    diag[-1] = sign
    rot = u @ np.diag(diag) @ vt
    trans = y_d.mean(axis=0) - rot @ y.mean(axis=0)
    return rot, trans


# ---------------------------------------------------------------------------
# registration.py:91-166 -- records the per-iteration [R_acc|t_acc] trajectory
# ---------------------------------------------------------------------------
@dataclass
class OracleResult:
    R: np.ndarray  # normalized frame R_acc
    t: np.ndarray  # normalized frame t_acc
    R_orig: np.ndarray
    t_orig: np.ndarray
    iterations: int
    converged: bool
    gpe_initial: float
    gpe_final: float
    deltas: list
    trajectory: list  # per-iteration 3x4 [R_acc|t_acc]
    accepted: list  # per-iteration interactions (sum over queries)


def setup(x, y, rho=16, max_depth=20, norm_range=(-5.0, 5.0), dt=0.1, eta=0.2):
    """registration.py:104-121 without the tree: normalized clouds, NIV mass
    fields and the rescale -> (xn, yn, mx, my, ctx)."""
    a, b = norm_range
    xn, yn, ctx = normalize_pair(x, y, a, b)
    mx, my = rescale(niv_masses(xn, rho, a, b, max_depth), niv_masses(yn, rho, a, b, max_depth),
                     dt, eta)
    return xn, yn, mx, my, ctx


def iterate(tree, pos, vel, my, r_acc, t_acc, theta, G, epsilon, dt=0.1, eta=0.2, nthreads=0):
    """One pass of the loop body (registration.py:130-142): forces, step,
    Kabsch, the rigid update of the swarm and the accumulated transform.
    Returns (pos, vel, r_acc, t_acc, grav, visits, accepted)."""
    grav, visits, acc = bh_forces(tree, pos, my, theta, G, epsilon, nthreads)
    v_new, disp = step(pos, vel, my, grav, dt, eta)
    R, t = solve_rigid(pos, pos + disp)
    return (pos @ R.T + t, v_new @ R.T, R @ r_acc, t + R @ t_acc, grav, visits, acc)


def register(x, y, G=66.7, epsilon=0.2, eta=0.2, dt=0.1, theta=0.6, rho=16, max_depth=20,
             norm_range=(-5.0, 5.0), conv_tol=1e-4, max_iters=100, x_weights=None,
             y_weights=None, normalize=True, nthreads=0, gpe=True, force_fn=None,
             landmarks=None, sigma=0.03):
    """registration.py:91-166; landmarks = (reference_indices, template_indices)."""
    a, b = norm_range
    if normalize:
        xn, yn, ctx = normalize_pair(x, y, a, b)
    else:
        xn, yn = _f64(x), _f64(y)
        z = np.zeros(xn.shape[1])
        ctx = NormCtx(z, z.copy(), a, b, a, b)
    sx = external_masses(x_weights, len(xn)) if x_weights is not None else niv_masses(
        xn, rho, a, b, max_depth)
    sy = external_masses(y_weights, len(yn)) if y_weights is not None else niv_masses(
        yn, rho, a, b, max_depth)
    if landmarks is not None and len(landmarks[0]) > 0:  # registration.py:74-83
        if x_weights is None:
            sx = sx * rbf_masses(xn, landmarks[0], sigma)
        if y_weights is None:
            sy = sy * rbf_masses(yn, landmarks[1], sigma)
    mx, my = rescale(sx, sy, dt, eta)
    tree = tree_build(xn, mx, max_depth)
    d = xn.shape[1]
    pos = yn.copy()
    vel = np.zeros_like(pos)
    r_acc, t_acc = np.eye(d), np.zeros(d)
    t_prev = np.hstack([r_acc, t_acc[:, None]])
    gi = globals()["gpe"](pos, my, xn, mx, G, epsilon, nthreads) if gpe else float("nan")
    deltas, traj, accs = [], [], []
    converged = False
    iterations = 0
    for it in range(max_iters):
        if force_fn is not None:
            grav = force_fn(pos, my)
            na = 0
            v_new, disp = step(pos, vel, my, grav, dt, eta)
            R, t = solve_rigid(pos, pos + disp)
            pos = pos @ R.T + t
            vel = v_new @ R.T
            r_acc = R @ r_acc
            t_acc = t + R @ t_acc
        else:
            pos, vel, r_acc, t_acc, _, _, acc = iterate(tree, pos, vel, my, r_acc, t_acc, theta,
                                                        G, epsilon, dt, eta, nthreads)
            na = int(acc.sum())
        t_curr = np.hstack([r_acc, t_acc[:, None]])
        delta = float(((t_curr - t_prev) ** 2).sum())
        t_prev = t_curr
        iterations = it + 1
        deltas.append(delta)
        traj.append(t_curr.copy())
        accs.append(na)
        if delta < conv_tol:
            converged = True
            break
    gf = globals()["gpe"](pos, my, xn, mx, G, epsilon, nthreads) if gpe else float("nan")
    t_orig = denormalize_translation(r_acc, t_acc, ctx)
    return OracleResult(r_acc, t_acc, r_acc, t_orig, iterations, converged, gi, gf, deltas,
                        traj, accs)


# ---------------------------------------------------------------------------
# registration.py:178-206 -- register_sequence; poses composed like
# core.py:87-96 (compose = self after other, inverse = (R^T, -R^T t))
# ---------------------------------------------------------------------------
@dataclass
class OracleSequence:
    pairwise: list  # (R, t) in the original frame per pair
    trajectory: list  # (R, t) absolute poses, frame-0 coordinates
    failed: list


def register_sequence(frames, **kw):
    """Frame i (template) onto frame i+1 (reference); a pair that raises the
    reference's validation errors (here: an empty cloud, or the degenerate
    extent of normalize.py:52-53) contributes an identity transform and
    failed=True."""
    frames = [_f64(f) for f in frames]
    d = frames[0].shape[1]
    pairwise, failed = [], []
    for i in range(len(frames) - 1):
        try:
            if len(frames[i]) == 0 or len(frames[i + 1]) == 0:
                raise ValueError("EmptyCloud")  # PointCloud.require_nonempty (core.py)
            r = register(frames[i + 1], frames[i], **kw)
            pairwise.append((r.R_orig, r.t_orig))
            failed.append(False)
        except ValueError:  # DegenerateExtent
            pairwise.append((np.eye(d), np.zeros(d)))
            failed.append(True)
    poses = [(np.eye(d), np.zeros(d))]
    for R, t in pairwise:
        Ri, ti = R.T, -R.T @ t  # inverse (core.py:94-96)
        P, p = poses[-1]
        poses.append((P @ Ri, P @ ti + p))  # compose (core.py:87-92)
    return OracleSequence(pairwise, poses, failed)
