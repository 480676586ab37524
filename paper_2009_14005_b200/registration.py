"""The registration driver (mirrors gravreg/registration.py).

``register`` keeps the reference signature and semantics
(registration.py:91-166) and runs the whole pipeline in one call into
libfga (``fga_register``): device normalization, NIV masses + rescale, GPU
octree build, energy, and the iteration loop -- force pass with the fused
Euler-Cromer step and Kabsch partial sums, fp64 3x3 SVD update, convergence
flag on the device -- then the denormalized transform.

B200-side options (extra ``RegisterOptions`` fields, defaults keep reference
behaviour): ``precision`` ("fp32" fast path / "fp64" reference arithmetic),
``poll_every`` (iterations enqueued between host polls), ``device``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .core import (
    FgaParams,
    IterationRecord,
    PointCloud,
    RegistrationResult,
    RigidTransform,
    default_params,
    validate,
)
from .errors import DeviceError, EmptyCloud, GravregError, InvalidParam
from .masses import check_weights

# Mass rescale constants (registration.py:41-54); the device applies them in
# setup.cu (launch_rescale); listed here for API parity.
FIELD_MASS = 16.0
FIELD_MASS_POINTS = 2000
REFERENCE_POINT_CAP = 0.022
TEMPLATE_PEAK_MASS = 0.1


@dataclass
class RegisterOptions:
    """Trace and behaviour flags (registration.py:22-31) + device knobs."""

    trace_gpe: bool = False
    normalize: bool = True
    x_weights: np.ndarray | None = None
    y_weights: np.ndarray | None = None
    record_iterations: bool = False
    precision: str = "fp32"
    poll_every: int = 8
    device: int | None = None
    compute_gpe: bool = True
    mass_field: str = "niv"   # "niv" (reference SPM default) or "knn" (configs[3])
    knn_k: int = 16
    count_visits: bool = False  # FP32 pass also counts node visits (2.5% slower)


def _c_options(options: RegisterOptions, xw, yw, lm=None) -> N.COptions:
    if options.precision not in ("fp32", "fp64"):
        raise GravregError(f"precision must be 'fp32' or 'fp64', got {options.precision!r}")
    if options.mass_field not in ("niv", "knn"):
        raise GravregError(f"mass_field must be 'niv' or 'knn', got {options.mass_field!r}")
    return N.COptions(int(bool(options.trace_gpe)), int(bool(options.normalize)),
                      int(bool(options.record_iterations)),
                      N.PREC_FP64 if options.precision == "fp64" else N.PREC_FP32,
                      N.ptr(xw), N.ptr(yw), int(options.poll_every),
                      int(bool(options.compute_gpe)), 1 if options.mass_field == "knn" else 0,
                      int(options.knn_k), N.ptr(lm[0]) if lm else None,
                      N.ptr(lm[1]) if lm else None, len(lm[0]) if lm else 0,
                      int(bool(options.count_visits)))


def _check_inputs(x, y, landmarks, params, options):
    validate(params)
    x.require_nonempty()
    y.require_nonempty()
    if x.dim != y.dim:
        raise EmptyCloud(f"dimension mismatch: {x.dim} vs {y.dim}")
    lm = None
    if landmarks is not None:
        landmarks.check_bounds(len(y), len(x))
        if len(landmarks) > 0:  # registration.py:74-83: SPM = NIV * RBF(landmarks)
            if params.sigma <= 0:
                raise InvalidParam("sigma", params.sigma)
            lm = (np.ascontiguousarray(landmarks.reference_indices(), dtype=np.int64),
                  np.ascontiguousarray(landmarks.template_indices(), dtype=np.int64))
    xw = check_weights(len(x), options.x_weights) if options.x_weights is not None else None
    yw = check_weights(len(y), options.y_weights) if options.y_weights is not None else None
    return xw, yw, lm


def register(x: PointCloud, y: PointCloud, landmarks=None, params: FgaParams | None = None,
             options: RegisterOptions | None = None) -> RegistrationResult:
    """Align template ``y`` to reference ``x``; the transform is expressed in
    the original (unnormalized) frame (registration.py:91-166)."""
    params = params or default_params()
    options = options or RegisterOptions()
    xw, yw, lm = _check_inputs(x, y, landmarks, params, options)
    c = N.context(options.device)
    mi = int(params.max_iters)
    deltas = np.zeros(mi)
    traj = np.zeros((mi, 3, 4))
    gtrace = np.zeros(mi)
    inter = np.zeros(mi, np.int64)
    res = N.CResult()
    cp = N.make_params(params)
    co = _c_options(options, xw, yw, lm)
    N.check(N.lib().fga_register(c.handle, N.ptr(x.points), len(x), N.ptr(y.points), len(y),
                                 x.dim, N.ctypes.byref(cp), N.ctypes.byref(co),
                                 N.ctypes.byref(res), N.ptr(deltas), N.ptr(traj), N.ptr(gtrace),
                                 N.ptr(inter)))
    return _result_from_c(res, deltas, traj, gtrace, inter, options, x.dim)


def _result_from_c(res, deltas, traj, gtrace, inter, options, dim=3) -> RegistrationResult:
    it = int(res.iterations)
    R = np.array(res.R).reshape(3, 3)[:dim, :dim].copy()
    t = np.array(res.t)[:dim].copy()
    if dim == 2:  # D = 2 ran as z = const: keep the in-plane block of [R|t]
        traj = traj[:, :2, [0, 1, 3]]
    gpe_trace = [float(v) for v in gtrace[:it]] if options.trace_gpe else []
    records = []
    if options.record_iterations:
        records = [IterationRecord(index=k, transform_delta=float(deltas[k]),
                                   gpe=gpe_trace[k] if options.trace_gpe else None)
                   for k in range(it)]
    compute_gpe = getattr(options, "compute_gpe", True)
    return RegistrationResult(
        transform=RigidTransform(R, t),
        iterations=it,
        gpe_trace=gpe_trace,
        converged=bool(res.converged),
        gpe_initial=float(res.gpe_initial) if compute_gpe else None,
        gpe_final=float(res.gpe_final) if compute_gpe else None,
        records=records,
        trajectory=traj[:it].copy(),
        interactions=inter[:it].copy(),
        timings_ms={"setup": float(res.setup_ms), "loop": float(res.loop_ms),
                    "gpe": float(res.gpe_ms)},
    )


@dataclass
class BatchResult:
    """Outcome of register_batch: one entry per pair; a pair that failed
    (empty / degenerate / unsupported) has results[i] = None and errors[i]
    set, the others are unaffected (like register_sequence's per-pair
    failure handling, registration.py:192-200)."""

    results: list
    errors: list
    interactions: np.ndarray | None = None
    status: np.ndarray | None = None  # per-pair FGA_* return code


def register_batch(pairs, params: FgaParams | None = None,
                   options: RegisterOptions | None = None,
                   workers: int | None = None) -> BatchResult:
    """register(x, y) for many independent (x, y) pairs: every pair the
    persistent batched kernel takes (D = 3, <= 8192 points per cloud, FP32
    forces, NIV or external masses, max_depth <= 21; csrc/batched.cu) runs in
    ONE launch, the others -- and any pair the kernel reports as over its
    limits (e.g. a node cap) -- through register() on up to `workers` host
    threads (default 4), so every pair gets the result register() gives it.  External weights in
    options.x_weights / y_weights must be lists (one array per pair); per-pair
    failures are reported in ``errors`` (registration.py:192-200)."""
    params = params or default_params()
    options = options or RegisterOptions()
    validate(params)
    pairs = list(pairs)
    P = len(pairs)
    if P == 0:
        return BatchResult([], [], np.zeros(0, np.int64), np.zeros(0, np.int32))
    for x, y in pairs:
        if x.dim != y.dim:
            raise EmptyCloud(f"dimension mismatch: {x.dim} vs {y.dim}")
    kernel_options = (options.precision == "fp32" and options.mass_field == "niv"
                      and not options.trace_gpe
                      and params.max_depth <= 21 and params.rho ** 3 <= 16384)
    in_kernel = [k for k, (x, y) in enumerate(pairs)
                 if kernel_options and x.dim == 3 and max(len(x), len(y)) <= 8192]
    results, errors = [None] * P, [None] * P
    inter = np.zeros(P, np.int64)
    status = np.zeros(P, np.int32)
    if in_kernel:
        br = _register_batch_kernel([pairs[k] for k in in_kernel], params, options,
                                    None if options.x_weights is None else
                                    [options.x_weights[k] for k in in_kernel],
                                    None if options.y_weights is None else
                                    [options.y_weights[k] for k in in_kernel])
        for j, k in enumerate(in_kernel):
            results[k], errors[k] = br.results[j], br.errors[j]
            inter[k], status[k] = br.interactions[j], br.status[j]
    kset = set(in_kernel)
    rest = [k for k in range(P) if k not in kset or status[k] == N.FGA_ERR_UNSUPPORTED]

    def one(k):
        x, y = pairs[k]
        o = RegisterOptions(**{**options.__dict__,
                               "x_weights": None if options.x_weights is None else
                               options.x_weights[k],
                               "y_weights": None if options.y_weights is None else
                               options.y_weights[k]})
        try:
            r = register(x, y, params=params, options=o)
            return r, None, int(r.interactions.sum()), 0
        except GravregError as e:
            return (None, e, 0,
                    N.FGA_ERR_UNSUPPORTED if isinstance(e, DeviceError) else N.FGA_ERR_INVALID)

    # the pairs the kernel does not take run through register() on up to
    # `workers` host threads, each with its own context and stream (one
    # pair's setup and tree build overlap another's iterations; results are
    # register()'s, whatever the thread)
    n_workers = min(workers or 4, len(rest))
    if n_workers > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=n_workers) as pool:
            outs = list(pool.map(one, rest))
    else:
        outs = [one(k) for k in rest]
    for k, (r, e, it, st) in zip(rest, outs):
        results[k], errors[k], inter[k], status[k] = r, e, it, st
    return BatchResult(results, errors, inter, status)


def _register_batch_kernel(pairs, params, options, xws, yws) -> BatchResult:
    """The persistent batched kernel on pairs it supports (fga_register_batch)."""
    P = len(pairs)
    xs = [np.ascontiguousarray(x.points, dtype=np.float64) for x, _ in pairs]
    ys = [np.ascontiguousarray(y.points, dtype=np.float64) for _, y in pairs]
    c = N.context(options.device)
    out = (N.CPairResult * P)()
    deltas = np.zeros((P, params.max_iters)) if options.record_iterations else None
    cp = N.make_params(params)
    if xws is None and yws is None:
        # one host array per cloud: staged to the device in the library (no
        # host-side concatenation of the clouds)
        co = _c_options(options, None, None)
        xp = np.array([a.ctypes.data for a in xs], dtype=np.uintp)
        yp = np.array([a.ctypes.data for a in ys], dtype=np.uintp)
        xn = np.array([len(a) for a in xs], dtype=np.int64)
        yn = np.array([len(a) for a in ys], dtype=np.int64)
        N.check(N.lib().fga_register_batch_list(c.handle, N.ptr(xp), N.ptr(xn), N.ptr(yp),
                                                N.ptr(yn), P, 3, N.ctypes.byref(cp),
                                                N.ctypes.byref(co), N.ctypes.addressof(out),
                                                N.ptr(deltas)))
    else:
        xoff = np.zeros(P + 1, np.int64)
        yoff = np.zeros(P + 1, np.int64)
        xoff[1:] = np.cumsum([len(a) for a in xs])
        yoff[1:] = np.cumsum([len(a) for a in ys])
        X = np.ascontiguousarray(np.concatenate(xs) if xoff[-1] else np.zeros((0, 3)))
        Y = np.ascontiguousarray(np.concatenate(ys) if yoff[-1] else np.zeros((0, 3)))
        xw = yw = None
        if xws is not None:
            xw = np.ascontiguousarray(np.concatenate(
                [check_weights(len(a), w) for a, w in zip(xs, xws)]))
        if yws is not None:
            yw = np.ascontiguousarray(np.concatenate(
                [check_weights(len(a), w) for a, w in zip(ys, yws)]))
        co = _c_options(options, xw, yw)
        N.check(N.lib().fga_register_batch(c.handle, N.ptr(X), N.ptr(xoff), N.ptr(Y), N.ptr(yoff),
                                           P, 3, N.ctypes.byref(cp), N.ctypes.byref(co),
                                           N.ctypes.addressof(out), N.ptr(deltas)))
    results, errors = [], []
    inter = np.zeros(P, np.int64)
    status = np.zeros(P, np.int32)
    for i, r in enumerate(out):
        inter[i] = r.interactions
        status[i] = r.status
        if r.status != 0:
            results.append(None)
            errors.append(N.error_for(r.status, f"pair {i}"))
            continue
        it = int(r.iterations)
        recs = []
        if deltas is not None:
            recs = [IterationRecord(index=k, transform_delta=float(deltas[i, k])) for k in range(it)]
        results.append(RegistrationResult(
            transform=RigidTransform(np.array(r.R).reshape(3, 3), np.array(r.t)),
            iterations=it, gpe_trace=[], converged=bool(r.converged),
            gpe_initial=float(r.gpe_initial) if options.compute_gpe else None,
            gpe_final=float(r.gpe_final) if options.compute_gpe else None,
            records=recs, interactions=None))
        errors.append(None)
    return BatchResult(results, errors, inter, status)


@dataclass
class SequenceResult:
    """Pairwise frame transforms plus composed absolute poses
    (registration.py:169-175)."""

    pairwise: list[RigidTransform]
    trajectory: list[RigidTransform]
    failed: list[bool] = field(default_factory=list)


def register_sequence(frames, params: FgaParams | None = None,
                      options: RegisterOptions | None = None, workers: int | None = None
                      ) -> SequenceResult:
    """Frame i (template) onto frame i+1 (reference), pairwise; a failed pair
    contributes an identity transform (registration.py:178-206).

    The pairs are independent, so they run concurrently: fragment-sized
    frames (<= 8192 points, no per-cloud weights) go to ONE persistent
    batched kernel (register_batch), larger ones (LiDAR scans) to `workers`
    host threads (default min(4, pairs)), each with its own context and
    stream, so one pair's setup and tree build overlap another's iterations
    (SURVEY §8(f) f2).  Each pair's result is the one register() gives."""
    frames = list(frames)
    if len(frames) < 2:
        raise EmptyCloud("sequence registration needs at least 2 frames")
    params = params or default_params()
    options = options or RegisterOptions()
    pairs = [(frames[i + 1], frames[i]) for i in range(len(frames) - 1)]
    batched = (len(pairs) > 1 and all(f.dim == 3 and len(f) <= 8192 for f in frames)
               and options.precision == "fp32" and options.mass_field == "niv"
               and not options.trace_gpe and options.normalize
               and options.x_weights is None and options.y_weights is None)
    if batched:
        # one persistent kernel; register_batch re-runs through register()
        # any pair over the kernel's limits (node cap, max_depth > 21)
        br = register_batch(pairs, params=params, options=options)
        outs = []
        for k, (res, err) in enumerate(zip(br.results, br.errors)):
            if err is not None and (not isinstance(err, GravregError)
                                    or isinstance(err, DeviceError)):
                raise err
            outs.append((res.transform, False) if res is not None else
                        (RigidTransform.identity(frames[k].dim), True))
    else:
        from concurrent.futures import ThreadPoolExecutor

        def one(k):
            x, y = pairs[k]
            try:
                return register(x=x, y=y, params=params, options=options).transform, False
            except DeviceError:
                raise
            except GravregError:
                return RigidTransform.identity(frames[k].dim), True

        n_workers = workers or min(4, len(pairs))
        if n_workers <= 1:
            outs = [one(k) for k in range(len(pairs))]
        else:
            with ThreadPoolExecutor(max_workers=n_workers) as pool:
                outs = list(pool.map(one, range(len(pairs))))
    pairwise = [o[0] for o in outs]
    failed = [o[1] for o in outs]
    poses = [RigidTransform.identity(frames[0].dim)]
    for tf in pairwise:
        poses.append(poses[-1].compose(tf.inverse()))
    return SequenceResult(pairwise=pairwise, trajectory=poses, failed=failed)
