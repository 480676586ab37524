"""Stepwise registration session (wraps the fga_session_* C ABI).

``register`` runs the whole loop inside one C call; this wrapper exposes the
same loop one stream-ordered piece at a time, for (a) the multi-GPU driver
(distributed.py), which all-reduces the 18-double sums buffer between the
force pass and the rigid update, and (b) bench.py, which times single
iterations on device-resident inputs.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .core import FgaParams, default_params, validate
from .masses import check_weights
from .registration import RegisterOptions, _c_options, _result_from_c

SUMS_LEN = 18
SUM_ACCEPTED = 15
SUM_VISITS = 16
SUM_GPE = 17


class Session:
    """One registration on one device (optionally one shard of the template)."""

    def __init__(self, x, y, params: FgaParams | None = None,
                 options: RegisterOptions | None = None, shard_rank: int = 0,
                 shard_count: int = 1, device: int | None = None, stream: int | None = None,
                 device_inputs: tuple | None = None, ctx: N.Context | None = None):
        """x, y: PointCloud (host) -- or ``device_inputs=(x_ptr, n, y_ptr, m)``
        for (n,3)/(m,3) fp64 arrays already resident on the device."""
        self.params = params or default_params()
        self.options = options or RegisterOptions()
        validate(self.params)
        self.ctx = ctx or N.context(device if device is not None else self.options.device)
        if stream is not None:
            self.ctx.set_stream(stream)
        self._cp = N.make_params(self.params)
        n_x = device_inputs[1] if device_inputs is not None else len(x)
        n_y = device_inputs[3] if device_inputs is not None else len(y)
        o = self.options
        self._xw = check_weights(n_x, o.x_weights) if o.x_weights is not None else None
        self._yw = check_weights(n_y, o.y_weights) if o.y_weights is not None else None
        self._co = _c_options(self.options, self._xw, self._yw)
        L = N.lib()
        h = self.ctx.handle
        if device_inputs is not None:
            xp, n, yp, m = device_inputs
            N.check(L.fga_session_begin_dev(h, xp, n, yp, m, 3, ctypes.byref(self._cp),
                                            ctypes.byref(self._co), shard_rank, shard_count))
        else:
            self._x, self._y = x, y
            N.check(L.fga_session_begin(h, N.ptr(x.points), len(x), N.ptr(y.points), len(y),
                                        x.dim, ctypes.byref(self._cp), ctypes.byref(self._co),
                                        shard_rank, shard_count))
        m_local = N._i64(0)
        nn = N._i64(0)
        N.check(L.fga_session_info(h, ctypes.byref(m_local), ctypes.byref(nn)))
        self.m_local = int(m_local.value)
        self.n_nodes = int(nn.value)
        self.shard_count = shard_count
        self.dim = 3 if device_inputs is not None else x.dim
        self.n, self.m = int(n_x), int(n_y)

    def get_state(self):
        """Iteration state entering the next iteration (normalized frame, input
        order): dict(positions, velocities, R_acc, t_acc, iteration)."""
        pos = np.zeros((self.m, 3))
        vel = np.zeros((self.m, 3))
        R = np.zeros(9)
        t = np.zeros(3)
        it = N._i64(0)
        N.check(N.lib().fga_session_get_state(self.ctx.handle, N.ptr(pos), N.ptr(vel), N.ptr(R),
                                              N.ptr(t), ctypes.byref(it)))
        return {"positions": pos, "velocities": vel, "R_acc": R.reshape(3, 3), "t_acc": t,
                "iteration": int(it.value)}

    def set_state(self, positions, velocities, R_acc, t_acc, iteration: int):
        """Resume from a state (see get_state); e.g. a checkpoint, or the
        reference's own state for teacher-forced parity."""
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(self.m, 3)
        vel = np.ascontiguousarray(velocities, dtype=np.float64).reshape(self.m, 3)
        R = np.ascontiguousarray(R_acc, dtype=np.float64).reshape(9)
        t = np.ascontiguousarray(t_acc, dtype=np.float64).reshape(3)
        N.check(N.lib().fga_session_set_state(self.ctx.handle, N.ptr(pos), N.ptr(vel), N.ptr(R),
                                              N.ptr(t), int(iteration)))

    def checkpoint(self):
        """Save this shard's iteration state on the device (fga_session_checkpoint)."""
        N.check(N.lib().fga_session_checkpoint(self.ctx.handle, 0))

    def restore(self):
        """Return to the last checkpoint (stream-ordered device copy)."""
        N.check(N.lib().fga_session_checkpoint(self.ctx.handle, 1))

    def masses(self):
        """(mx, my): the rescaled mass fields in input order (fga_session_masses)."""
        mx = np.empty(self.n)
        my = np.empty(self.m)
        N.check(N.lib().fga_session_masses(self.ctx.handle, N.ptr(mx), N.ptr(my)))
        return mx, my

    # ---- stream-ordered pieces
    def bind_sums(self, dev_ptr: int):
        N.check(N.lib().fga_session_bind_sums(self.ctx.handle, dev_ptr))

    def sums_ptr(self) -> int:
        p = N._vp()
        N.check(N.lib().fga_session_sums(self.ctx.handle, ctypes.byref(p)))
        return int(p.value)

    def forces(self):
        N.check(N.lib().fga_session_forces(self.ctx.handle))

    def update(self):
        N.check(N.lib().fga_session_update(self.ctx.handle))

    def iterate(self, k: int = 1):
        N.check(N.lib().fga_session_iterate(self.ctx.handle, int(k)))

    def gpe(self):
        N.check(N.lib().fga_session_gpe(self.ctx.handle))

    def take_gpe(self) -> float:
        v = N._dbl(0.0)
        N.check(N.lib().fga_session_take_gpe(self.ctx.handle, ctypes.byref(v)))
        return float(v.value)

    def set_gpe(self, which: int, value: float):
        N.check(N.lib().fga_session_set_gpe(self.ctx.handle, int(which), float(value)))

    def apply_pending(self):
        N.check(N.lib().fga_session_apply_pending(self.ctx.handle))

    def poll(self):
        done = N._c_int(0)
        it = N._i64(0)
        N.check(N.lib().fga_session_poll(self.ctx.handle, ctypes.byref(done), ctypes.byref(it)))
        return bool(done.value), int(it.value)

    def finish(self):
        mi = int(self.params.max_iters)
        deltas = np.zeros(mi)
        traj = np.zeros((mi, 3, 4))
        gtrace = np.zeros(mi)
        inter = np.zeros(mi, np.int64)
        visits = np.zeros(mi, np.int64)
        res = N.CResult()
        N.check(N.lib().fga_session_finish(self.ctx.handle, ctypes.byref(res), N.ptr(deltas),
                                           N.ptr(traj), N.ptr(gtrace), N.ptr(inter),
                                           N.ptr(visits)))
        out = _result_from_c(res, deltas, traj, gtrace, inter, self.options, self.dim)
        out.visits_per_iter = visits[:out.iterations].copy()
        return out
