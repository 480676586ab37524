"""ctypes binding of libfga.so (the C ABI declared in include/fga.h).

The library is built in-tree (``paper_2009_14005_b200/_lib/libfga.so``, see
``csrc/Makefile`` / ``__graft_entry__.build``).  There is no CPU fallback:
if the library or a CUDA device is missing every call raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os
import re
import sys
import threading

import numpy as np

from .errors import (
    SingularCollocation,
    DegenerateExtent,
    DeviceError,
    EmptyCloud,
    InvalidParam,
    LengthMismatch,
    NonFiniteWeight,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libfga.so")
# A/B experiments only: FGA_LIB_PATH points at an alternative in-tree build
LIB_PATH = os.environ.get("FGA_LIB_PATH") or LIB_PATH

FGA_OK = 0
FGA_ERR_INVALID = -1
FGA_ERR_CUDA = -2
FGA_ERR_NOMEM = -3
FGA_ERR_UNSUPPORTED = -4
FGA_ERR_EMPTY = -5
FGA_ERR_DEGENERATE = -6
FGA_ERR_NONFINITE = -7
FGA_ERR_LENGTH = -8
FGA_ERR_STATE = -9
FGA_ERR_SINGULAR = -10
FGA_ERR_PARSE = -11

PREC_FP32 = 0
PREC_FP64 = 1

_c_int = ctypes.c_int
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_dbl = ctypes.c_double
_vp = ctypes.c_void_p


class CParams(ctypes.Structure):
    """fga_params (include/fga.h)."""

    _fields_ = [("G", _dbl), ("epsilon", _dbl), ("eta", _dbl), ("dt", _dbl), ("theta", _dbl),
                ("sigma", _dbl), ("rho", _i32), ("max_depth", _i32), ("norm_a", _dbl),
                ("norm_b", _dbl), ("conv_tol", _dbl), ("max_iters", _i32), ("pad_", _i32)]


class COptions(ctypes.Structure):
    """fga_options (include/fga.h)."""

    _fields_ = [("trace_gpe", _i32), ("normalize", _i32), ("record_iterations", _i32),
                ("precision", _i32), ("x_weights", _vp), ("y_weights", _vp),
                ("poll_every", _i32), ("compute_gpe", _i32), ("mass_field", _i32),
                ("knn_k", _i32), ("x_landmarks", _vp), ("y_landmarks", _vp),
                ("n_landmarks", _i32), ("count_visits", _i32)]


class CResult(ctypes.Structure):
    """fga_result (include/fga.h)."""

    _fields_ = [("R", _dbl * 9), ("t", _dbl * 3), ("R_norm", _dbl * 9), ("t_norm", _dbl * 3),
                ("iterations", _i64), ("converged", _i32), ("pad_", _i32),
                ("gpe_initial", _dbl), ("gpe_final", _dbl), ("norm_ctx", _dbl * 10),
                ("interactions", _i64), ("visits", _i64), ("n_nodes", _i64),
                ("setup_ms", _dbl), ("loop_ms", _dbl), ("gpe_ms", _dbl)]


class CPairResult(ctypes.Structure):
    """fga_pair_result (include/fga.h)."""

    _fields_ = [("R", _dbl * 9), ("t", _dbl * 3), ("iterations", _i64), ("converged", _i32),
                ("status", _i32), ("gpe_initial", _dbl), ("gpe_final", _dbl),
                ("interactions", _i64), ("n_nodes", _i64)]


# name -> (restype, argtypes); every symbol include/fga.h declares
SIGNATURES = {
    "fga_version": (_c_int, []),
    "fga_last_error": (ctypes.c_char_p, []),
    "fga_device_count": (_c_int, [ctypes.POINTER(_c_int)]),
    "fga_create": (_c_int, [ctypes.POINTER(_vp), _c_int]),
    "fga_destroy": (_c_int, [_vp]),
    "fga_set_stream": (_c_int, [_vp, _vp]),
    "fga_synchronize": (_c_int, [_vp]),
    "fga_register": (_c_int, [_vp, _vp, _i64, _vp, _i64, _c_int, ctypes.POINTER(CParams),
                              ctypes.POINTER(COptions), ctypes.POINTER(CResult), _vp, _vp, _vp,
                              _vp]),
    "fga_register_batch": (_c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _c_int,
                                    ctypes.POINTER(CParams), ctypes.POINTER(COptions), _vp,
                                    _vp]),
    "fga_register_batch_list": (_c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _c_int,
                                         ctypes.POINTER(CParams), ctypes.POINTER(COptions), _vp,
                                         _vp]),
    "fga_register_batch_dev": (_c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _c_int, _c_int, _c_int,
                                        ctypes.POINTER(CParams), ctypes.POINTER(COptions), _vp,
                                        _vp]),
    "fga_session_begin": (_c_int, [_vp, _vp, _i64, _vp, _i64, _c_int, ctypes.POINTER(CParams),
                                   ctypes.POINTER(COptions), _c_int, _c_int]),
    "fga_session_begin_dev": (_c_int, [_vp, _vp, _i64, _vp, _i64, _c_int,
                                       ctypes.POINTER(CParams), ctypes.POINTER(COptions), _c_int,
                                       _c_int]),
    "fga_session_forces": (_c_int, [_vp]),
    "fga_session_sums": (_c_int, [_vp, ctypes.POINTER(_vp)]),
    "fga_session_bind_sums": (_c_int, [_vp, _vp]),
    "fga_session_update": (_c_int, [_vp]),
    "fga_session_iterate": (_c_int, [_vp, _c_int]),
    "fga_session_gpe": (_c_int, [_vp]),
    "fga_session_take_gpe": (_c_int, [_vp, ctypes.POINTER(_dbl)]),
    "fga_session_apply_pending": (_c_int, [_vp]),
    "fga_session_poll": (_c_int, [_vp, ctypes.POINTER(_c_int), ctypes.POINTER(_i64)]),
    "fga_session_finish": (_c_int, [_vp, ctypes.POINTER(CResult), _vp, _vp, _vp, _vp, _vp]),
    "fga_session_set_gpe": (_c_int, [_vp, _c_int, _dbl]),
    "fga_session_get_state": (_c_int, [_vp, _vp, _vp, _vp, _vp, ctypes.POINTER(_i64)]),
    "fga_session_set_state": (_c_int, [_vp, _vp, _vp, _vp, _vp, _i64]),
    "fga_parse_cloud": (_c_int, [ctypes.c_char_p, _i64, _vp, _i64, ctypes.POINTER(_i64),
                                 ctypes.POINTER(_c_int)]),
    "fga_parse_weights": (_c_int, [ctypes.c_char_p, _i64, _vp, _i64, ctypes.POINTER(_i64)]),
    "fga_session_masses": (_c_int, [_vp, _vp, _vp]),
    "fga_session_checkpoint": (_c_int, [_vp, _c_int]),
    "fga_session_info": (_c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "fga_tree_build": (_c_int, [_vp, _vp, _vp, _i64, _c_int, _c_int, ctypes.POINTER(_i64)]),
    "fga_tree_build_dev": (_c_int, [_vp, _vp, _vp, _i64, _c_int, ctypes.POINTER(_i64)]),
    "fga_tree_export": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "fga_tree_upload": (_c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _c_int, _c_int]),
    "fga_tree_generation": (_c_int, [_vp, ctypes.POINTER(_i64)]),
    "fga_last_interactions": (_c_int, [_vp, ctypes.POINTER(_i64)]),
    "fga_tree_forces": (_c_int, [_vp, _vp, _vp, _i64, _dbl, _dbl, _dbl, _c_int, _vp, _vp, _vp]),
    "fga_bh_forces_kernel": (_c_int, [_vp, _vp, _vp, _vp, _vp, _i64, _c_int, _vp, _vp, _i64,
                                      _c_int, _dbl, _dbl, _dbl, _i64, _vp, _vp]),
    "fga_direct_forces": (_c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _i64, _c_int, _dbl, _dbl,
                                   _c_int, _vp]),
    "fga_gpe_kernel": (_c_int, [_vp, _vp, _vp, _i64, _vp, _vp, _i64, _c_int, _dbl, _dbl, _c_int,
                                ctypes.POINTER(_dbl)]),
    "fga_knn": (_c_int, [_vp, _vp, _i64, _c_int, _c_int, _vp, _vp]),
    "fga_knn_masses": (_c_int, [_vp, _vp, _i64, _c_int, _c_int, _vp]),
    "fga_rbf_masses": (_c_int, [_vp, _vp, _i64, _c_int, _vp, _c_int, _dbl, _vp]),
    "fga_niv_masses": (_c_int, [_vp, _vp, _i64, _c_int, _c_int, _dbl, _dbl, _c_int, _vp]),
    "fga_normalize_pair": (_c_int, [_vp, _vp, _i64, _vp, _i64, _c_int, _dbl, _dbl, _vp, _vp,
                                    _vp]),
    "fga_solve_rigid": (_c_int, [_vp, _vp, _vp, _i64, _c_int, _vp, _vp,
                                 ctypes.POINTER(_i32)]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libfga.so (raises DeviceError when it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise DeviceError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import "
                        "__graft_entry__ as g; g.build()'` (no CPU fallback exists)")
                L = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def last_error() -> str:
    msg = lib().fga_last_error()
    return msg.decode() if msg else ""


_INVALID_RE = re.compile(r"invalid parameter (\w+)=(.*)$")


def error_for(rc: int, msg: str = ""):
    """Exception instance for a C return code (None for FGA_OK)."""
    if rc == FGA_OK:
        return None
    try:
        check_msg(rc, msg)
    except Exception as e:  # noqa: BLE001
        return e
    return None


def check_msg(rc: int, msg: str) -> None:
    """Raise the reference exception for return code ``rc`` with ``msg``."""
    if rc == FGA_OK:
        return
    if rc == FGA_ERR_INVALID:
        m = _INVALID_RE.search(msg)
        if m:
            raise InvalidParam(m.group(1), m.group(2))
        raise InvalidParam("argument", msg)
    if rc == FGA_ERR_EMPTY:
        raise EmptyCloud(msg)
    if rc == FGA_ERR_DEGENERATE:
        raise DegenerateExtent(msg)
    if rc == FGA_ERR_NONFINITE:
        raise NonFiniteWeight(msg)
    if rc == FGA_ERR_LENGTH:
        raise LengthMismatch(msg)
    if rc == FGA_ERR_SINGULAR:
        raise SingularCollocation(msg)
    raise DeviceError(f"libfga error {rc}: {msg}")


def check(rc: int) -> None:
    """Map a C return code onto the reference's exception classes."""
    if rc != FGA_OK:
        check_msg(rc, last_error())


def ptr(a) -> int | None:
    """Host numpy array -> void* (None passes NULL)."""
    if a is None:
        return None
    return a.ctypes.data


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class Context:
    """One fga_ctx (device memory + stream) per (process, device, thread)."""

    def __init__(self, device: int = 0):
        h = _vp()
        check(lib().fga_create(ctypes.byref(h), int(device)))
        self.handle = h
        self.device = int(device)

    def close(self):
        if getattr(self, "handle", None):
            lib().fga_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        check(lib().fga_set_stream(self.handle, stream_ptr))

    def sync(self):
        check(lib().fga_synchronize(self.handle))

    def tree_generation(self) -> int:
        """Counter bumped by every build/upload into this context's tree."""
        g = _i64(0)
        check(lib().fga_tree_generation(self.handle, ctypes.byref(g)))
        return int(g.value)


_ctx_local = threading.local()


def context(device: int | None = None) -> Context:
    """The calling thread's context for ``device`` (default: current torch
    device if torch is imported and CUDA is available, else 0)."""
    if device is None:
        device = 0
        torch = sys.modules.get("torch")
        if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
            device = torch.cuda.current_device()
    cache = getattr(_ctx_local, "cache", None)
    if cache is None:
        cache = _ctx_local.cache = {}
    c = cache.get(device)
    if c is None:
        c = cache[device] = Context(device)
    return c


def device_count() -> int:
    n = _c_int(0)
    rc = lib().fga_device_count(ctypes.byref(n))
    return int(n.value) if rc == FGA_OK else 0


def make_params(p) -> CParams:
    a, b = p.norm_range
    return CParams(float(p.G), float(p.epsilon), float(p.eta), float(p.dt), float(p.theta),
                   float(p.sigma), int(p.rho), int(p.max_depth), float(a), float(b),
                   float(p.conv_tol), int(p.max_iters), 0)
