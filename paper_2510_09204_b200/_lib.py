"""ctypes binding of the C ABI in include/sfb.h (libsfb.so, built in-tree).

Loading fails loudly: there is no CPU fallback for the SF solve."""

from __future__ import annotations

import ctypes
import os

from .errors import NativeError, SetupError, ShapeError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFB_LIB", os.path.join(HERE, "libsfb.so"))

SFB_OK, SFB_EINVAL, SFB_ESETUP, SFB_ECUDA, SFB_ENOMEM = 0, 1, 2, 3, 4
MODE = {"projection": 0, "smoothness": 1}
STATUS = {0: "max_iters", 1: "converged_primal", 2: "converged_fp"}
EXPORTS = ("sfb_plan_create", "sfb_plan_destroy", "sfb_plan_cond", "sfb_solve",
           "sfb_smem_bytes", "sfb_launch_info", "sfb_last_error", "sfb_abi_version", "sfb_kinematic_peaks",
           "sfb_trajectory_metrics", "sfb_trajectory_metrics_work", "sfb_analysis_vars")


class Dims(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("n_d", ctypes.c_int32), ("n_basis", ctypes.c_int32),
                ("num_steps", ctypes.c_int32), ("n_obs", ctypes.c_int32), ("n_bnd", ctypes.c_int32)]


class Batch(ctypes.Structure):
    _fields_ = [("n_members", ctypes.c_int32), ("n_instances", ctypes.c_int32),
                ("member_instance", ctypes.c_void_p), ("xi0", ctypes.c_void_p),
                ("lam0", ctypes.c_void_p), ("target", ctypes.c_void_p),
                ("bvals", ctypes.c_void_p), ("box", ctypes.c_void_p),
                ("obs_pos", ctypes.c_void_p), ("obs_axes", ctypes.c_void_p),
                ("pair_axes", ctypes.c_void_p), ("flags", ctypes.c_int32)]


BATCH_STATIC_OBSTACLES = 1


class Config(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_double), ("primal_tol", ctypes.c_double),
                ("fp_tol", ctypes.c_double), ("d_max", ctypes.c_double),
                ("max_iters", ctypes.c_int32), ("early_exit", ctypes.c_int32),
                ("cluster", ctypes.c_int32)]


class Out(ctypes.Structure):
    _fields_ = [("xi", ctypes.c_void_p), ("lam", ctypes.c_void_p), ("primal", ctypes.c_void_p),
                ("eq_max", ctypes.c_void_p), ("iterations", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("trace", ctypes.c_void_p),
                ("counters", ctypes.c_void_p)]


_LIB = None


def lib() -> ctypes.CDLL:
    """Load libsfb.so once; raise NativeError if it is missing or incomplete."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise NativeError(f"cannot load {LIB_PATH}: {exc}") from exc
    for name in EXPORTS:
        if not hasattr(L, name):
            raise NativeError(f"{LIB_PATH} does not export {name}")
    vp = ctypes.c_void_p
    L.sfb_plan_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(Dims), vp, vp, vp,
                                  ctypes.c_double, ctypes.c_int32]
    L.sfb_plan_create.restype = ctypes.c_int
    L.sfb_plan_destroy.argtypes = [vp]
    L.sfb_plan_destroy.restype = None
    L.sfb_plan_cond.argtypes = [vp]
    L.sfb_plan_cond.restype = ctypes.c_double
    L.sfb_smem_bytes.argtypes = [vp]
    L.sfb_smem_bytes.restype = ctypes.c_int64
    i32p = ctypes.POINTER(ctypes.c_int32)
    L.sfb_launch_info.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, i32p, i32p, i32p]
    L.sfb_launch_info.restype = ctypes.c_int
    L.sfb_solve.argtypes = [vp, ctypes.POINTER(Batch), ctypes.POINTER(Config), ctypes.POINTER(Out), vp]
    L.sfb_solve.restype = ctypes.c_int
    L.sfb_kinematic_peaks.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, vp, vp, ctypes.c_int32, vp, vp, vp]
    L.sfb_kinematic_peaks.restype = ctypes.c_int
    i32, i64 = ctypes.c_int32, ctypes.c_int64
    L.sfb_trajectory_metrics.argtypes = [vp, i32, i32, i32, i32, vp, i32, vp, vp, i32, vp, i32, i64,
                                         vp, vp, vp]
    L.sfb_trajectory_metrics.restype = ctypes.c_int
    L.sfb_trajectory_metrics_work.argtypes = [i32, i32, i32, i32, i32, i32]
    L.sfb_trajectory_metrics_work.restype = ctypes.c_int64
    L.sfb_analysis_vars.argtypes = [vp, i32, vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp,
                                    ctypes.c_double, vp, vp, vp, vp, vp, vp, vp, vp]
    L.sfb_analysis_vars.restype = ctypes.c_int
    L.sfb_last_error.argtypes = []
    L.sfb_last_error.restype = ctypes.c_char_p
    L.sfb_abi_version.argtypes = []
    L.sfb_abi_version.restype = ctypes.c_int32
    if L.sfb_abi_version() != 1:
        raise NativeError("libsfb.so ABI version mismatch")
    _LIB = L
    return L


def check(rc: int, what: str) -> None:
    if rc == SFB_OK:
        return
    msg = lib().sfb_last_error().decode(errors="replace")
    if rc == SFB_ESETUP:
        raise SetupError(msg)
    if rc == SFB_EINVAL:
        raise ShapeError(f"{what}: {msg}")
    raise NativeError(f"{what}: {msg} (code {rc})")
