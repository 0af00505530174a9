"""ctypes binding of the C ABI in include/jmppi.h (libjmppi.so, built in-tree).

There is no CPU fallback: if the library is missing or the GPU is absent the
call raises.  Structures mirror the header field by field.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["JM_LIB"]) if os.environ.get("JM_LIB") else _HERE / "libjmppi.so"  # JM_LIB: tuning builds

JM_OK = 0
JM_ERR_CONFIG = 1
JM_ERR_VALUE = 2
JM_ERR_NO_VIABLE = 3
JM_ERR_NOISE = 4
JM_ERR_CUDA = 5
JM_ERR_UNSUPPORTED = 6
JM_ERR_DIVERGED = 7

JM_MODEL_INTEGRATOR, JM_MODEL_CARTPOLE, JM_MODEL_QUADROTOR, JM_MODEL_LINEAR = 0, 1, 2, 3
JM_COST_DIAG_QUADRATIC, JM_COST_CARTPOLE_SWINGUP, JM_COST_QUADROTOR_HOVER = 0, 1, 2
JM_JUMP_CONTROL, JM_JUMP_STATE = 0, 1
JM_NOISE_PHILOX, JM_NOISE_HBM = 0, 1
JM_F32, JM_F64 = 0, 1
JM_JUMPS_BERNOULLI, JM_JUMPS_POISSON = 0, 1

_d = C.c_double
_i32 = C.c_int32
_i64 = C.c_int64
_u64 = C.c_uint64
_pd = C.POINTER(C.c_double)
_pi64 = C.POINTER(C.c_int64)
_pi32 = C.POINTER(C.c_int32)
_pu64 = C.POINTER(C.c_uint64)
_vp = C.c_void_p


class ModelDesc(C.Structure):
    _fields_ = [
        ("kind", _i32), ("state_dim", _i32), ("control_dim", _i32), ("has_limits", _i32),
        ("params", _d * 8), ("u_lo", _d * 4), ("u_hi", _d * 4),
        ("jump_channel", _i32), ("jump_dim", _i32), ("jump_rows", _i32 * 4),
        ("jump_scale_unit", _i32), ("pad_lin_", _i32), ("lin_A", _d * 144), ("lin_G", _d * 48),
    ]


class CostDesc(C.Structure):
    _fields_ = [
        ("kind", _i32), ("pad_", _i32),
        ("weights", _d * 12), ("target", _d * 12), ("terminal_scale", _d),
        ("R", _d * 16), ("lambda_", _d), ("c", _d),
        ("general_channel", _i32), ("pad2_", _i32), ("cal_b", _d * 16), ("bb", _d * 16),
    ]


class MppiDesc(C.Structure):
    _fields_ = [
        ("lambda_", _d), ("c", _d), ("dt", _d), ("nu", _d),
        ("horizon", _i32), ("samples", _i32), ("control_dim", _i32), ("jump_enabled", _i32),
        ("sigma_d", _d * 16), ("sigma_j", _d * 16), ("mark_mean", _d * 4),
        ("precision", _i32), ("noise_source", _i32), ("sample_offset", _i64),
        ("block_threads", _i32), ("jump_process", _i32),
    ]


class Diag(C.Structure):
    _fields_ = [("min_cost", _d), ("ess", _d), ("normaliser", _d), ("n_finite", _i64)]


# name -> (restype, argtypes); every symbol include/jmppi.h declares
SIGNATURES = {
    "jm_abi_version": (C.c_int, []),
    "jm_last_error": (C.c_char_p, [_vp]),
    "jm_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "jm_create": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(CostDesc), C.POINTER(MppiDesc), C.c_int,
                            C.POINTER(_vp)]),
    "jm_destroy": (C.c_int, [_vp]),
    "jm_set_stream": (C.c_int, [_vp, _vp]),
    "jm_record_doubles": (C.c_int, [_vp, _pi64]),
    "jm_iteration_host": (C.c_int, [_vp, _pd, _pd, _u64, _u64, _vp, _vp, _pd, _pd, _pd, _pd, _pd, _pd,
                                    _pi64, C.POINTER(Diag), _pd, _pd, _pu64]),
    "jm_stash_fetch": (C.c_int, [_vp, _u64, _d, _d, _pd]),
    "jm_iteration_dropin": (C.c_int, [_vp, _vp, _vp, _vp, _u64, _u64, _vp, _vp]),
    "jm_dropin_doubles": (C.c_int64, [_vp]),
    "jm_stash_release": (C.c_int, [_vp, _u64]),
    "jm_upload_inputs": (C.c_int, [_vp, _pd, _pd]),
    "jm_rollout_dev": (C.c_int, [_vp, _vp, _vp, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "jm_reduce_dev": (C.c_int, [_vp, _vp]),
    "jm_finalize_dev": (C.c_int, [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "jm_weights_dev": (C.c_int, [_vp, _vp, _vp, _vp]),
    "jm_shift_dev": (C.c_int, [_vp, _vp, _vp, _vp]),
    "jm_shift_host": (C.c_int, [C.c_int, _i32, _i32, _pd, _pd, _pd]),
    "jm_compute_weights_host": (C.c_int, [C.c_int, _i64, _pd, _d, _pd]),
    "jm_update_controls_host": (C.c_int, [C.c_int, _i64, _i32, _i32, _pd, _pd, _d, _d, _pd, _pd, _pd, _pd]),
    "jm_sample_noise_host": (C.c_int, [_vp, _u64, _u64, _pd, _pi64, _pd, _pd]),
    "jm_sample_noise_dev": (C.c_int, [_vp, _u64, _u64, _vp, _vp]),
    "jm_closed_loop_host": (C.c_int, [_vp, _pd, _pd, _u64, _i32, _pd, _pd, _pi64, _pd, _pi32, _pi32]),
    "jm_peer_buffer_doubles": (C.c_int64, [_vp, _i32]),
    "jm_loop_rollout_push": (C.c_int, [_vp, _vp, _i32, _i32]),
    "jm_loop_finish_peers": (C.c_int, [_vp, _vp, _i32]),
    "jm_loop_rollout_reduce_push": (C.c_int, [_vp, _vp, _i32, _i32]),
    "jm_loop_finish_reduced_peers": (C.c_int, [_vp, _vp, _i32]),
    "jm_batch_loop_host": (C.c_int, [_vp, _i32, _pd, _pd, _pu64, _pi32, _i32, _pd, _pd, _pi64, _pd, _pi32, _pi32]),
    "jm_loop_init": (C.c_int, [_vp, _pd, _pd, _u64, _u64, _i32]),
    "jm_loop_step": (C.c_int, [_vp]),
    "jm_loop_history": (C.c_int, [_vp, _i32, _pd, _pd, _pi64]),
    "jm_loop_timeline": (C.c_int, [_vp, _i32, _pu64]),
    "jm_loop_rollout": (C.c_int, [_vp, _vp]),
    "jm_loop_finish": (C.c_int, [_vp, _vp, _i32]),
    "jm_loop_read": (C.c_int, [_vp, _pd, _pu64, _pi32, _pi32, _pi32]),
    "jm_microbench": (C.c_int, [C.c_int, _pd, _pd, _pd]),
    "jm_bench_loop": (C.c_int, [_vp, _i32, _i64, _i32, _pd, _pd]),
    "jm_bench_iteration": (C.c_int, [_vp, _i32, _i64, _pd, _pd]),
    "jm_kernel_name": (C.c_char_p, [_vp]),
    "jm_launches_per_iteration": (C.c_int, [_vp, _pi32, _pi32]),
    "jm_transfer_bytes": (C.c_int, [_pi64, _pi64]),
}

_lock = threading.Lock()
_lib = None


class LibraryMissing(RuntimeError):
    pass


def load(path: os.PathLike = LIB_PATH) -> C.CDLL:
    """Load libjmppi.so (once).  Raises LibraryMissing when it was not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path)
        if not p.exists():
            raise LibraryMissing(
                f"{p} is not built (run `make -j8` or __graft_entry__.build()); "
                "this package has no CPU fallback"
            )
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.jm_abi_version() != 5:
            raise LibraryMissing("libjmppi.so ABI version mismatch")
        _lib = lib
        return lib


def last_error(ctx=None) -> str:
    msg = load().jm_last_error(ctx)
    return msg.decode() if msg else ""


def dptr(a):
    """double* of a C-contiguous float64 numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_pd)


def vptr(a):
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


def i64ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_pi64)
