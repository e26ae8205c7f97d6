"""ctypes binding of the C ABI in include/pf_b200.h (libpf_b200.so).

The shared library is the only compute path.  If it is missing the import
fails loudly -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.environ.get("PF_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                         "libpf_b200.so")

PF_OK, PF_EINVAL, PF_EDEGENERATE, PF_ECUDA, PF_ENOMEM, PF_EIO = 0, 1, 2, 3, 4, 5
PF_FP64, PF_FP32, PF_FP16, PF_FP16_PACKED = 0, 1, 2, 3


class pf_params(C.Structure):
    _fields_ = [
        ("drift_x", C.c_double),
        ("std_x", C.c_double),
        ("drift_y", C.c_double),
        ("std_y", C.c_double),
        ("bg_mean", C.c_double),
        ("fg_mean", C.c_double),
        ("likelihood_scale", C.c_double),
        ("disk_radius", C.c_int32),
        ("noise_std", C.c_double),
    ]


class pf_config(C.Structure):
    _fields_ = [
        ("precision", C.c_int32),
        ("K", C.c_int64),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("n_tracks", C.c_int32),
        ("n_videos", C.c_int32),
        ("seeds", C.POINTER(C.c_uint64)),
        ("params", pf_params),
        ("offsets_xy", C.POINTER(C.c_int32)),
        ("n_offsets", C.c_int32),
        ("tpb", C.c_int32),
        ("device", C.c_int32),
        ("start_x", C.c_double),
        ("start_y", C.c_double),
    ]


# every symbol include/pf_b200.h declares: (name, restype, argtypes)
_VP = C.c_void_p
SIGNATURES = [
    ("pf_version", C.c_char_p, []),
    ("pf_global_error", C.c_char_p, []),
    ("pf_create", C.c_int, [C.POINTER(_VP), C.POINTER(pf_config)]),
    ("pf_destroy", C.c_int, [_VP]),
    ("pf_last_error", C.c_char_p, [_VP]),
    ("pf_reset", C.c_int, [_VP, C.c_double, C.c_double]),
    ("pf_run", C.c_int, [_VP, _VP, C.c_int32, C.c_int32, _VP]),
    ("pf_step", C.c_int, [_VP, _VP, C.c_int32, _VP]),
    ("pf_run_async", C.c_int, [_VP, _VP, C.c_int32, C.c_int32, _VP, _VP]),
    ("pf_step_async", C.c_int, [_VP, _VP, C.c_int32, _VP, _VP]),
    ("pf_sync", C.c_int, [_VP]),
    ("pf_stream_wait", C.c_int, [_VP, _VP]),
    ("pf_degenerate_frame", C.c_int, [_VP]),
    ("pf_likelihood_maps", C.c_int, [_VP, _VP, C.c_int32, _VP]),
    ("pf_set_profiling", C.c_int, [_VP, C.c_int32]),
    ("pf_last_timings", C.c_int, [_VP, C.POINTER(C.c_float)]),
    ("pf_last_launches", C.c_int64, [_VP]),
    ("pf_set_trace", C.c_int, [_VP, C.c_int32]),
    ("pf_generate_video", C.c_int, [C.POINTER(pf_params), C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                    C.c_uint64, _VP, C.c_int32, _VP, _VP, C.c_int32]),
    ("pf_pfvd_info", C.c_int, [C.c_char_p, _VP]),
    ("pf_read_pfvd", C.c_int, [C.c_char_p, _VP, C.c_int64, _VP, C.c_int32]),
    ("pf_shard_create", C.c_int, [C.POINTER(_VP), C.POINTER(pf_config), C.c_int32, C.c_int32]),
    ("pf_shard_info", C.c_int, [_VP, _VP]),
    ("pf_shard_buffers", C.c_int, [_VP, _VP]),
    ("pf_shard_ipc_export", C.c_int, [_VP, _VP]),
    ("pf_shard_set_peer", C.c_int, [_VP, C.c_int32, _VP]),
    ("pf_shard_open_peer", C.c_int, [_VP, C.c_int32, _VP]),
    ("pf_shard_exchange", C.c_int, [_VP, _VP]),
    ("pf_shard_stream", C.c_void_p, [_VP]),
    ("pf_shard_begin", C.c_int, [_VP, _VP, C.c_int32, C.c_int32]),
    ("pf_shard_fused", C.c_int, [_VP, C.c_int32]),
    ("pf_shard_tables", C.c_int, [_VP]),
    ("pf_shard_finish", C.c_int, [_VP, C.c_int32]),
    ("pf_shard_end", C.c_int, [_VP, C.c_int32, _VP]),
    ("pf_shard_local_allgather", C.c_int, [_VP, C.c_int32, C.c_int32]),
    ("pf_get_trace", C.c_int, [_VP, _VP, C.c_int64]),
    ("pf_get_state", C.c_int, [_VP, C.c_int32, _VP, _VP, _VP]),
    ("pf_set_rng_philox", C.c_int, [_VP, _VP]),
    ("pf_set_state", C.c_int, [_VP, C.c_int32, _VP, _VP, C.c_int64]),
    ("pf_get_debug", C.c_int, [_VP, C.c_int32, _VP, _VP]),
    ("pf_stage_create", C.c_int, [C.POINTER(_VP), C.c_int32, C.c_int64, C.POINTER(pf_params), _VP, C.c_int32, C.c_int32]),
    ("pf_stage_destroy", C.c_int, [_VP]),
    ("pf_stage_error", C.c_char_p, [_VP]),
    ("pf_stage_init", C.c_int, [_VP, C.c_double, C.c_double]),
    ("pf_stage_propagate", C.c_int, [_VP, _VP]),
    ("pf_stage_likelihood", C.c_int, [_VP, _VP, C.c_int32, C.c_int32]),
    ("pf_stage_max", C.c_int, [_VP, C.POINTER(C.c_double)]),
    ("pf_stage_weight", C.c_int, [_VP, C.c_double, C.POINTER(C.c_double)]),
    ("pf_stage_normalize", C.c_int, [_VP, C.c_double]),
    ("pf_stage_estimate", C.c_int, [_VP, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("pf_stage_resample", C.c_int, [_VP, C.c_double]),
    ("pf_stage_get", C.c_int, [_VP, C.c_int32, _VP]),
    ("pf_stage_set", C.c_int, [_VP, C.c_int32, _VP]),
    ("pf_systematic_ancestors", C.c_int, [_VP, C.c_int64, C.c_double, _VP, C.c_int32]),
    ("pf_rng_normals", C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, _VP, C.c_int32]),
    ("pf_rng_uniforms", C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, _VP, C.c_int32]),
    ("pf_exp16_table", C.c_int, [_VP]),
    ("pf_exp16_device", C.c_int, [_VP, C.c_int32]),
    ("pf_philox_create", C.c_int, [C.POINTER(_VP), _VP, C.c_int32]),
    ("pf_philox_destroy", C.c_int, [_VP]),
    ("pf_philox_normals", C.c_int, [_VP, C.c_int64, _VP]),
    ("pf_philox_uniforms", C.c_int, [_VP, C.c_int64, _VP]),
    ("pf_philox_normals_device", C.c_int, [_VP, C.c_int64, _VP, _VP]),
]

_lib = None


def lib():
    """Load libpf_b200.so (raises if the CUDA extension has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            if os.environ.get("PF_B200_LIB") and not hasattr(L, name):
                continue  # A/B runs against an older build (tools/ab.sh)
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def check(rc: int, msg_fn):
    if rc == PF_OK:
        return
    msg = msg_fn()
    if isinstance(msg, bytes):
        msg = msg.decode(errors="replace")
    raise NativeError(rc, msg)
