"""ctypes binding of libsfb.so (include/sfb.h).

There is no fallback: importing the solver without the built library, or
using it without a CUDA device, raises.  The library is built in-tree by
``python -m paper_1604_01093_b200._build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libsfb.so"

SFB_OK = 0
SFB_E_ARG = 1
SFB_E_CUDA = 2
SFB_E_OOM = 3
SFB_E_PCG_NONFINITE = 4
SFB_E_STATE = 5


class SfbError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"sfb error {code}: {message}")
        self.code = code


class FrameDesc(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32),
        ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
        ("valid_depth", C.c_void_p), ("valid_normal", C.c_void_p),
        ("points", C.c_void_p), ("normals", C.c_void_p), ("grad", C.c_void_p),
    ]


class Weights(C.Structure):
    _fields_ = [("sparse", C.c_double), ("photo", C.c_double), ("geo", C.c_double)]


class Config(C.Structure):
    _fields_ = [
        ("geo_distance_max", C.c_double), ("geo_normal_min", C.c_double),
        ("dense_pixel_stride", C.c_int32), ("dense_bidirectional", C.c_int32),
    ]


class Rounding(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("matvec_c", "matvec_f", "gemm33", "apply_n", "apply_1", "dot3")]


class VerifyConfig(C.Structure):
    _fields_ = [("depth_max", C.c_double), ("normal_min", C.c_double), ("color_max", C.c_double),
                ("apply_n", C.c_int32), ("apply_1", C.c_int32), ("apply_nf", C.c_int32),
                ("apply_1f", C.c_int32)]


class IterResult(C.Structure):
    _fields_ = [
        ("e_sparse", C.c_double), ("e_photo", C.c_double), ("e_geo", C.c_double),
        ("pcg_iterations", C.c_int32), ("pcg_status", C.c_int32),
        ("pcg_relative", C.c_double), ("step_norm", C.c_double),
        ("ea_sparse", C.c_double), ("ea_photo", C.c_double), ("ea_geo", C.c_double),
    ]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double
_PD = C.POINTER(C.c_double)
# sfb_allreduce_fn (include/sfb.h): sum a device buffer across ranks in place
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)

# name -> argtypes (all return int status except the two noted)
SIGNATURES = {
    "sfb_ctx_create": [_I32, C.POINTER(_P)],
    "sfb_ctx_destroy": [_P],
    "sfb_ctx_set_rounding": [_P, C.POINTER(Rounding)],
    "sfb_frames_upload": [_P, _I32, C.POINTER(FrameDesc), _P],
    "sfb_frames_release": [_P, _I32, _P],
    "sfb_problem_create": [_P, _I32, _P, _I32, _P, _P, _P, _P, _P, C.POINTER(_P)],
    "sfb_problem_attach_frames": [_P, _P],
    "sfb_problem_destroy": [_P],
    "sfb_problem_stream": [_P, C.POINTER(_P)],
    "sfb_set_poses": [_P, _P, _P, _P],
    "sfb_get_poses": [_P, _P, _P],
    "sfb_save_best": [_P],
    "sfb_restore_best": [_P],
    "sfb_build_dense_edges": [_P, _D, C.POINTER(_I64)],
    "sfb_get_dense_edges": [_P, _P],
    "sfb_set_dense_edges": [_P, _I64, _P],
    "sfb_frustum_overlap": [_P, _I64, _P, _P],
    "sfb_linearize": [_P, C.POINTER(Weights), _D, C.POINTER(Config), _P],
    "sfb_pcg": [_P, _I32, _D, _I32, C.POINTER(_I32), C.POINTER(_D), C.POINTER(_I32)],
    "sfb_get_solution": [_P, _P],
    "sfb_pcg_dense": [_P, _I32, _P, _P, _P, _I32, _D, _I32, _P, C.POINTER(_I32), C.POINTER(_D),
                      C.POINTER(_I32)],
    "sfb_apply_step": [_P, C.POINTER(_D)],
    "sfb_energy_frozen": [_P, _I32, _P],
    "sfb_gn_iteration": [_P, C.POINTER(Weights), _D, C.POINTER(Config), _I32, _D, _I32,
                         C.POINTER(IterResult)],
    "sfb_system_dims": [_P, C.POINTER(_I32), C.POINTER(_I64), C.POINTER(_I64)],
    "sfb_matvec": [_P, _P, _P],
    "sfb_get_gradient": [_P, _P],
    "sfb_get_diagonal": [_P, _P],
    "sfb_get_blocks": [_P, _P, _P, _P],
    "sfb_get_sparse_world": [_P, _P, _P],
    "sfb_sparse_residuals": [_P, _P],
    "sfb_sparse_set_max": [_P, _P],
    "sfb_associate": [_P, _I32, _I32, _I32, C.POINTER(Config), _P, _P],
    "sfb_point_eval": [_P, _I32, _I32, _I32, _I64, _P, _P, _P, _P, _P],
    "sfb_energy_and_linearize": [_P, C.POINTER(Weights), _I32, _D, C.POINTER(Config), _P],
    "sfb_set_shard": [_P, _I32, _I32],
    "sfb_set_preconditioner": [_P, _I32],
    "sfb_problem_drop_sets": [_P, _I64, _P],
    "sfb_set_shard_mode": [_P, _I32],
    "sfb_ipc_export": [_P, _I32, _P, C.POINTER(_I64)],
    "sfb_ipc_attach": [_P, _I32, _I32, _P],
    "sfb_set_p2p": [_P, _I32],
    "sfb_linearize_end_system": [_P],
    "sfb_linearize_finish": [_P, _P],
    "sfb_pcg_sharded": [_P, _I32, _D, _I32, ALLREDUCE_FN, _P, C.POINTER(_I32), C.POINTER(_D),
                        C.POINTER(_I32)],
    "sfb_exchange_buffer": [_P, _I32, C.POINTER(_P), C.POINTER(_I64)],
    "sfb_build_dense_edges_begin": [_P, _D],
    "sfb_build_dense_edges_end": [_P, C.POINTER(_I64)],
    "sfb_linearize_begin": [_P, C.POINTER(Weights), _D, C.POINTER(Config), C.POINTER(_I32)],
    "sfb_linearize_end": [_P, _P],
    "sfb_energy_and_linearize_begin": [_P, C.POINTER(Weights), _I32, _D, C.POINTER(Config),
                                       C.POINTER(_I32)],
    "sfb_energy_and_linearize_end": [_P, _P],
    "sfb_energy_frozen_begin": [_P, _I32, C.POINTER(_I32)],
    "sfb_energy_frozen_end": [_P, _P],
    "sfb_profile": [_P, _I32],
    "sfb_profile_read": [_P, _P, _P, _I32],
    "sfb_launch_count": [C.POINTER(_I64)],
    "sfb_frames_set_intensity": [_P, _I32, _P, _P],
    "sfb_host_alloc": [_I64, C.POINTER(_P)],
    "sfb_host_free": [_P],
    "sfb_gn_step_begin": [_P, _I32, _D, _I32, C.POINTER(Weights), _I32, _I32, _D,
                          C.POINTER(Config), C.POINTER(_I32)],
    "sfb_gn_step_end": [_P, _P],
    "sfb_tsdf_create": [_P, _D, _D, _I32, C.POINTER(_P)],
    "sfb_tsdf_destroy": [_P],
    "sfb_tsdf_apply": [_P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _I32, _P, _P, _I32, _P, _I32,
                       C.POINTER(_I32), _P],
    "sfb_tsdf_count": [_P, C.POINTER(_I64)],
    "sfb_tsdf_export": [_P, _I64, _P, _P, _P, _P],
    "sfb_tsdf_import": [_P, _I64, _P, _P, _P, _P],
    "sfb_tsdf_get_block": [_P, _P, C.POINTER(_I32), _P, _P, _P],
    "sfb_build_cache": [_P, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, _I32, _P, _P],
    "sfb_gn_step": [_P, _I32, _D, _I32, C.POINTER(Weights), _I32, _I32, _D, C.POINTER(Config),
                    _P],
    "sfb_dense_verify": [_P, _I32, _P, _P, _P, _P, _P, C.POINTER(VerifyConfig), _P, _P],
}

PROF_CLASSES = ("dense_linearize", "frozen_energy", "pcg", "pair_filter", "sparse_term",
                "assembly", "pose_update", "other")


def launch_count() -> int:
    n = C.c_int64()
    check(load().sfb_launch_count(C.byref(n)))
    return n.value

_lib = None
_lock = threading.Lock()


def load(path: os.PathLike | None = None) -> C.CDLL:
    """Load libsfb.so and declare every exported symbol; raises if missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else Path(os.environ.get("SFB_LIB", LIB_PATH))
        if not p.exists():
            raise ImportError(
                f"{p} is not built; run `python -m paper_1604_01093_b200._build` "
                "(the CUDA extension is required: there is no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = C.c_int
        lib.sfb_last_error.argtypes = [_P]
        lib.sfb_last_error.restype = C.c_char_p
        lib.sfb_abi_version.argtypes = []
        lib.sfb_abi_version.restype = C.c_int
        _lib = lib
        return lib


def check(rc: int, handle=None) -> None:
    if rc != SFB_OK:
        msg = load().sfb_last_error(handle)
        raise SfbError(rc, msg.decode() if msg else "")


def ptr(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)
