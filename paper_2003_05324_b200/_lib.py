"""ctypes binding of libmixtile_b200.so (declared in include/mixtile_b200.h).

There is no fallback: if the shared library is missing or no CUDA device is
present, every compute entry point raises.  torch supplies device memory and
the current stream; the library only ever sees raw pointers.
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# MIXTILE_LIB: load a differently-built copy (A/B of compile-time kernel variants)
LIB_PATH = os.environ.get("MIXTILE_LIB") or os.path.join(HERE, "libmixtile_b200.so")

MT_OK, MT_E_NOT_SPD, MT_E_OVERFLOW, MT_E_BAD_ARG, MT_E_CUDA = 0, 1, 2, 3, 4
MODE_CODE = {"dp": 0, "mp": 1, "dst": 2}
METRIC_CODE = {"euclidean": 0, "great_circle": 1}


class MtTiles(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("nb", ctypes.c_int32),
        ("p", ctypes.c_int32),
        ("t", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("dp_pool", ctypes.c_void_p),
        ("sp_pool", ctypes.c_void_p),
        ("scratch", ctypes.c_void_p),
        ("status", ctypes.c_void_p),
        ("split", ctypes.c_void_p),
        ("col_stride", ctypes.c_int32),
        ("col_offset", ctypes.c_int32),
        ("dpanel", ctypes.c_void_p),
        ("row_stride", ctypes.c_int32),
        ("row_offset", ctypes.c_int32),
        ("panel_slots", ctypes.c_int32),
    ]


class MtMatern(ctypes.Structure):
    _fields_ = [
        ("variance", ctypes.c_double),
        ("spatial_range", ctypes.c_double),
        ("smoothness", ctypes.c_double),
        ("kind", ctypes.c_int32),
        ("nl", ctypes.c_int32),
        ("mu", ctypes.c_double),
        ("gam1", ctypes.c_double),
        ("gam2", ctypes.c_double),
        ("rp", ctypes.c_double),
        ("rm", ctypes.c_double),
        ("fact", ctypes.c_double),
        ("scale", ctypes.c_double),
    ]


_P = ctypes.POINTER
_V = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double

# name -> (restype, argtypes); the exported surface of include/mixtile_b200.h
SIGNATURES = {
    "mt_version": (_I32, []),
    "mt_last_error": (ctypes.c_char_p, []),
    "mt_dp_tiles": (_I64, [_I32, _I32, _I32]),
    "mt_sp_tiles": (_I64, [_I32, _I32, _I32]),
    "mt_scratch_tiles": (_I64, [_I32, _I32, _I32, _I32]),
    "mt_split_tiles": (_I64, [_I32, _I32, _I32]),
    "mt_work_doubles": (_I64, [_P(MtTiles)]),
    "mt_matern_prepare": (ctypes.c_int, [_D, _D, _D, _P(MtMatern)]),
    "mt_generate": (ctypes.c_int, [_P(MtTiles), _V, _I32, _D, _P(MtMatern), _V]),
    "mt_scan_duplicates": (ctypes.c_int, [_P(MtTiles), _V, _I32, _D, _V]),
    "mt_matern_array": (ctypes.c_int, [_V, _I64, _P(MtMatern), _V, _V]),
    "mt_cross_work_doubles": (_I64, [_I64, _I64]),
    "mt_cross_gemv": (ctypes.c_int, [_V, _I64, _V, _I64, _I32, _D, _P(MtMatern), _V, _V, _V, _V]),
    "mt_cholesky": (ctypes.c_int, [_P(MtTiles), _I32, _V]),
    "mt_cholesky_quad": (ctypes.c_int, [_P(MtTiles), _I32, _V, _V, _V, _V]),
    "mt_logdet": (ctypes.c_int, [_P(MtTiles), _V, _V, _V]),
    "mt_solve": (ctypes.c_int, [_P(MtTiles), _V, _I64, _I32, _V]),
    "mt_quad": (ctypes.c_int, [_P(MtTiles), _V, _V, _V, _V]),
    "mt_matvec_lower": (ctypes.c_int, [_P(MtTiles), _V, _V, _V]),
    "mt_evaluate": (ctypes.c_int, [_P(MtTiles), _V, _I32, _D, _P(MtMatern), _V, _V, _V, _I32, _V]),
    "mt_read_status": (ctypes.c_int, [_P(MtTiles), _P(_I64), _P(_I64), _P(_I64), _V]),
    "mt_reset_status": (ctypes.c_int, [_P(MtTiles), _V]),
    "mt_get_tile": (ctypes.c_int, [_P(MtTiles), _I32, _I32, _I32, _V, _V]),
    "mt_put_tile": (ctypes.c_int, [_P(MtTiles), _I32, _I32, _I32, _V, _V]),
    "mt_set_option": (_I32, [_I32, _I32]),
    "mt_panel": (ctypes.c_int, [_P(MtTiles), _I32, _V]),
    "mt_panel_factor": (ctypes.c_int, [_P(MtTiles), _I32, _V]),
    "mt_panel_solve": (ctypes.c_int, [_P(MtTiles), _I32, _V]),
    "mt_diag_regions": (ctypes.c_int, [_P(MtTiles), _I32, _P(_I64)]),
    "mt_update": (ctypes.c_int, [_P(MtTiles), _I32, _I32, _I32, _V]),
    "mt_update_ex": (ctypes.c_int, [_P(MtTiles), _I32, _I32, _I32, _I32, _V]),
    "mt_yield_request": (ctypes.c_int, [_I32, _V]),
    "mt_logdet_partials": (ctypes.c_int, [_P(MtTiles), _V, _V]),
    "mt_fwd_step": (ctypes.c_int, [_P(MtTiles), _I32, _V, _V]),
    "mt_fwd_step_ex": (ctypes.c_int, [_P(MtTiles), _I32, _I32, _V, _V]),
    "mt_tcf_stats": (ctypes.c_int, [_P(ctypes.c_double)]),
    "mt_sumsq": (ctypes.c_int, [_V, _I64, _V, _V, _V]),
    "mt_local_tiles": (ctypes.c_int, [_I32, _I32, _I32, _I32, _I32, _P(_I64), _P(_I64)]),
    "mt_dpanel_tiles": (_I64, [_I32, _I32, _I32]),
    "mt_local_tiles_ex": (ctypes.c_int, [_I32, _I32, _I32, _I32, _I32, _I32, _I32, _P(_I64),
                                         _P(_I64)]),
    "mt_dpanel_tiles_ex": (_I64, [_I32, _I32, _I32]),
    "mt_split_tiles_ex": (_I64, [_I32, _I32, _I32, _I32, _I32]),
    "mt_ring_pos": (_I32, [_I32, _I32, _I32, _I32]),
    "mt_ring_tiles": (ctypes.c_int, [_I32, _I32, _I32, _I32, _I32, _I32, _I32, _P(_I64), _P(_I64),
                                     _P(_I64)]),
    "mt_launch_count": (ctypes.c_longlong, []),
    "mt_prof_begin": (ctypes.c_int, [_I32]),
    "mt_prof_end": (ctypes.c_int, [_I32, _V, _V, _V, _V]),
    "mt_prof_sm_weighted": (ctypes.c_int, [_I32, _V]),
    "mt_peak_probe": (ctypes.c_int, [_I32, _I32, _P(_D)]),
    "mt_evaluate_host": (ctypes.c_int, [_I64, _I32, _I32, _I32, _V, _V, _I32, _D, _P(MtMatern),
                                        _V, _P(_I64)]),
}

_lib = None


def load():
    """Load the library (no CUDA device needed); raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2003_05324_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class MixtileCudaError(RuntimeError):
    pass


def check(rc, what=""):
    """Map a C status code onto the reference's exception types."""
    if rc == MT_OK:
        return
    msg = load().mt_last_error().decode(errors="replace")
    if rc == MT_E_BAD_ARG:
        raise ValueError(f"{what}: {msg}")
    raise MixtileCudaError(f"{what}: {msg} (code {rc})")


def matern_struct(variance, spatial_range, smoothness):
    th = MtMatern()
    check(load().mt_matern_prepare(float(variance), float(spatial_range), float(smoothness),
                                   ctypes.byref(th)), "mt_matern_prepare")
    return th


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2003_05324_b200 needs a CUDA device (no CPU fallback)")
    load()
    return torch


def stream_handle():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def np_ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


__all__ = ["load", "check", "MtTiles", "MtMatern", "matern_struct", "require_cuda",
           "stream_handle", "ptr", "np_ptr", "MODE_CODE", "METRIC_CODE", "MixtileCudaError",
           "SIGNATURES", "np"]
