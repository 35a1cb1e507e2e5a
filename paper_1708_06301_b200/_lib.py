"""ctypes binding of the C ABI in ``include/egostereo_b200.h``.

The library is loaded lazily on first use and never replaced by a CPU path:
if ``libegostereo_b200.so`` is missing or no CUDA device is usable, calls
raise ``DeviceUnavailableError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceUnavailableError, DeviceUnsupportedError, PointAtInfinityError

HERE = os.path.dirname(os.path.abspath(__file__))
# ES_LIB_PATH: load an alternative build of the same library (A/B profiling)
LIB_PATH = os.environ.get("ES_LIB_PATH") or os.path.join(HERE, "libegostereo_b200.so")

ES_OK, ES_ERR_VALUE, ES_ERR_POINT_AT_INFINITY, ES_ERR_NONPOSITIVE_D = 0, 1, 2, 3
ES_ERR_CUDA, ES_ERR_UNSUPPORTED = 4, 5

# FrameResult map selectors (es_ctx_export)
(ES_PRED_D, ES_PRED_P, ES_PRED_VALID, ES_LO, ES_HI, ES_MEAS_D, ES_MEAS_VALID, ES_MEAS_R,
 ES_KEEP, ES_FUSED_D, ES_FUSED_P, ES_FUSED_VALID, ES_COST_DENSE, ES_TOTAL_DENSE,
 ES_FUSED_KITTI) = range(15)


class EsRig(ctypes.Structure):
    _fields_ = [("f", ctypes.c_double), ("b", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
                ("d_max", ctypes.c_int32)]


class EsParams(ctypes.Structure):
    _fields_ = [("window", ctypes.c_int32), ("p1", ctypes.c_double), ("p2", ctypes.c_double),
                ("s_max", ctypes.c_double), ("r_min", ctypes.c_double),
                ("tau_lr", ctypes.c_double), ("tau_sad", ctypes.c_double),
                ("q", ctypes.c_double), ("gamma_f", ctypes.c_double),
                ("gamma_e", ctypes.c_double), ("edge_window", ctypes.c_int32),
                ("edge_reject", ctypes.c_int32), ("fill_holes", ctypes.c_int32),
                ("p_init", ctypes.c_double), ("baseline", ctypes.c_int32)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_L = ctypes.c_int64

# symbol -> argtypes (every entry point declared in include/egostereo_b200.h)
SIGNATURES = {
    "es_last_error": [],
    "es_version": [],
    "es_device_count": [_P],
    "es_ctx_create": [_I, _P, _P, _I, _P],
    "es_ctx_destroy": [_P],
    "es_ctx_reset": [_P],
    "es_ctx_step": [_P, _P, _I, _P, _P, _I],
    "es_ctx_sync": [_P],
    "es_ctx_fence": [_P],
    "es_ctx_frame": [_P, _I, _P],
    "es_ctx_cells": [_P, _I, _P, _P],
    "es_ctx_have_state": [_P, _I, _P],
    "es_ctx_cells_acc": [_P, _P, _I],
    "es_ctx_profile": [_P, _I],
    "es_ctx_shared_batch": [_P, _I],
    "es_ctx_stage_times": [_P, _P, _P],
    "es_ctx_export": [_P, _I, _I, _I, _P],
    "es_ctx_export_all": [_P, _I, _I, _P, _I],
    "es_ctx_device_ptr": [_P, _I, _I, _I, _P],
    "es_ctx_stream": [_P, _P],
    "es_search_intervals": [_P, _P, _P, _I, _I, _I, _P, _P],
    "es_matching_cost": [_P, _P, _I, _I, _P, _P, _I, _I, _I, _P],
    "es_aggregate_paths": [_P, _I, _I, _I, _D, _D, _P],
    "es_select_disparity": [_P, _I, _I, _I, _P, _P],
    "es_matching_variance_map": [_P, _P, _P, _P, _I, _I, _I, _D, _D, _P],
    "es_lr_consistency": [_P, _P, _P, _P, _I, _I, _D, _P, _P],
    "es_sad_check": [_P, _P, _P, _P, _I, _I, _I, _D, _I, _P],
    "es_fuse_maps": [_P, _P, _P, _P, _P, _P, _I, _D, _P, _P, _P],
    "es_predict_view": [_P, _P, _P, _P, _P, _P, _P, _P, _P],
    "es_fill_zoom_holes": [_P, _P, _P, _I, _I, _D, _D, _P, _P, _P],
    "es_reject_edges": [_P, _P, _I, _I, _D, _I, _P],
    "es_warp_points": [_P, _P, _I, _P],
    "es_box_sum": [_P, _I, _I, _I, _P],
    "es_matching_variance_scalar": [_P, _I, _I, _D, _D, _P],
    "es_render": [_P, _P, _I, _P, _P, _I, _D, _I, _P, _P, _P],
    "es_render_prims": [_P, _P, _I, _P, _P, _I, _D, _I, _P, _P, _P],
    "es_bad_pixel_counts": [_P, _P, _P, _P, _L, _I, _I, _P, _P, _P],
    "es_ctx_metrics": [_P, _I, _P, _P, _L, _I, _P],
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load (once) and return the CDLL; raises if the library is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceUnavailableError(
                f"{path} is missing: build it with `python -m paper_1708_06301_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_char_p if name == "es_last_error" else ctypes.c_int
        _lib = lib
        return lib


def check(status: int) -> None:
    if status == ES_OK:
        return
    msg = load().es_last_error().decode(errors="replace")
    if status == ES_ERR_POINT_AT_INFINITY:
        raise PointAtInfinityError(msg)
    if status in (ES_ERR_VALUE, ES_ERR_NONPOSITIVE_D):
        raise ValueError(msg)
    if status == ES_ERR_UNSUPPORTED:
        raise DeviceUnsupportedError(msg)
    if status == ES_ERR_CUDA and "no CUDA-capable device" in msg:
        raise DeviceUnavailableError(msg)
    raise RuntimeError(f"egostereo_b200: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def ptr(a: np.ndarray):
    """Raw data pointer of a C-contiguous array."""
    assert a.flags["C_CONTIGUOUS"], "arrays passed to the C ABI must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def c_array(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def rig_struct(rig) -> EsRig:
    return EsRig(float(rig.f), float(rig.b), float(rig.cx), float(rig.cy), int(rig.width),
                 int(rig.height), int(rig.d_max))


def params_struct(sgm=None, prediction=None, fusion=None, baseline=False) -> EsParams:
    from .fusion import FusionParams
    from .prediction import PredictionParams
    from .sgm import SgmParams
    s = sgm or SgmParams()
    p = prediction or PredictionParams()
    f = fusion or FusionParams()
    return EsParams(int(s.window), float(s.p1), float(s.p2), float(s.s_max), float(s.r_min),
                    float(s.tau_lr), float(s.tau_sad), float(p.q), float(p.gamma_f),
                    float(p.gamma_e), int(p.edge_window), int(bool(p.edge_reject)),
                    int(bool(p.fill_holes)), float(f.p_init), int(bool(baseline)))
