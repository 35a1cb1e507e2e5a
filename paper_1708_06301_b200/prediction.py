"""Forward warping of the disparity belief: drop-in for ``egostereo.prediction``.

Edge rejection (prediction.py:50-64), the warp + deterministic z-buffer +
variance propagation (prediction.py:80-126) and zoom-hole filling
(prediction.py:148-183) run on the device; see csrc/es_predict.cu.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DisparityMap, FilterState, VarianceMap, validate_rigid_motion
from .geometry import disparity_homography, right_motion

__all__ = ["PredictionParams", "reject_edges", "propagate_variance", "predict_maps",
           "fill_zoom_holes"]


@dataclass(frozen=True)
class PredictionParams:
    """prediction.py:23-47."""

    q: float = 0.5
    gamma_f: float = 3.0
    gamma_e: float = 3.0
    edge_window: int = 1
    edge_reject: bool = True
    fill_holes: bool = True

    def __post_init__(self):
        if self.q < 0:
            raise ValueError(f"q must be >= 0, got {self.q}")
        if self.gamma_f <= 0 or self.gamma_e <= 0:
            raise ValueError("gamma_f and gamma_e must be positive")
        if self.edge_window < 1:
            raise ValueError(f"edge_window must be >= 1, got {self.edge_window}")


def reject_edges(disp, gamma_e: float, edge_window: int) -> np.ndarray:
    """Valid pixels whose valid-neighbourhood range exceeds gamma_e."""
    d = _lib.c_array(disp.values, np.float64)
    v = _lib.c_array(disp.valid, np.uint8)
    h, w = d.shape
    out = np.empty((h, w), np.uint8)
    _lib.call("es_reject_edges", _lib.ptr(d), _lib.ptr(v), h, w, ctypes.c_double(gamma_e),
              int(edge_window), _lib.ptr(out))
    return out.astype(bool)


def propagate_variance(d_prev, d_pred, p_prev, q: float):
    """(d_pred / d_prev)^2 p_prev + q (prediction.py:67-77).  Elementwise
    helper of the public API; the frame step evaluates it inside the device
    warp kernel."""
    d_prev = np.asarray(d_prev, dtype=np.float64)
    if np.any(d_prev <= 0):
        raise ValueError("previous disparity must be positive")
    ratio = np.asarray(d_pred, dtype=np.float64) / d_prev
    return ratio * ratio * np.asarray(p_prev, dtype=np.float64) + q


def _predict_view(disp, var, H, rig, params):
    """One view's forward splat (prediction.py:80-126) on the device."""
    from .sgm import SgmParams
    d = _lib.c_array(disp.values, np.float64)
    p = _lib.c_array(var.values, np.float64)
    v = _lib.c_array(disp.valid, np.uint8)
    Hc = _lib.c_array(H, np.float64)
    h, w = d.shape
    od = np.empty((h, w), np.float64)
    op = np.empty((h, w), np.float64)
    ov = np.empty((h, w), np.uint8)
    rs = _lib.rig_struct(rig)
    ps = _lib.params_struct(SgmParams(), params)
    _lib.call("es_predict_view", _lib.ptr(d), _lib.ptr(p), _lib.ptr(v), _lib.ptr(Hc),
              ctypes.byref(rs), ctypes.byref(ps), _lib.ptr(od), _lib.ptr(op), _lib.ptr(ov))
    return DisparityMap(od, ov.astype(bool)), VarianceMap(op)


def predict_maps(state, T, rig, params) -> FilterState:
    """Warp both views of the previous state (prediction.py:129-145)."""
    if state.shape != rig.shape:
        raise ValueError(f"state shape {state.shape} != rig shape {rig.shape}")
    T = validate_rigid_motion(T)
    H_left = disparity_homography(rig, T)
    H_right = disparity_homography(rig, right_motion(rig, T))
    ld, lp = _predict_view(state.left, state.left_var, H_left, rig, params)
    rd, rp = _predict_view(state.right, state.right_var, H_right, rig, params)
    return FilterState(ld, lp, rd, rp, frame=state.frame + 1)


def fill_zoom_holes(disp, var, gamma_f: float, q: float):
    """Single-gap interpolation, horizontal then vertical (prediction.py:169-183)."""
    d = _lib.c_array(disp.values, np.float64)
    p = _lib.c_array(var.values, np.float64)
    v = _lib.c_array(disp.valid, np.uint8)
    h, w = d.shape
    od = np.empty((h, w), np.float64)
    op = np.empty((h, w), np.float64)
    ov = np.empty((h, w), np.uint8)
    _lib.call("es_fill_zoom_holes", _lib.ptr(d), _lib.ptr(p), _lib.ptr(v), h, w,
              ctypes.c_double(gamma_f), ctypes.c_double(q), _lib.ptr(od), _lib.ptr(op),
              _lib.ptr(ov))
    return DisparityMap(od, ov.astype(bool)), VarianceMap(op)
