"""Per-pixel Kalman update: drop-in for ``egostereo.fusion`` (fusion.py:19-79).
``fuse_maps`` runs on the device; the scalar helpers are the reference's
elementwise formulas."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DisparityMap, VarianceMap

__all__ = ["FusionParams", "kalman_gain", "fuse_pixel", "fuse_maps"]


@dataclass(frozen=True)
class FusionParams:
    p_init: float = 1.0

    def __post_init__(self):
        if self.p_init <= 0:
            raise ValueError(f"p_init must be positive, got {self.p_init}")


def kalman_gain(p, r):
    return np.asarray(p, dtype=np.float64) / (np.asarray(p) + np.asarray(r))


def fuse_pixel(d_pred: float, p_pred: float, d_meas: float, r_meas: float):
    k = p_pred / (p_pred + r_meas)
    return d_pred + k * (d_meas - d_pred), (1.0 - k) * p_pred


def fuse_maps(d_pred, p_pred, d_meas, r_meas, params):
    """Both valid -> blend; measurement only -> adopt at p_init; otherwise
    invalid (fusion.py:45-79)."""
    if d_pred.shape != d_meas.shape:
        raise ValueError("map dimensions differ")
    dp = _lib.c_array(d_pred.values, np.float64)
    pp = _lib.c_array(p_pred.values, np.float64)
    vp = _lib.c_array(d_pred.valid, np.uint8)
    dm = _lib.c_array(d_meas.values, np.float64)
    rm = _lib.c_array(r_meas.values, np.float64)
    vm = _lib.c_array(d_meas.valid, np.uint8)
    n = dp.size
    od = np.empty(dp.shape, np.float64)
    op = np.empty(dp.shape, np.float64)
    ov = np.empty(dp.shape, np.uint8)
    _lib.call("es_fuse_maps", _lib.ptr(dp), _lib.ptr(pp), _lib.ptr(vp), _lib.ptr(dm), _lib.ptr(rm),
              _lib.ptr(vm), n, ctypes.c_double(params.p_init), _lib.ptr(od), _lib.ptr(op),
              _lib.ptr(ov))
    return DisparityMap(od, ov.astype(bool)), VarianceMap(op)
