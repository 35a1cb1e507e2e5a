"""Interval-restricted SGM: drop-in for the reference's ``egostereo.sgm``.

Every function keeps the reference signature and return types (host numpy
in, host numpy out) and runs on the B200 through the C ABI: search
intervals (sgm.py:105-127), windowed SAD cost (sgm.py:160-196), 8-path
aggregation (sgm.py:257-272), WTA (sgm.py:275-284), matching variance
(sgm.py:287-344), LR and SAD checks (sgm.py:347-396).  Dense volumes are the
interchange format at this boundary; on the device they live in the
row-ragged pair layout (see csrc/es_common.cuh).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DisparityMap, VarianceMap

__all__ = ["SgmParams", "IntervalMap", "CostVolume", "full_range_intervals",
           "search_intervals", "matching_cost", "aggregate_paths", "select_disparity",
           "matching_variance", "matching_variance_map", "lr_consistency", "sad_check",
           "_box_sum"]

_BORDER_INTENSITY_COST = 255
_VIEWS = {"left": 0, "right": 1}


@dataclass(frozen=True)
class SgmParams:
    """Matcher tunables (sgm.py:28-60)."""

    window: int = 3
    p1: float = 7.0
    p2: float = 86.0
    s_max: float = 10.0
    r_min: float = 0.25
    tau_lr: float = 1.0
    tau_sad: float = 200.0

    def __post_init__(self):
        if self.window < 3 or self.window % 2 == 0:
            raise ValueError(f"window must be odd and >= 3, got {self.window}")
        if not (0 < self.p1 <= self.p2):
            raise ValueError(f"penalties must satisfy 0 < P1 <= P2, got {self.p1}, {self.p2}")
        if self.s_max <= 0:
            raise ValueError(f"s_max must be positive, got {self.s_max}")
        if self.r_min <= 0:
            raise ValueError(f"r_min must be positive, got {self.r_min}")

    @property
    def border_cost(self) -> float:
        return float(self.window * self.window * _BORDER_INTENSITY_COST)


@dataclass(eq=False)
class IntervalMap:
    """Per-pixel inclusive interval [lo, hi] (sgm.py:63-84)."""

    lo: np.ndarray
    hi: np.ndarray
    d_max: int

    def __post_init__(self):
        self.lo = np.asarray(self.lo, dtype=np.int64)
        self.hi = np.asarray(self.hi, dtype=np.int64)
        if self.lo.shape != self.hi.shape:
            raise ValueError("lo/hi shape mismatch")
        if self.lo.min() < 0 or self.hi.max() > self.d_max or np.any(self.lo > self.hi):
            raise ValueError("intervals must satisfy 0 <= lo <= hi <= d_max")

    @property
    def shape(self) -> tuple[int, int]:
        return self.lo.shape

    def contains(self, d: int) -> np.ndarray:
        return (self.lo <= d) & (d <= self.hi)


@dataclass(eq=False)
class CostVolume:
    """Dense (H, W, d_max+1) float32 costs, +inf outside the interval."""

    data: np.ndarray
    intervals: IntervalMap


def _data(img):
    return img.data if hasattr(img, "data") else np.asarray(img)


def full_range_intervals(rig) -> IntervalMap:
    """sgm.py:95-102."""
    return IntervalMap(np.zeros(rig.shape, np.int64), np.full(rig.shape, rig.d_max, np.int64),
                       rig.d_max)


def search_intervals(d_pred, p_pred, rig) -> IntervalMap:
    """[floor(d - 3 sqrt p), ceil(d + 3 sqrt p)], clamped, widened to >= 2,
    full range where unpredicted (sgm.py:105-127) -- on the device."""
    d = _lib.c_array(d_pred.values, np.float64)
    p = _lib.c_array(p_pred.values, np.float64)
    v = _lib.c_array(d_pred.valid, np.uint8)
    h, w = d.shape
    lo = np.empty((h, w), np.int64)
    hi = np.empty((h, w), np.int64)
    _lib.call("es_search_intervals", _lib.ptr(d), _lib.ptr(p), _lib.ptr(v), h, w,
              int(rig.d_max), _lib.ptr(lo), _lib.ptr(hi))
    return IntervalMap(lo, hi, rig.d_max)


def matching_cost(left, right, intervals, params, view: str = "left") -> CostVolume:
    """Windowed SAD over each pixel's interval (sgm.py:160-196)."""
    L, R = _data(left), _data(right)
    if L.shape != R.shape:
        raise ValueError(f"image dimensions differ: {L.shape} vs {R.shape}")
    if view not in _VIEWS:
        raise ValueError(f"view must be 'left' or 'right', got {view!r}")
    L = _lib.c_array(L, np.uint8)
    R = _lib.c_array(R, np.uint8)
    lo = _lib.c_array(intervals.lo, np.int64)
    hi = _lib.c_array(intervals.hi, np.int64)
    h, w = L.shape
    d_max = int(intervals.d_max)
    out = np.empty((h, w, d_max + 1), np.float32)
    _lib.call("es_matching_cost", _lib.ptr(L), _lib.ptr(R), h, w, _lib.ptr(lo), _lib.ptr(hi),
              d_max, int(params.window), _VIEWS[view], _lib.ptr(out))
    return CostVolume(out, intervals)


def aggregate_paths(volume, params) -> CostVolume:
    """Sum of the eight SGM path recurrences (sgm.py:257-272)."""
    data = _lib.c_array(volume.data, np.float32)
    h, w, D = data.shape
    out = np.empty_like(data)
    _lib.call("es_aggregate_paths", _lib.ptr(data), h, w, D, ctypes.c_double(params.p1),
              ctypes.c_double(params.p2), _lib.ptr(out))
    return CostVolume(out, volume.intervals)


def select_disparity(aggregated) -> DisparityMap:
    """argmin over planes, ties to the smaller d; d* = 0 is invalid
    (sgm.py:275-284)."""
    data = _lib.c_array(aggregated.data, np.float32)
    h, w, D = data.shape
    d = np.empty((h, w), np.float64)
    v = np.empty((h, w), np.uint8)
    _lib.call("es_select_disparity", _lib.ptr(data), h, w, D, _lib.ptr(d), _lib.ptr(v))
    return DisparityMap(d, v.astype(bool))


def _box_sum(a, radius: int) -> np.ndarray:
    """Exact integer window sums with edge replication (sgm.py:130-136),
    on the device; int64 (H, W) like the reference."""
    a = np.ascontiguousarray(np.asarray(a).astype(np.int64))
    if a.ndim != 2:
        raise ValueError("_box_sum expects a 2-D array")
    out = np.empty_like(a)
    _lib.call("es_box_sum", _lib.ptr(a), a.shape[0], a.shape[1], int(radius), _lib.ptr(out))
    return out


def matching_variance_map(aggregated, disp, params) -> VarianceMap:
    """Outward cost-budget walk from the winner (sgm.py:319-344).  Like the
    reference (``disp.values.astype(np.int64)``, sgm.py:326) the winners are
    truncated toward zero, so fractional maps are accepted."""
    data = _lib.c_array(aggregated.data, np.float32)
    h, w, D = data.shape
    lo = _lib.c_array(aggregated.intervals.lo, np.int64)
    hi = _lib.c_array(aggregated.intervals.hi, np.int64)
    d = np.asarray(disp.values, dtype=np.float64).astype(np.int64).astype(np.float64)
    if d.size and (d.min() < 0 or d.max() >= D):
        raise IndexError(f"winners outside [0, {D}) for a volume of {D} planes")
    d = np.ascontiguousarray(d)
    r = np.empty((h, w), np.float64)
    _lib.call("es_matching_variance_map", _lib.ptr(data), _lib.ptr(lo), _lib.ptr(hi), _lib.ptr(d),
              h, w, D, ctypes.c_double(params.s_max), ctypes.c_double(params.r_min), _lib.ptr(r))
    return VarianceMap(r)


def matching_variance(costs, lo: int, d_star: int, params) -> float:
    """Scalar form over one pixel's interval costs (sgm.py:287-316): the
    float64 walk, one device thread."""
    costs = np.ascontiguousarray(np.asarray(costs, dtype=np.float64).ravel())
    center = d_star - lo
    if not 0 <= center < costs.size:
        raise ValueError(f"selected disparity {d_star} outside interval starting at {lo}")
    r = ctypes.c_double()
    _lib.call("es_matching_variance_scalar", _lib.ptr(costs), costs.size, int(center),
              ctypes.c_double(params.s_max), ctypes.c_double(params.r_min), ctypes.byref(r))
    return float(r.value)


def lr_consistency(d_left, d_right, tau_lr: float):
    """(keep_left, keep_right) cross-check (sgm.py:347-370)."""
    if d_left.shape != d_right.shape:
        raise ValueError("map dimensions differ")
    dl = _lib.c_array(d_left.values, np.float64)
    vl = _lib.c_array(d_left.valid, np.uint8)
    dr = _lib.c_array(d_right.values, np.float64)
    vr = _lib.c_array(d_right.valid, np.uint8)
    h, w = dl.shape
    kl = np.empty((h, w), np.uint8)
    kr = np.empty((h, w), np.uint8)
    _lib.call("es_lr_consistency", _lib.ptr(dl), _lib.ptr(vl), _lib.ptr(dr), _lib.ptr(vr), h, w,
              ctypes.c_double(tau_lr), _lib.ptr(kl), _lib.ptr(kr))
    return kl.astype(bool), kr.astype(bool)


def sad_check(left, right, disp, window: int, tau_sad: float, view: str = "left") -> np.ndarray:
    """Window SAD at rint(d) <= tau_sad with an on-image match centre
    (sgm.py:373-396)."""
    L = _lib.c_array(_data(left), np.uint8)
    R = _lib.c_array(_data(right), np.uint8)
    d = _lib.c_array(disp.values, np.float64)
    v = _lib.c_array(disp.valid, np.uint8)
    h, w = d.shape
    keep = np.empty((h, w), np.uint8)
    _lib.call("es_sad_check", _lib.ptr(L), _lib.ptr(R), _lib.ptr(d), _lib.ptr(v), h, w,
              int(window), ctypes.c_double(tau_sad), _VIEWS[view], _lib.ptr(keep))
    return keep.astype(bool)
