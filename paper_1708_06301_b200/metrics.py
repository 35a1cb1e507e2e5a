"""Disparity-map evaluation on the device: bad-pixel rates, bad mask, error
image, density, search-space size -- the reference's metrics module
(metrics.py:1-117) with the same names, dataclass and argument meaning.

The per-pixel test runs in ``es_metrics.cu`` (float64, the reference's
operation order) through ``es_bad_pixel_counts``; rates are formed on the
host from exact integer counts exactly as metrics.py:62-78 does.  There is
no CPU fallback: without the library or a GPU every call raises.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["ABS_THRESHOLD", "REL_THRESHOLD", "BadPixelResult", "bad_pixel_rate",
           "bad_pixel_mask", "density", "search_space_fraction", "error_image",
           "rates_from_counts"]

ABS_THRESHOLD = 3.0     # metrics.py:20
REL_THRESHOLD = 0.05    # metrics.py:21
_MODES = {"or": 0, "and": 1}


@dataclass(frozen=True)
class BadPixelResult:
    """Error rates of an estimate against ground truth (metrics.py:24-37).

    rate          bad fraction over pixels valid in both maps
    rate_all      bad fraction over all ground-truth pixels, counting
                  pixels the estimate missed as bad
    density       fraction of ground-truth pixels the estimate covers
    """

    rate: float
    rate_all: float
    density: float


def rates_from_counts(n_gt: int, n_both: int, n_bad: int) -> BadPixelResult:
    """metrics.py:62-78 on exact counts."""
    if n_gt == 0:
        return BadPixelResult(0.0, 0.0, 0.0)
    n_missing = n_gt - n_both
    rate = n_bad / n_both if n_both else 0.0
    return BadPixelResult(rate, (n_bad + n_missing) / n_gt, n_both / n_gt)


def _mode(mode: str) -> int:
    if mode not in _MODES:
        raise ValueError(f"mode must be 'or' or 'and', got {mode!r}")
    return _MODES[mode]


def _device_counts(estimate, truth, mode, mask=False, rgb=False):
    m = _mode(mode)
    if estimate.shape != truth.shape:
        raise ValueError("map dimensions differ")
    est = _lib.c_array(estimate.values, np.float64)
    ev = _lib.c_array(estimate.valid, np.uint8)
    gt = _lib.c_array(truth.values, np.float64)
    gv = _lib.c_array(truth.valid, np.uint8)
    n = est.size
    counts = np.zeros(4, dtype=np.uint64)
    mk = np.zeros(estimate.shape, dtype=np.uint8) if mask else None
    im = np.zeros(estimate.shape + (3,), dtype=np.uint8) if rgb else None
    _lib.call("es_bad_pixel_counts", _lib.ptr(est), _lib.ptr(ev), _lib.ptr(gt), _lib.ptr(gv),
              n, 1, m, _lib.ptr(counts), _lib.ptr(mk) if mask else None,
              _lib.ptr(im) if rgb else None)
    return counts, mk, im


def bad_pixel_rate(estimate, truth, mode: str = "or") -> BadPixelResult:
    """Fraction of pixels whose disparity error is beyond threshold
    (metrics.py:39-78).  mode="or": bad iff |err| > 3 px or > 5 % of the true
    disparity; mode="and": both (KITTI 2015).  Pixels invalid in the ground
    truth are ignored entirely."""
    counts, _, _ = _device_counts(estimate, truth, mode)
    return rates_from_counts(int(counts[0]), int(counts[1]), int(counts[2]))


def bad_pixel_mask(estimate, truth, mode: str = "or") -> np.ndarray:
    """Boolean mask of bad pixels over the jointly valid region
    (metrics.py:81-92)."""
    _, mk, _ = _device_counts(estimate, truth, mode, mask=True)
    return mk.astype(bool)


def density(estimate) -> float:
    """Valid fraction of the map (metrics.py:95-97)."""
    return float(np.asarray(estimate.valid).mean())


def search_space_fraction(intervals) -> float:
    """Searched cost-volume cells as a fraction of the full-range volume
    (metrics.py:100-104).  The frame step counts the cells on the device;
    this form serves host IntervalMaps."""
    widths = np.asarray(intervals.hi) - np.asarray(intervals.lo) + 1
    return float(widths.sum() / (np.asarray(intervals.lo).size * (intervals.d_max + 1)))


def error_image(estimate, truth, mode: str = "or") -> np.ndarray:
    """RGB visualization: blue = within threshold, red = bad, black = no data
    (metrics.py:106-117)."""
    _, _, im = _device_counts(estimate, truth, mode, rgb=True)
    return im
