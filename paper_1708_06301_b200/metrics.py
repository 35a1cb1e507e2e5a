"""Per-frame statistics used by the engine (reference metrics.py:81-90).
Evaluation metrics (bad-pixel rates, error images) are out of scope (SURVEY §2
row 7)."""

from __future__ import annotations

import numpy as np

__all__ = ["density", "search_space_fraction"]


def density(estimate) -> float:
    """Valid fraction of a host map (metrics.py:81-83)."""
    return float(np.asarray(estimate.valid).mean())


def search_space_fraction(intervals) -> float:
    """Searched cells / full-range cells (metrics.py:86-90).  The frame step
    counts the cells on the device; this form serves host IntervalMaps."""
    widths = np.asarray(intervals.hi) - np.asarray(intervals.lo) + 1
    return float(widths.sum() / (np.asarray(intervals.lo).size * (intervals.d_max + 1)))
