"""Disparity-space homographies (reference geometry.py).

The 4x4 builds (``gamma``, ``disparity_homography``, ``right_motion``) are
host-side kernel arguments and use the reference's exact
expression so H is bit-identical.  Per-pixel warping runs on the device
(``es_predict_view`` / the frame step); ``warp_point`` / ``warp_pixels`` are
thin wrappers over the device warp.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .core import make_motion, validate_rigid_motion
from .errors import BehindCameraError, PointAtInfinityError

__all__ = ["PointAtInfinityError", "BehindCameraError", "gamma", "gamma_inv",
           "disparity_homography", "baseline_offset", "right_motion", "warp_point",
           "euclidean_warp_oracle", "warp_pixels"]


def gamma(rig) -> np.ndarray:
    """geometry.py:36-46."""
    f, fb = rig.f, rig.f * rig.b
    return np.array([[f, 0.0, 0.0, 0.0], [0.0, f, 0.0, 0.0], [0.0, 0.0, 0.0, fb],
                     [0.0, 0.0, 1.0, 0.0]])


def gamma_inv(rig) -> np.ndarray:
    """geometry.py:49-59 (closed form)."""
    f, fb = rig.f, rig.f * rig.b
    return np.array([[1.0 / f, 0.0, 0.0, 0.0], [0.0, 1.0 / f, 0.0, 0.0],
                     [0.0, 0.0, 0.0, 1.0], [0.0, 0.0, 1.0 / fb, 0.0]])


def disparity_homography(rig, T) -> np.ndarray:
    """H = Gamma T Gamma^-1; exact identity for T == I (geometry.py:62-75)."""
    T = validate_rigid_motion(T)
    if np.array_equal(T, np.eye(4)):
        return np.eye(4)
    H = gamma(rig) @ T @ gamma_inv(rig)
    if abs(np.linalg.det(H)) <= 1e-12:
        raise RuntimeError("disparity homography is singular; rig is corrupt")
    return H


def baseline_offset(rig) -> np.ndarray:
    return make_motion(t=(rig.b, 0.0, 0.0))


def right_motion(rig, T) -> np.ndarray:
    """B^-1 T B (geometry.py:83-92)."""
    B = make_motion(t=(rig.b, 0.0, 0.0))
    B_inv = make_motion(t=(-rig.b, 0.0, 0.0))
    return B_inv @ T @ B


def warp_point(H, w) -> np.ndarray:
    """Apply H to principal-point-relative (x, y, d) points on the device
    (geometry.py:95-115); raises PointAtInfinityError."""
    w = np.asarray(w, dtype=np.float64)
    single = w.ndim == 1
    pts = np.ascontiguousarray(np.atleast_2d(w).reshape(-1, 3))
    out = np.empty_like(pts)
    Hc = _lib.c_array(H, np.float64)
    _lib.call("es_warp_points", _lib.ptr(Hc), _lib.ptr(pts), ctypes.c_int(pts.shape[0]),
              _lib.ptr(out))
    out = out.reshape(np.atleast_2d(w).shape)
    return out[0] if single else out


def warp_pixels(rig, H, xs, ys, ds):
    """geometry.py:147-159."""
    xs = np.asarray(xs, dtype=np.float64)
    ys = np.asarray(ys, dtype=np.float64)
    ds = np.asarray(ds, dtype=np.float64)
    out = warp_point(H, np.stack([xs - rig.cx, ys - rig.cy, ds], axis=-1))
    return out[..., 0] + rig.cx, out[..., 1] + rig.cy, out[..., 2]


def euclidean_warp_oracle(rig, T, w) -> np.ndarray:
    """Triangulate, move, reproject (geometry.py:118-144).  A cross-check of
    warp_point kept for API completeness; not used by the device path."""
    T = validate_rigid_motion(T)
    w = np.asarray(w, dtype=np.float64)
    single = w.ndim == 1
    pts = np.atleast_2d(w)
    x, y, d = pts[..., 0], pts[..., 1], pts[..., 2]
    if np.any(d <= 0):
        raise ValueError("disparity must be positive to triangulate")
    Z = rig.fb / d
    M = np.stack([x * Z / rig.f, y * Z / rig.f, Z, np.ones_like(Z)], axis=-1)
    Mp = M @ T.T
    Zp = Mp[..., 2]
    if np.any(Zp <= 0):
        raise BehindCameraError("transformed point has nonpositive depth")
    res = np.stack([rig.f * Mp[..., 0] / Zp, rig.f * Mp[..., 1] / Zp, rig.fb / Zp], axis=-1)
    return res[0] if single else res
