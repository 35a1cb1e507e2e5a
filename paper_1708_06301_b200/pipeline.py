"""Per-frame engine: drop-in for ``egostereo.pipeline`` (pipeline.py:53-302).

``DisparityPipeline.process_frame`` (pipeline.py:108-170) runs the whole
frame on the B200 through one ``es_ctx_step`` call: warp + z-buffer + Kalman
predict, hole fill, intervals, ragged SAD cost, 8-path SGM, WTA + variance,
LR + SAD checks and the Kalman update.  The filter state stays resident in
HBM (double-buffered); ``FrameResult`` maps are copied to the host only when
read (``FrameResult`` materialises itself before the engine overwrites the
buffers it refers to).

``BatchedPipeline`` advances B independent sequences per call (config 5,
SURVEY 8(e)); multi-GPU runs shard sequences across processes.
"""

from __future__ import annotations

import ctypes
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import (DisparityMap, FilterState, StereoRig, VarianceMap, make_empty_state,
                   validate_rigid_motion)
from .fusion import FusionParams
from .geometry import disparity_homography, right_motion
from .prediction import PredictionParams
from .sgm import IntervalMap, SgmParams

__all__ = ["FrameResult", "PipelineParams", "DisparityPipeline", "BatchedPipeline",
           "StereoEngine"]


@dataclass
class PipelineParams:
    """pipeline.py:75-82."""

    sgm: SgmParams = field(default_factory=SgmParams)
    prediction: PredictionParams = field(default_factory=PredictionParams)
    fusion: FusionParams = field(default_factory=FusionParams)
    baseline: bool = False


_U8_MAPS = {_lib.ES_PRED_VALID, _lib.ES_MEAS_VALID, _lib.ES_KEEP, _lib.ES_FUSED_VALID}
_I64_MAPS = {_lib.ES_LO, _lib.ES_HI}


class StereoEngine:
    """Owner of one ``es_ctx``: B sequences of one rig on one device."""

    def __init__(self, rig, params: PipelineParams | None = None, batch: int = 1,
                 device: int = 0):
        self.rig = rig
        self.params = params or PipelineParams()
        self.batch = int(batch)
        self.device = int(device)
        self._rs = _lib.rig_struct(rig)
        p = self.params
        self._ps = _lib.params_struct(p.sgm, p.prediction, p.fusion, p.baseline)
        h = ctypes.c_void_p()
        _lib.call("es_ctx_create", self.device, ctypes.byref(self._rs), ctypes.byref(self._ps),
                  self.batch, ctypes.byref(h))
        self._h = h
        self.generation = 0
        self._Hm = np.zeros((self.batch, 2, 16), np.float64)
        self._given = np.zeros(self.batch, np.uint8)
        self._have_state = np.zeros(self.batch, bool)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().es_ctx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reset(self):
        _lib.call("es_ctx_reset", self._h)
        self._have_state[:] = False
        self.generation += 1

    def homographies(self, motions):
        """Host-side 4x4 builds (geometry.py:62-92) for sequences that will
        predict; the device receives 16 doubles per view."""
        self._given[:] = 0
        for s, T in enumerate(motions):
            if T is None or self.params.baseline or not self._have_state[s]:
                continue
            T = validate_rigid_motion(T)
            self._Hm[s, 0] = disparity_homography(self.rig, T).ravel()
            self._Hm[s, 1] = disparity_homography(self.rig, right_motion(self.rig, T)).ravel()
            self._given[s] = 1

    def step(self, images, motions, sync: bool = True, images_dev: int | None = None):
        """Advance every sequence one frame.  ``images`` is a host uint8
        array (B, 2, H, W) or, with ``images_dev``, a device pointer."""
        self.homographies(motions)
        if images_dev is None:
            img = _lib.c_array(images, np.uint8)
            if img.shape != (self.batch, 2, self.rig.height, self.rig.width):
                raise ValueError(f"images must be (B, 2, H, W), got {img.shape}")
            src, on_dev = _lib.ptr(img), 0
        else:
            src, on_dev = ctypes.c_void_p(images_dev), 1
        self.generation += 1
        _lib.call("es_ctx_step", self._h, src, on_dev, _lib.ptr(self._Hm), _lib.ptr(self._given),
                  1 if sync else 0)
        if sync:
            self._refresh_state_flags()
        else:
            self._have_state[:] = True

    def sync(self):
        _lib.call("es_ctx_sync", self._h)
        self._refresh_state_flags()

    def _refresh_state_flags(self):
        # have_state (pipeline.py:122): any valid pixel in either view, as
        # counted on the device by the Kalman-update step
        f = ctypes.c_int64()
        for s in range(self.batch):
            _lib.call("es_ctx_have_state", self._h, s, ctypes.byref(f))
            self._have_state[s] = bool(f.value)

    def export(self, what: int, seq: int = 0, view: int = 0) -> np.ndarray:
        h, w = self.rig.height, self.rig.width
        if what in (_lib.ES_COST_DENSE, _lib.ES_TOTAL_DENSE):
            out = np.empty((h, w, self.rig.d_max + 1), np.float32)
        elif what == _lib.ES_FUSED_KITTI:
            out = np.empty((h, w), np.uint16)
        elif what in _U8_MAPS:
            out = np.empty((h, w), np.uint8)
        elif what in _I64_MAPS:
            out = np.empty((h, w), np.int64)
        else:
            out = np.empty((h, w), np.float64)
        _lib.call("es_ctx_export", self._h, int(what), int(seq), int(view), _lib.ptr(out))
        return out.astype(bool) if what in _U8_MAPS else out

    def cells(self, seq: int = 0):
        l, r = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.call("es_ctx_cells", self._h, int(seq), ctypes.byref(l), ctypes.byref(r))
        return int(l.value), int(r.value)

    def frame(self, seq: int = 0) -> int:
        f = ctypes.c_int64()
        _lib.call("es_ctx_frame", self._h, int(seq), ctypes.byref(f))
        return int(f.value)

    def stream(self) -> int:
        s = ctypes.c_void_p()
        _lib.call("es_ctx_stream", self._h, ctypes.byref(s))
        return s.value or 0


# every map of one frame, as the device step left it: the engine, the
# sequence, the step generation and the maps already read back
_MAP_KEYS = ((_lib.ES_PRED_D, _lib.ES_PRED_VALID, _lib.ES_PRED_P, _lib.ES_LO, _lib.ES_HI,
              _lib.ES_MEAS_D, _lib.ES_MEAS_VALID, _lib.ES_MEAS_R, _lib.ES_KEEP, _lib.ES_FUSED_D,
              _lib.ES_FUSED_VALID, _lib.ES_FUSED_P))


class _FrameMaps:
    """Read-back cache of one frame's maps.  FrameResult and the lazy fused
    state share it (neither references the other, so dropping both frees it
    at once); the owning pipeline reads every map back before a later step
    would overwrite them, if anything still holds the cache."""

    def __init__(self, engine, seq):
        self.engine = engine
        self.seq = seq
        self.gen = engine.generation
        self.cache = {}

    def get(self, what, view):
        key = (what, view)
        if key not in self.cache:
            if self.engine.generation != self.gen:
                raise RuntimeError("FrameResult maps were overwritten by a later frame")
            self.cache[key] = self.engine.export(what, self.seq, view)
        return self.cache[key]

    def materialize(self):
        for what in _MAP_KEYS:
            for view in (0, 1):
                self.get(what, view)


class _LazyFilterState(FilterState):
    """A FilterState whose maps are exported from the device on first access
    (reading ``res.fused.left`` costs two device->host copies, not six)."""

    def __init__(self, maps, frame):
        object.__setattr__(self, "_maps", maps)
        object.__setattr__(self, "frame", frame)

    left = property(lambda s: DisparityMap(s._maps.get(_lib.ES_FUSED_D, 0),
                                           s._maps.get(_lib.ES_FUSED_VALID, 0)))
    left_var = property(lambda s: VarianceMap(s._maps.get(_lib.ES_FUSED_P, 0)))
    right = property(lambda s: DisparityMap(s._maps.get(_lib.ES_FUSED_D, 1),
                                            s._maps.get(_lib.ES_FUSED_VALID, 1)))
    right_var = property(lambda s: VarianceMap(s._maps.get(_lib.ES_FUSED_P, 1)))


class FrameResult:
    """Everything the pipeline derived for one frame (pipeline.py:53-72).

    Maps are read from the device on first access; the owning pipeline
    forces materialisation before its next step overwrites them."""

    def __init__(self, engine: StereoEngine, seq: int, frame: int):
        self._maps = _FrameMaps(engine, seq)
        self._engine = engine
        self.frame = frame
        self._fused = None
        l, r = engine.cells(seq)
        total = engine.rig.width * engine.rig.height * (engine.rig.d_max + 1)
        self.search_fraction_left = float(l / total)
        self.search_fraction_right = float(r / total)

    def _get(self, what, view):
        return self._maps.get(what, view)

    def materialize(self):
        self._maps.materialize()
        return self

    def _pred(self, v):
        return DisparityMap(self._get(_lib.ES_PRED_D, v), self._get(_lib.ES_PRED_VALID, v))

    def _meas(self, v):
        return DisparityMap(self._get(_lib.ES_MEAS_D, v), self._get(_lib.ES_MEAS_VALID, v))

    def _iv(self, v):
        return IntervalMap(self._get(_lib.ES_LO, v), self._get(_lib.ES_HI, v),
                           self._engine.rig.d_max)

    predicted_left = property(lambda s: s._pred(0))
    predicted_right = property(lambda s: s._pred(1))
    predicted_left_var = property(lambda s: VarianceMap(s._get(_lib.ES_PRED_P, 0)))
    predicted_right_var = property(lambda s: VarianceMap(s._get(_lib.ES_PRED_P, 1)))
    intervals_left = property(lambda s: s._iv(0))
    intervals_right = property(lambda s: s._iv(1))
    measured_left = property(lambda s: s._meas(0))
    measured_right = property(lambda s: s._meas(1))
    measured_left_var = property(lambda s: VarianceMap(s._get(_lib.ES_MEAS_R, 0)))
    measured_right_var = property(lambda s: VarianceMap(s._get(_lib.ES_MEAS_R, 1)))
    keep_left = property(lambda s: s._get(_lib.ES_KEEP, 0))
    keep_right = property(lambda s: s._get(_lib.ES_KEEP, 1))

    @property
    def fused(self) -> FilterState:
        """The posterior state (pipeline.py:64); its four maps are read from
        the device one by one, on first access."""
        if self._fused is None:
            self._fused = _LazyFilterState(self._maps, self.frame)
        return self._fused

    def cost_volume(self, view: int = 0) -> np.ndarray:
        """Dense export of the raw cost (parity / debugging)."""
        return self._get(_lib.ES_COST_DENSE, view)

    def total_volume(self, view: int = 0) -> np.ndarray:
        """Dense export of the aggregated cost (parity / debugging)."""
        return self._get(_lib.ES_TOTAL_DENSE, view)


class DisparityPipeline:
    """Stateful per-sequence engine (pipeline.py:90-170) on one B200."""

    def __init__(self, rig: StereoRig, params: PipelineParams | None = None, device: int = 0):
        self.rig = rig
        self.params = params or PipelineParams()
        self._engine = StereoEngine(rig, self.params, batch=1, device=device)
        self._last = None
        self._img = np.empty((1, 2, rig.height, rig.width), np.uint8)

    def reset(self) -> None:
        self._flush()
        self._engine.reset()

    @property
    def state(self) -> FilterState:
        f = self._engine.frame(0)
        if f < 0:
            return make_empty_state(self.rig, frame=-1)
        e = self._engine
        return FilterState(
            DisparityMap(e.export(_lib.ES_FUSED_D, 0, 0), e.export(_lib.ES_FUSED_VALID, 0, 0)),
            VarianceMap(e.export(_lib.ES_FUSED_P, 0, 0)),
            DisparityMap(e.export(_lib.ES_FUSED_D, 0, 1), e.export(_lib.ES_FUSED_VALID, 0, 1)),
            VarianceMap(e.export(_lib.ES_FUSED_P, 0, 1)), frame=f)

    def _flush(self):
        last = self._last() if self._last is not None else None
        if last is not None:
            last.materialize()
        self._last = None

    def process_frame(self, left, right, motion=None) -> FrameResult:
        """Advance the filter by one stereo pair (pipeline.py:108-170)."""
        L = left.data if hasattr(left, "data") else np.asarray(left)
        R = right.data if hasattr(right, "data") else np.asarray(right)
        if L.shape != self.rig.shape or R.shape != self.rig.shape:
            raise ValueError(f"image dimensions {L.shape}/{R.shape} != rig {self.rig.shape}")
        self._flush()
        self._img[0, 0] = L
        self._img[0, 1] = R
        self._engine.step(self._img, [motion], sync=True)
        res = FrameResult(self._engine, 0, self._engine.frame(0))
        self._last = weakref.ref(res._maps)
        return res


def default_groups(batch: int) -> int:
    """Device contexts a batch is split into (see BatchedPipeline): the
    divisor of the batch whose contexts come closest to 16 sequences, none
    below 12.  Measured on a B200 (frames/s, one context -> split): B = 24
    1262 -> 1539 (2 x 12), B = 32 1626 -> 1776 (2 x 16; 4 x 8: 1461), B = 48
    1460 -> 1915 (3 x 16; 2 x 24: 1896), B = 64 1715 -> 2005 (4 x 16; 2 x 32:
    1937; 8 x 8: 1550), B = 96 1958 (6 x 16; 3 x 32: 1925), B = 128 1967
    (8 x 16; 4 x 32: 1945)."""
    best, score = 1, abs(batch - 16)
    for g in range(2, batch // 12 + 1):
        if batch % g == 0 and abs(batch // g - 16) < score:
            best, score = g, abs(batch // g - 16)
    return best


class BatchedPipeline:
    """B independent sequences advanced together (config 5).

    From 24 sequences up the batch runs as ``groups`` device contexts of
    about 16 sequences each (``default_groups``), every context on its own
    streams: a step enqueues every group before any waits, so one group's
    latency-bound SGM aggregation (the fused sweeps hold one SM per view for
    ~9.5 ms) overlaps the other groups' bandwidth-bound stages and the
    groups' sweeps pack the SMs.  Each context is told the whole batch
    (``es_ctx_shared_batch``) so that its aggregation keeps the GPU-filling
    schedule.  Sequences are independent, so the results are
    those of one context."""

    def __init__(self, rig: StereoRig, batch: int, params: PipelineParams | None = None,
                 device: int = 0, groups: int | None = None):
        self.rig = rig
        self.batch = int(batch)
        self.params = params or PipelineParams()
        if groups is None:
            groups = default_groups(self.batch)
        if groups < 1 or self.batch % groups:
            raise ValueError(f"batch {batch} does not split into {groups} groups")
        self.groups = int(groups)
        self.per = self.batch // self.groups
        self.engines = [StereoEngine(rig, self.params, batch=self.per, device=device)
                        for _ in range(self.groups)]
        if self.groups > 1:
            for e in self.engines:
                _lib.call("es_ctx_shared_batch", e._h, self.batch)

    @property
    def engine(self) -> StereoEngine:
        """The context of a single-group pipeline."""
        if self.groups != 1:
            raise AttributeError("a grouped BatchedPipeline has one engine per group: use .engines")
        return self.engines[0]

    def reset(self):
        for e in self.engines:
            e.reset()

    def process_frames(self, images, motions, sync: bool = True, images_dev=None):
        """images: (B, 2, H, W) uint8 host array (or device pointer via
        ``images_dev``); motions: list of B 4x4 arrays or None."""
        if len(self.engines) == 1:
            self.engines[0].step(images, motions, sync=sync, images_dev=images_dev)
            return
        if images_dev is None:
            images = _lib.c_array(images, np.uint8)
            if images.shape != (self.batch, 2, self.rig.height, self.rig.width):
                raise ValueError(f"images must be (B, 2, H, W), got {images.shape}")
        motions = list(motions)
        if len(motions) != self.batch:
            raise ValueError(f"expected {self.batch} motions, got {len(motions)}")
        step_bytes = self.per * 2 * self.rig.height * self.rig.width
        for g, e in enumerate(self.engines):
            lo, hi = g * self.per, (g + 1) * self.per
            if images_dev is None:
                e.step(images[lo:hi], motions[lo:hi], sync=False)
            else:
                e.step(None, motions[lo:hi], sync=False, images_dev=int(images_dev) + g * step_bytes)
        if sync:
            self.sync()

    def sync(self):
        for e in self.engines:
            e.sync()

    def fence(self):
        """Order the engines' compute streams after every transfer issued so
        far (uploads and exports run on their own copy streams)."""
        for e in self.engines:
            _lib.call("es_ctx_fence", e._h)

    def fused_kitti(self, view: int = 0, out=None, sync: bool = True) -> np.ndarray:
        """Fused disparity of every sequence in the KITTI uint16 encoding
        (kitti_io.py:38-46), one batched device->host copy per group.  With
        ``sync=False`` the copies are only enqueued (``out`` should be pinned)."""
        h, w = self.rig.height, self.rig.width
        if out is None:
            out = np.empty((self.batch, h, w), np.uint16)
        for g, e in enumerate(self.engines):
            part = out[g * self.per:(g + 1) * self.per]
            _lib.call("es_ctx_export_all", e._h, _lib.ES_FUSED_KITTI, int(view),
                      _lib.ptr(part), 1 if sync else 0)
        return out

    def result(self, seq: int) -> FrameResult:
        if not 0 <= seq < self.batch:
            raise IndexError(f"sequence {seq} out of range for batch {self.batch}")
        e = self.engines[seq // self.per]
        s = seq % self.per
        return FrameResult(e, s, e.frame(s))

    def metrics(self, gt_dev: int, gt_valid_dev: int, gt_stride: int, view: int = 0,
                mode: str = "or"):
        """Per-sequence evaluation of the current fused maps against device
        ground truth (sequence s at ``gt_dev + s * gt_stride`` float64 values
        and ``gt_valid_dev + s * gt_stride`` uint8 flags): a list of
        (metrics.BadPixelResult, density) -- metrics.py:39-97 on the device,
        one 32-byte-per-sequence read back."""
        from . import metrics as M
        counts = np.zeros((self.batch, 4), np.uint64)
        for g, e in enumerate(self.engines):
            off = g * self.per * int(gt_stride)
            _lib.call("es_ctx_metrics", e._h, int(view), ctypes.c_void_p(int(gt_dev) + 8 * off),
                      ctypes.c_void_p(int(gt_valid_dev) + off), int(gt_stride), M._mode(mode),
                      _lib.ptr(counts[g * self.per:(g + 1) * self.per]))
        hw = self.rig.width * self.rig.height
        return [(M.rates_from_counts(int(c[0]), int(c[1]), int(c[2])), int(c[3]) / hw)
                for c in counts]
