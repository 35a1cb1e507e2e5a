"""numpy restatement of the egostereo hot path (TEST INFRASTRUCTURE ONLY).

See ``oracle/__init__.py`` for the rules.  All maps are row-major (H, W)
numpy arrays; "views" are ``"left"`` / ``"right"``.  Reference citations are
relative to ``/root/reference/pkg/src/egostereo/``.

The code deliberately does not mirror the reference's structure: costs are
gathered by clamped indexing (not integral images), every aggregation path is
reduced to a single top-to-bottom sweep by transposing / flipping the volume,
and the SAD check gathers per pixel instead of looping over unique winners.
The arithmetic (dtype, operation order, rounding mode) follows the reference
exactly so results are bit-identical.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "OracleParams",
    "bad_mask",
    "bad_rate",
    "error_rgb",
    "border_cost",
    "full_intervals",
    "predicted_intervals",
    "sad_volume",
    "sgm_paths",
    "sgm_total",
    "wta",
    "variance_counts",
    "lr_masks",
    "sad_masks",
    "kalman_fuse",
    "edge_mask",
    "homography",
    "right_view_motion",
    "warp_view",
    "fill_holes",
    "OracleStereo",
    "PATH_ORDER",
    "render_boxes",
]


class OracleParams:
    """Defaults of sgm.py:40-46, prediction.py:34-39, fusion.py:23."""

    def __init__(self, **kw):
        self.window = 3
        self.p1 = 7.0
        self.p2 = 86.0
        self.s_max = 10.0
        self.r_min = 0.25
        self.tau_lr = 1.0
        self.tau_sad = 200.0
        self.q = 0.5
        self.gamma_f = 3.0
        self.gamma_e = 3.0
        self.edge_window = 1
        self.edge_reject = True
        self.fill_holes = True
        self.p_init = 1.0
        self.baseline = False
        for k, v in kw.items():
            if not hasattr(self, k):
                raise KeyError(k)
            setattr(self, k, v)


def border_cost(window: int) -> float:
    """sgm.py:25,58-60: saturating cost of an off-image match centre."""
    return float(window * window * 255)


# --------------------------------------------------------------------------
# search intervals (sgm.py:95-127)
# --------------------------------------------------------------------------

def full_intervals(h: int, w: int, d_max: int):
    """sgm.py:95-102."""
    return np.zeros((h, w), np.int64), np.full((h, w), d_max, np.int64)


def predicted_intervals(d, p, valid, d_max: int):
    """sgm.py:105-127: [floor(d-3s), ceil(d+3s)] clipped, widened to >= 2."""
    spread = 3.0 * np.sqrt(np.maximum(p, 0.0))
    with np.errstate(invalid="ignore"):
        lo = np.clip(np.floor(d - spread).astype(np.int64), 0, d_max)
        hi = np.clip(np.ceil(d + spread).astype(np.int64), 0, d_max)
    for _ in range(2):
        lo = lo - (((hi - lo) < 2) & (lo > 0)).astype(np.int64)
        hi = hi + (((hi - lo) < 2) & (hi < d_max)).astype(np.int64)
    lo = np.where(valid, lo, 0)
    hi = np.where(valid, hi, d_max)
    return lo, hi


# --------------------------------------------------------------------------
# windowed SAD cost (sgm.py:130-196; tests/reference_sgm.py:24-47)
# --------------------------------------------------------------------------

def _clamped_window_sum(img, radius):
    """Sum over a (2r+1)^2 window with edge replication (sgm.py:130-136)."""
    h, w = img.shape
    rows = np.clip(np.arange(h)[:, None] + np.arange(-radius, radius + 1), 0, h - 1)
    cols = np.clip(np.arange(w)[:, None] + np.arange(-radius, radius + 1), 0, w - 1)
    vert = img[rows].sum(axis=1)              # (h, w)
    return vert[:, cols].sum(axis=2)          # (h, w)


def _match_columns(w: int, d: int, view: str):
    """Column of the other image matched by each reference column, and the
    off-image mask (sgm.py:139-157)."""
    xs = np.arange(w)
    tgt = xs - d if view == "left" else xs + d
    return np.clip(tgt, 0, w - 1), (tgt < 0) | (tgt > w - 1)


def sad_volume(left, right, lo, hi, d_max: int, window: int = 3, view: str = "left"):
    """Dense (H, W, d_max+1) float32 cost volume, +inf outside [lo, hi]
    (sgm.py:160-196)."""
    ref = (left if view == "left" else right).astype(np.int32)
    oth = (right if view == "left" else left).astype(np.int32)
    h, w = ref.shape
    vol = np.full((h, w, d_max + 1), np.inf, np.float32)
    bc = np.float32(border_cost(window))
    for d in range(int(lo.min()), int(hi.max()) + 1):
        inside = (lo <= d) & (d <= hi)
        if not inside.any():
            continue
        cols, off = _match_columns(w, d, view)
        diff = np.abs(ref - oth[:, cols])
        sad = _clamped_window_sum(diff, window // 2).astype(np.float32)
        sad[:, off] = bc
        vol[..., d][inside] = sad[inside]
    return vol


# --------------------------------------------------------------------------
# SGM aggregation (sgm.py:199-272)
# --------------------------------------------------------------------------

# (dx, dy) of the eight paths, in the reference's summation order
# (sgm.py:266-270): H->, H<-, then dy=+1 with dx=-1,0,1, then dy=-1 with
# dx=-1,0,1.  The predecessor of pixel (x, y) on path (dx, dy) is
# (x - dx, y - dy).
PATH_ORDER = [(1, 0), (-1, 0), (-1, 1), (0, 1), (1, 1), (-1, -1), (0, -1), (1, -1)]


def _recurrence(prev, cost, p1, p2):
    """One SGM step over a line of pixels (sgm.py:199-209), float32."""
    m = prev.min(axis=-1, keepdims=True)
    best = np.minimum(prev, m + p2)
    best[..., 1:] = np.minimum(best[..., 1:], prev[..., :-1] + p1)
    best[..., :-1] = np.minimum(best[..., :-1], prev[..., 1:] + p1)
    return cost + (best - m)


def _sweep_down(vol, shift, p1, p2):
    """Rows top to bottom; the predecessor of column x is column x - shift
    of the previous row; pixels without one restart at their raw cost."""
    out = np.empty_like(vol)
    out[0] = vol[0]
    for i in range(1, vol.shape[0]):
        if shift == 0:
            out[i] = _recurrence(out[i - 1], vol[i], p1, p2)
        elif shift > 0:
            out[i, :shift] = vol[i, :shift]
            out[i, shift:] = _recurrence(out[i - 1, :-shift], vol[i, shift:], p1, p2)
        else:
            out[i, shift:] = vol[i, shift:]
            out[i, :shift] = _recurrence(out[i - 1, -shift:], vol[i, :shift], p1, p2)
    return out


def sgm_paths(cost, dx: int, dy: int, p1: float, p2: float):
    """Path volume L_r for direction (dx, dy) (sgm.py:212-254)."""
    p1, p2 = np.float32(p1), np.float32(p2)
    if dy == 0:  # horizontal path == vertical sweep of the transposed volume
        return sgm_paths(cost.transpose(1, 0, 2), 0, dx, p1, p2).transpose(1, 0, 2)
    if dy > 0:
        return _sweep_down(cost, dx, p1, p2)
    return _sweep_down(cost[::-1], dx, p1, p2)[::-1]


def sgm_total(cost, p1: float, p2: float):
    """Sum of the eight paths in reference order; +inf where cost is +inf
    (sgm.py:257-272)."""
    cost = np.asarray(cost, np.float32)
    total = np.zeros_like(cost)
    for dx, dy in PATH_ORDER:
        total += sgm_paths(cost, dx, dy, p1, p2)
    total[~np.isfinite(cost)] = np.inf
    return total


# --------------------------------------------------------------------------
# WTA, matching variance (sgm.py:275-344)
# --------------------------------------------------------------------------

def wta(total):
    """argmin with first-index ties; winner 0 is invalid (sgm.py:275-284)."""
    win = np.argmin(total, axis=2)
    return win.astype(np.float64), win > 0


def variance_counts(total, lo, hi, winners, s_max: float, r_min: float):
    """Outward walk from the winner counting neighbours while the cumulative
    cost excess stays strictly below s_max (sgm.py:287-344); returns r."""
    h, w, D = total.shape
    ds = winners.astype(np.int64)
    c0 = np.take_along_axis(total, ds[..., None], 2)[..., 0]
    count = np.zeros((h, w), np.int64)
    for step, bound in ((-1, lo), (1, hi)):
        acc = np.zeros((h, w), np.float64)
        live = np.ones((h, w), bool)
        k = 1
        while k < D and live.any():
            j = ds + step * k
            live &= (j >= bound) if step < 0 else (j <= bound)
            c = np.take_along_axis(total, np.clip(j, 0, D - 1)[..., None], 2)[..., 0]
            with np.errstate(invalid="ignore"):
                acc = np.where(live, acc + (c - c0), acc)
            live = live & (acc < s_max)
            count += live
            k += 1
    return np.maximum(count.astype(np.float64), r_min)


# --------------------------------------------------------------------------
# consistency checks (sgm.py:347-396)
# --------------------------------------------------------------------------

def lr_masks(dl, vl, dr, vr, tau_lr: float):
    """sgm.py:347-370."""
    h, w = dl.shape
    xs = np.arange(w)[None, :]
    ys = np.arange(h)[:, None]

    def one(ds, vs, dd, vd, sign):
        partner = xs + sign * np.rint(ds).astype(np.int64)
        inb = (partner >= 0) & (partner < w)
        pc = np.clip(partner, 0, w - 1)
        return vs & inb & vd[ys, pc] & (np.abs(ds - dd[ys, pc]) <= tau_lr)

    return one(dl, vl, dr, vr, -1), one(dr, vr, dl, vl, 1)


def sad_masks(left, right, d, valid, window: int, tau_sad: float, view: str):
    """sgm.py:373-396: valid, on-image match centre, window SAD <= tau."""
    ref = (left if view == "left" else right).astype(np.int64)
    oth = (right if view == "left" else left).astype(np.int64)
    h, w = ref.shape
    r = window // 2
    di = np.where(valid, np.rint(d), 0).astype(np.int64)
    sign = -1 if view == "left" else 1
    ys = np.arange(h)[:, None]
    xs = np.arange(w)[None, :]
    sad = np.zeros((h, w), np.int64)
    for oy in range(-r, r + 1):
        yy = np.clip(ys + oy, 0, h - 1)
        for ox in range(-r, r + 1):
            xx = np.clip(xs + ox, 0, w - 1)
            xm = np.clip(xx + sign * di, 0, w - 1)
            sad += np.abs(ref[yy, xx] - oth[yy, xm])
    centre = xs + sign * di
    on = (centre >= 0) & (centre <= w - 1)
    return valid & on & (sad <= tau_sad)


# --------------------------------------------------------------------------
# Kalman update (fusion.py:45-79)
# --------------------------------------------------------------------------

def kalman_fuse(dp, pp, vp, dm, rm, vm, p_init: float):
    """Both valid -> blend; measurement only -> adopt at p_init; else drop."""
    both = vp & vm
    adopt = vm & ~vp
    with np.errstate(invalid="ignore", divide="ignore"):
        k = np.where(both, pp / (pp + rm), 0.0)
    d = np.where(both, dp + k * (dm - dp), 0.0)
    p = np.where(both, (1.0 - k) * pp, 0.0)
    d = np.where(adopt, dm, d)
    p = np.where(adopt, p_init, p)
    valid = both | adopt
    return np.where(valid, d, 0.0), np.where(valid, p, 0.0), valid


# --------------------------------------------------------------------------
# prediction (geometry.py:36-159, prediction.py:50-183)
# --------------------------------------------------------------------------

def homography(f: float, b: float, T):
    """geometry.py:36-75: H = Gamma T Gamma^-1, exact I for T == I."""
    T = np.asarray(T, np.float64)
    if np.array_equal(T, np.eye(4)):
        return np.eye(4)
    fb = f * b
    G = np.array([[f, 0, 0, 0], [0, f, 0, 0], [0, 0, 0, fb], [0, 0, 1, 0]], np.float64)
    Gi = np.array(
        [[1.0 / f, 0, 0, 0], [0, 1.0 / f, 0, 0], [0, 0, 0, 1.0], [0, 0, 1.0 / fb, 0]],
        np.float64,
    )
    H = G @ T @ Gi
    if abs(np.linalg.det(H)) <= 1e-12:
        raise RuntimeError("singular disparity homography")
    return H


def right_view_motion(b: float, T):
    """geometry.py:83-92: B^-1 T B with B = translation (b, 0, 0)."""
    B = np.eye(4)
    B[0, 3] = b
    Bi = np.eye(4)
    Bi[0, 3] = -b
    return Bi @ np.asarray(T, np.float64) @ B


def edge_mask(d, valid, gamma_e: float, radius: int):
    """prediction.py:50-64: valid pixels whose valid-neighbour range exceeds
    gamma_e; off-image neighbours are ignored."""
    h, w = d.shape
    hi_src = np.pad(np.where(valid, d, -np.inf), radius, constant_values=-np.inf)
    lo_src = np.pad(np.where(valid, d, np.inf), radius, constant_values=np.inf)
    hi = np.full((h, w), -np.inf)
    lo = np.full((h, w), np.inf)
    k = 2 * radius + 1
    for oy in range(k):
        for ox in range(k):
            hi = np.maximum(hi, hi_src[oy:oy + h, ox:ox + w])
            lo = np.minimum(lo, lo_src[oy:oy + h, ox:ox + w])
    with np.errstate(invalid="ignore"):
        return valid & ((hi - lo) > gamma_e)


def _warp(H, x, y, d, cx, cy):
    """geometry.py:95-115,147-159 with an explicit k = 0..3 dot product
    (the reference uses BLAS; see DESIGN.md on last-ulp parity)."""
    px = x - cx
    py = y - cy
    o = [((H[r, 0] * px + H[r, 1] * py) + H[r, 2] * d) + H[r, 3] for r in range(4)]
    w4 = o[3]
    if np.any(np.abs(w4) < 1e-12):
        raise ValueError("warped point has ~zero fourth homogeneous component")
    return o[0] / w4 + cx, o[1] / w4 + cy, o[2] / w4


def warp_view(d, p, valid, H, cx, cy, d_max, q, gamma_e, edge_window, edge_reject=True):
    """prediction.py:80-126 + 67-77: forward splat with a max-d z-buffer,
    ties to the smallest row-major source index."""
    h, w = d.shape
    src = valid.copy()
    if edge_reject:
        src &= ~edge_mask(d, valid, gamma_e, edge_window)
    od = np.zeros((h, w))
    op = np.zeros((h, w))
    ov = np.zeros((h, w), bool)
    if not src.any():
        return od, op, ov
    sy, sx = np.nonzero(src)
    ds = d[sy, sx]
    ps = p[sy, sx]
    xp, yp, dp = _warp(H, sx.astype(np.float64), sy.astype(np.float64), ds, cx, cy)
    tx = np.rint(xp).astype(np.int64)
    ty = np.rint(yp).astype(np.int64)
    ok = (tx >= 0) & (tx < w) & (ty >= 0) & (ty < h) & (dp > 0) & (dp <= d_max)
    if not ok.any():
        return od, op, ov
    if np.any(ds[ok] <= 0):
        raise ValueError("previous disparity must be positive")
    ratio = dp[ok] / ds[ok]
    pn = ratio * ratio * ps[ok] + q
    tgt = ty[ok] * w + tx[ok]
    sidx = sy[ok] * w + sx[ok]
    dn = dp[ok]
    # winner per target: largest d', then smallest source index
    order = np.argsort(sidx, kind="stable")
    order = order[np.argsort(-dn[order], kind="stable")]
    order = order[np.argsort(tgt[order], kind="stable")]
    tgt, dn, pn = tgt[order], dn[order], pn[order]
    head = np.ones(tgt.size, bool)
    head[1:] = tgt[1:] != tgt[:-1]
    od.flat[tgt[head]] = dn[head]
    op.flat[tgt[head]] = pn[head]
    ov.flat[tgt[head]] = True
    return od, op, ov


def _fill_pass(d, p, v, gamma_f, q, axis):
    """prediction.py:148-166: simultaneous single-gap fill along one axis."""
    def nb(a, s, fill):
        out = np.full_like(a, fill)
        if axis == 1:
            if s > 0:
                out[:, 1:] = a[:, :-1]
            else:
                out[:, :-1] = a[:, 1:]
        else:
            if s > 0:
                out[1:] = a[:-1]
            else:
                out[:-1] = a[1:]
        return out

    da, db = nb(d, 1, 0.0), nb(d, -1, 0.0)
    pa, pb = nb(p, 1, 0.0), nb(p, -1, 0.0)
    va, vb = nb(v, 1, False), nb(v, -1, False)
    fill = ~v & va & vb & (np.abs(da - db) < gamma_f)
    return (np.where(fill, 0.5 * (da + db), d),
            np.where(fill, np.maximum(pa, pb) + q, p),
            v | fill)


def fill_holes(d, p, v, gamma_f: float, q: float):
    """prediction.py:169-183: horizontal pass, then vertical on the result."""
    d, p, v = _fill_pass(d, p, v, gamma_f, q, axis=1)
    d, p, v = _fill_pass(d, p, v, gamma_f, q, axis=0)
    return np.where(v, d, 0.0), p, v


# --------------------------------------------------------------------------
# evaluation metrics (metrics.py:39-103)
# --------------------------------------------------------------------------

ABS_THRESHOLD = 3.0      # metrics.py:20
REL_THRESHOLD = 0.05     # metrics.py:21


def bad_mask(est_d, est_v, gt_d, gt_v, mode: str = "or"):
    """metrics.py:81-92: bad over the jointly valid region; "or" flags
    |err| > 3 px OR > 5 % of the true disparity, "and" requires both."""
    err = np.abs(est_d - gt_d)
    over_abs = err > ABS_THRESHOLD
    over_rel = err > REL_THRESHOLD * gt_d
    bad = (over_abs | over_rel) if mode == "or" else (over_abs & over_rel)
    return bad & est_v & gt_v


def bad_rate(est_d, est_v, gt_d, gt_v, mode: str = "or"):
    """metrics.py:39-78: (rate over jointly valid, rate counting missed
    ground-truth pixels as bad, ground-truth coverage)."""
    n_gt = int(gt_v.sum())
    if n_gt == 0:
        return 0.0, 0.0, 0.0
    both = gt_v & est_v
    n_both = int(both.sum())
    n_bad = int(bad_mask(est_d, est_v, gt_d, gt_v, mode).sum())
    rate = n_bad / n_both if n_both else 0.0
    return rate, (n_bad + n_gt - n_both) / n_gt, n_both / n_gt


def error_rgb(est_d, est_v, gt_d, gt_v, mode: str = "or"):
    """metrics.py:106-117: blue within threshold, red bad, black no data."""
    img = np.zeros(est_d.shape + (3,), dtype=np.uint8)
    both = est_v & gt_v
    bad = bad_mask(est_d, est_v, gt_d, gt_v, mode)
    img[both & ~bad] = (40, 90, 220)
    img[bad] = (220, 50, 40)
    return img


# --------------------------------------------------------------------------
# the frame step (pipeline.py:90-170)
# --------------------------------------------------------------------------

class OracleStereo:
    """Stateful per-sequence oracle of DisparityPipeline (pipeline.py:90-170).

    ``step`` returns a dict of every intermediate the GPU path is compared
    against (both views)."""

    def __init__(self, f, b, cx, cy, width, height, d_max, params=None):
        self.f, self.b, self.cx, self.cy = f, b, cx, cy
        self.w, self.h, self.d_max = width, height, d_max
        self.prm = params or OracleParams()
        self.reset()

    def reset(self):
        z = np.zeros((self.h, self.w))
        zb = np.zeros((self.h, self.w), bool)
        self.state = {v: (z.copy(), z.copy(), zb.copy()) for v in ("left", "right")}
        self.frame = -1

    def step(self, left, right, motion=None, keep_volumes=False):
        P = self.prm
        h, w, D = self.h, self.w, self.d_max
        have = any(self.state[v][2].any() for v in ("left", "right"))
        out = {"frame": self.frame + 1}
        if motion is not None and have and not P.baseline:
            Hs = {"left": homography(self.f, self.b, motion),
                  "right": homography(self.f, self.b, right_view_motion(self.b, motion))}
            for v in ("left", "right"):
                d, p, ok = self.state[v]
                pd, pp, pv = warp_view(d, p, ok, Hs[v], self.cx, self.cy, D, P.q,
                                       P.gamma_e, P.edge_window, P.edge_reject)
                if P.fill_holes:
                    pd, pp, pv = fill_holes(pd, pp, pv, P.gamma_f, P.q)
                lo, hi = predicted_intervals(pd, pp, pv, D)
                out[v + "_pred"] = (pd, pp, pv)
                out[v + "_iv"] = (lo, hi)
        else:
            for v in ("left", "right"):
                out[v + "_pred"] = (np.zeros((h, w)), np.zeros((h, w)), np.zeros((h, w), bool))
                out[v + "_iv"] = full_intervals(h, w, D)
        for v in ("left", "right"):
            lo, hi = out[v + "_iv"]
            cost = sad_volume(left, right, lo, hi, D, P.window, v)
            total = sgm_total(cost, P.p1, P.p2)
            dm, vm = wta(total)
            r = variance_counts(total, lo, hi, dm, P.s_max, P.r_min)
            out[v + "_meas"] = (dm, r, vm)
            if keep_volumes:
                out[v + "_cost"] = cost
                out[v + "_total"] = total
        dl, rl, vl = out["left_meas"]
        dr, rr, vr = out["right_meas"]
        kl, kr = lr_masks(dl, vl, dr, vr, P.tau_lr)
        kl &= sad_masks(left, right, dl, vl, P.window, P.tau_sad, "left")
        kr &= sad_masks(left, right, dr, vr, P.window, P.tau_sad, "right")
        out["left_keep"], out["right_keep"] = kl, kr
        for v, keep in (("left", kl), ("right", kr)):
            dm, r, vm = out[v + "_meas"]
            km = vm & keep
            pd, pp, pv = out[v + "_pred"]
            fd, fp, fv = kalman_fuse(pd, pp, pv, np.where(km, dm, 0.0), r, km, P.p_init)
            self.state[v] = (fd, fp, fv)
            out[v + "_fused"] = (fd, fp, fv)
            lo, hi = out[v + "_iv"]
            out[v + "_fraction"] = float((hi - lo + 1).sum() / (lo.size * (D + 1)))
        self.frame += 1
        return out


# --------------------------------------------------------------- renderer
# synth.py:87-218 restated for axis-aligned boxes (the bench scenes): only
# the bench's port-fallback CPU arm (no reference installed) uses it, to
# build its inputs; pinned against synth.render_frame's own output in
# tests/test_oracle_golden.py::test_render_boxes_matches_reference_synth.

def _lattice(ix, iy, iz, seed):
    """synth.py:87-103 (uint64 splitmix-style finaliser)."""
    u = np.uint64
    with np.errstate(over="ignore"):
        h = ix.astype(np.int64).view(u) * u(0x9E3779B97F4A7C15)
        h ^= iy.astype(np.int64).view(u) * u(0xC2B2AE3D27D4EB4F)
        h ^= iz.astype(np.int64).view(u) * u(0x165667B19E3779F9)
        h ^= u(seed & 0xFFFFFFFFFFFFFFFF) * u(0x27D4EB2F165667C5)
        for sh, mul in ((30, 0xBF58476D1CE4E5B9), (27, 0x94D049BB133111EB)):
            h ^= h >> u(sh)
            h *= u(mul)
        h ^= h >> u(31)
    return (h >> u(11)).astype(np.float64) / float(1 << 53)


def _noise(q, seed):
    """synth.py:106-120: trilinear value noise, corners summed in order."""
    base = np.floor(q)
    fr = q - base
    fr = fr * fr * (3.0 - 2.0 * fr)
    bi = base.astype(np.int64)
    acc = np.zeros(q.shape[:-1])
    for c in range(8):
        o = [(c >> k) & 1 for k in range(3)]
        w = [fr[..., k] if o[k] else 1.0 - fr[..., k] for k in range(3)]
        acc += _lattice(bi[..., 0] + o[0], bi[..., 1] + o[1], bi[..., 2] + o[2], seed) * w[0] * w[1] * w[2]
    return acc


def render_boxes(cs, k):
    """(2, H, W) uint8 images of frame k of a scenes.ConfigSequence
    (synth.render_frame, synth.py:195-218, for Box primitives)."""
    r = cs.rig
    h, w, f = r["height"], r["width"], r["f"]
    pose = np.asarray(cs.poses[k], np.float64)
    R, c0 = pose[:3, :3], pose[:3, 3]
    ys, xs = np.mgrid[0:h, 0:w]
    dc = np.stack([(xs - r["cx"]) / f, (ys - r["cy"]) / f, np.ones((h, w))], axis=-1)
    dirs = dc @ R.T                      # BLAS, as synth.py:175
    out = []
    for c in (c0, c0 + R @ np.array([r["b"], 0.0, 0.0])):
        tb = np.full((h, w), np.inf)
        with np.errstate(divide="ignore", invalid="ignore"):
            for bx in cs.boxes[k]:
                tn, tf = np.full((h, w), -np.inf), np.full((h, w), np.inf)
                for ax in range(3):
                    d = dirs[..., ax]
                    inv = np.where(d != 0.0, 1.0 / d, np.inf)
                    t1, t2 = (bx[2 * ax] - c[ax]) * inv, (bx[2 * ax + 1] - c[ax]) * inv
                    inside = (c[ax] >= bx[2 * ax]) & (c[ax] <= bx[2 * ax + 1])
                    lo = np.where(d == 0.0, -np.inf if inside else np.inf, np.minimum(t1, t2))
                    hi = np.where(d == 0.0, np.inf if inside else -np.inf, np.maximum(t1, t2))
                    tn, tf = np.maximum(tn, lo), np.minimum(tf, hi)
                tb = np.minimum(tb, np.where((tn <= tf) & (tn > 1e-6), tn, np.inf))
        hit = np.isfinite(tb)
        pts = c + np.where(hit, tb, 0.0)[..., None] * dirs
        q = pts / cs.texture_scale
        v = 0.65 * _noise(q, cs.texture_seed) + 0.35 * _noise(2.0 * q, cs.texture_seed + 1)
        tex = 20.0 + 215.0 * np.clip(v, 0.0, 1.0)
        out.append(np.clip(np.rint(np.where(hit, tex, float(cs.background))), 0, 255).astype(np.uint8))
    return np.stack(out)
