"""Seeded synthetic inputs for the benchmark configurations (BASELINE.json).

Config 1 (``config1_pair``): a single 1242x375 pair. The left image is seeded
fractal value noise, normalised to mean 128 / std 40. The right image is the
left image forward-splatted through a ground-truth disparity field (a ground
plane and 8 fronto-parallel boxes, disparity 0-127), with a z-buffer that
keeps the largest disparity. These are stand-ins for the paper's KITTI data,
which is not available here.

Configs 2-5 are ray-cast sequences (boxes and planes with value-noise
texture).  They come from the device renderer ``es_render_views`` in
``csrc/render.cu``; ``sequence_spec`` builds their scene and trajectory
parameters here.
"""

from __future__ import annotations

import numpy as np

__all__ = ["fbm_texture", "config1_pair", "box_scene", "sequence_spec"]


def fbm_texture(h: int, w: int, rng, octaves: int = 5, period: float = 24.0):
    """Fractal value noise (smoothstep-bilinear lattice, octaves halving
    amplitude and period), affinely normalised to mean 128 / std 40."""
    img = np.zeros((h, w))
    amp = 1.0
    for _ in range(octaves):
        gh, gw = int(h / period) + 3, int(w / period) + 3
        lat = rng.random((gh, gw))
        oy, ox = rng.random(2) * period
        fy = (np.arange(h) + oy) / period
        fx = (np.arange(w) + ox) / period
        iy, ix = np.floor(fy).astype(int), np.floor(fx).astype(int)
        ty, tx = fy - iy, fx - ix
        ty = ty * ty * (3 - 2 * ty)
        tx = tx * tx * (3 - 2 * tx)
        a = lat[iy][:, ix]
        b = lat[iy][:, ix + 1]
        c = lat[iy + 1][:, ix]
        d = lat[iy + 1][:, ix + 1]
        top = a + (b - a) * tx[None, :]
        bot = c + (d - c) * tx[None, :]
        img += amp * (top + (bot - top) * ty[:, None])
        amp *= 0.5
        period = max(period / 2.0, 1.5)
    img = (img - img.mean()) / max(img.std(), 1e-12) * 40.0 + 128.0
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def config1_pair(seed: int = 1000, width: int = 1242, height: int = 375,
                 d_max: int = 127, b: float = 0.54, cy: float = 185.0,
                 h_cam: float = 1.65, n_boxes: int = 8):
    """(left, right, gt_left) for config 1; gt is float64 with 0 = no data."""
    rng = np.random.default_rng(seed)
    left = fbm_texture(height, width, rng)
    ys = np.arange(height, dtype=np.float64)
    ground = np.where(ys > cy, b * (ys - cy) / h_cam, 0.0)
    gt = np.repeat(ground[:, None], width, axis=1)
    gt = np.maximum(gt, 1.0)
    for _ in range(n_boxes):
        bw = int(rng.integers(40, 260))
        bh = int(rng.integers(30, 160))
        x0 = int(rng.integers(0, width - bw))
        y0 = int(rng.integers(0, height - bh))
        disp = float(rng.uniform(2.0, d_max - 7.0))
        blk = gt[y0:y0 + bh, x0:x0 + bw]
        np.maximum(blk, disp, out=blk)
    gt = np.minimum(gt, float(d_max))
    # forward splat left -> right with a max-disparity z-buffer
    right = fbm_texture(height, width, np.random.default_rng(seed + 7919))
    zbuf = np.full((height, width), -1.0)
    yy, xx = np.mgrid[0:height, 0:width]
    tx = xx - np.rint(gt).astype(np.int64)
    ok = tx >= 0
    order = np.argsort(gt[ok], kind="stable")  # nearer surfaces written last
    sy, sx, st = yy[ok][order], xx[ok][order], tx[ok][order]
    right[sy, st] = left[sy, sx]
    zbuf[sy, st] = gt[sy, sx]
    return left, right, gt


def box_scene(rng, n_boxes: int = 8, z_range=(5.0, 60.0)):
    """Ground slab, n seeded boxes and a far wall (configs 2-5).

    Returns a float64 array (n, 6) of boxes (x0, x1, y0, y1, z0, z1); the far
    wall is a very thin box.  World frame: x right, y down, z forward."""
    boxes = [(-60.0, 60.0, 1.65, 1.8, 3.0, 90.0),      # ground slab
             (-400.0, 400.0, -200.0, 200.0, 95.0, 95.5)]  # far wall
    for _ in range(n_boxes):
        z0 = float(rng.uniform(*z_range))
        depth = float(rng.uniform(0.5, 3.0))
        wdt = float(rng.uniform(0.8, 4.0))
        hgt = float(rng.uniform(0.8, 3.0))
        side = 1.0 if rng.random() < 0.5 else -1.0   # keep the driving corridor clear
        xc = side * (2.5 + wdt / 2 + float(rng.uniform(0.0, 0.4)) * z0)
        boxes.append((xc - wdt / 2, xc + wdt / 2, 1.65 - hgt, 1.65, z0, z0 + depth))
    return np.asarray(boxes, np.float64)


def _rot(yaw, pitch, roll):
    cy, sy = np.cos(yaw), np.sin(yaw)
    cp, sp = np.cos(pitch), np.sin(pitch)
    cr, sr = np.cos(roll), np.sin(roll)
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rx = np.array([[1, 0, 0], [0, cp, -sp], [0, sp, cp]])
    Rz = np.array([[cr, -sr, 0], [sr, cr, 0], [0, 0, 1]])
    return Ry @ Rx @ Rz


def sequence_spec(seed: int, n_frames: int, step: float = 1.0,
                  step_sigma: float = 0.05, yaw_deg: float = 0.5,
                  tilt_deg: float = 0.1, n_boxes: int = 8, z_range=(5.0, 60.0)):
    """Scene boxes plus world-from-camera poses and relative motions
    (frame k-1 -> k, the reference's ``relative_motion``)."""
    rng = np.random.default_rng(seed)
    boxes = box_scene(rng, n_boxes, z_range)
    poses = []
    pos = np.zeros(3)
    yaw = pitch = roll = 0.0
    for k in range(n_frames):
        if k:
            yaw += np.deg2rad(rng.normal(0.0, yaw_deg))
            pitch = np.deg2rad(rng.normal(0.0, tilt_deg))
            roll = np.deg2rad(rng.normal(0.0, tilt_deg))
            R = _rot(yaw, pitch, roll)
            pos = pos + R @ np.array([0.0, 0.0, step + rng.normal(0.0, step_sigma)])
        T = np.eye(4)
        T[:3, :3] = _rot(yaw, pitch, roll)
        T[:3, 3] = pos
        poses.append(T)
    motions = [None] + [np.linalg.inv(poses[k]) @ poses[k - 1] for k in range(1, n_frames)]
    return boxes, poses, motions
