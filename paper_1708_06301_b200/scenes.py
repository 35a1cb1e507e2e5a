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

__all__ = ["fbm_texture", "config1_pair", "box_scene", "sequence_spec", "CONFIG_RIGS",
           "ConfigSequence", "config_sequence", "apply_salt", "TEXTURE_SCALE", "BACKGROUND"]


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


def box_scene(rng, n_boxes: int = 8, z_range=(5.0, 60.0), ground_z1: float = 90.0,
              wall_z: float = 95.0):
    """Ground slab, n seeded boxes and a far wall (configs 2-5).

    Returns a float64 array (n, 6) of boxes (x0, x1, y0, y1, z0, z1); the far
    wall is a very thin box.  World frame: x right, y down, z forward."""
    boxes = [(-60.0, 60.0, 1.65, 1.8, 3.0, ground_z1),      # ground slab
             (-400.0, 400.0, -200.0, 200.0, wall_z, wall_z + 0.5)]  # far wall
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
                  tilt_deg: float = 0.1, n_boxes: int = 8, z_range=(5.0, 60.0),
                  ground_z1: float = 90.0, wall_z: float = 95.0):
    """Scene boxes plus world-from-camera poses and relative motions
    (frame k-1 -> k, the reference's ``relative_motion``)."""
    rng = np.random.default_rng(seed)
    boxes = box_scene(rng, n_boxes, z_range, ground_z1, wall_z)
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


# ----------------------------------------------------------------------------
# BASELINE.json configs 2-5 as concrete seeded sequences.  One definition
# serves the bench (config 5, and config 4 via --config 4), the full-size
# parity tests and the golden generator (oracle/make_golden_configs.py), which
# renders the same scenes with the reference's own synth.render_frame: the
# device renderer is bit-exact with it, so every consumer sees identical bytes.

TEXTURE_SCALE = 0.05   # world lattice (m): paper-like ~50% search fractions
BACKGROUND = 12
TEXTURE_SEED0 = 17     # texture seed of sequence s = TEXTURE_SEED0 + s

_RIG_S = dict(f=718.9, b=0.54, cx=607.0, cy=185.0, width=1242, height=375, d_max=127)
CONFIG_RIGS = {
    2: _RIG_S, 3: _RIG_S, 5: _RIG_S,
    4: dict(f=1400.0, b=0.3, cx=1023.5, cy=511.5, width=2048, height=1024, d_max=255),
}
# scene seed of sequence s = seed0 + s
CONFIG_SEQS = {
    2: dict(frames=10, step=1.0, yaw_deg=0.5, seed0=2000),
    # 100 frames at 1 m/frame: the static scene extends to 160 m (boxes), 250 m
    # (ground) and 260 m (wall) so the camera never drives out of it; three
    # extra boxes move on their own (forward 0.3-1.5 m/frame, lateral drift),
    # violating the ego-motion prediction; 2% salt noise per view and frame.
    3: dict(frames=100, step=1.0, yaw_deg=0.5, seed0=3000, z_range=(5.0, 160.0),
            ground_z1=250.0, wall_z=260.0, movers=3, salt=0.02),
    4: dict(frames=30, step=1.5, yaw_deg=1.0, seed0=4000),
    5: dict(frames=50, step=1.0, yaw_deg=0.5, seed0=1000),
}


class ConfigSequence:
    """One seeded sequence of a BASELINE config: ``boxes[k]`` (n, 6) per
    frame, world-from-camera ``poses[k]``, relative ``motions[k]`` (None for
    frame 0), texture seed, salt-noise rate and seed."""

    def __init__(self, config, seq, rig, boxes, poses, motions, texture_seed, salt, salt_seed):
        self.config, self.seq, self.rig = config, seq, rig
        self.boxes, self.poses, self.motions = boxes, poses, motions
        self.texture_seed = texture_seed
        self.texture_scale = TEXTURE_SCALE
        self.background = BACKGROUND
        self.salt, self.salt_seed = salt, salt_seed

    @property
    def n_frames(self):
        return len(self.poses)


def config_sequence(config: int, seq: int = 0, n_frames: int | None = None) -> ConfigSequence:
    c = CONFIG_SEQS[config]
    n = c["frames"] if n_frames is None else n_frames
    kw = {k: c[k] for k in ("z_range", "ground_z1", "wall_z") if k in c}
    boxes, poses, motions = sequence_spec(seed=c["seed0"] + seq, n_frames=n, step=c["step"],
                                          yaw_deg=c["yaw_deg"], **kw)
    per_frame = [boxes] * n
    movers = c.get("movers", 0)
    if movers:
        rng = np.random.default_rng(c["seed0"] + seq + 7777)
        start = []
        for _ in range(movers):
            z0 = float(rng.uniform(8.0, 40.0))
            wdt, hgt, dep = (float(rng.uniform(0.8, 2.5)), float(rng.uniform(0.8, 2.0)),
                             float(rng.uniform(0.5, 2.0)))
            xc = float(rng.uniform(-4.0, 4.0))
            start.append((xc - wdt / 2, xc + wdt / 2, 1.65 - hgt, 1.65, z0, z0 + dep))
        start = np.asarray(start, np.float64)
        vel = np.stack([rng.uniform(-0.08, 0.08, movers), np.zeros(movers),
                        rng.uniform(0.3, 1.5, movers)], axis=1)
        per_frame = []
        for k in range(n):
            mv = start.copy()
            mv[:, 0:2] += (vel[:, 0] * k)[:, None]
            mv[:, 4:6] += (vel[:, 2] * k)[:, None]
            per_frame.append(np.concatenate([boxes, mv]))
    return ConfigSequence(config, seq, CONFIG_RIGS[config], per_frame, poses, motions,
                          TEXTURE_SEED0 + seq, c.get("salt", 0.0), c["seed0"] + seq + 31337)


def apply_salt(pair: np.ndarray, cs: ConfigSequence, frame: int) -> np.ndarray:
    """Salt noise of config 3: each pixel of each view independently set to
    255 with probability ``cs.salt`` (seeded per sequence and frame).
    Modifies and returns ``pair`` (2, H, W) uint8."""
    if cs.salt > 0.0:
        rng = np.random.default_rng([cs.salt_seed, frame])
        for v in range(2):
            pair[v][rng.random(pair[v].shape) < cs.salt] = 255
    return pair
