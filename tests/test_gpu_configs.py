"""Parity on scaled-down versions of BASELINE.json configs 3 and 4, against
the CPU oracle (itself pinned to the reference by tests/golden):

* config 4 shape class: D = 256 (d_max = 255, two-register u16 chunks, the
  wide-interval kernels) on a 640x160 rig, 3 frames, forward motion;
* config 3 features: independently moving boxes (per-frame scene), 2% salt
  noise per view, long-ish horizon (6 frames) so fallback windows, LR
  rejection and the Kalman adopt/drop rule all occur.

Inputs come from the device renderer; the oracle sees the same bytes."""

import ctypes

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _render(rig, boxes_per_frame, poses, seed, scale):
    import torch
    from paper_1708_06301_b200 import _lib
    rs = _lib.rig_struct(rig)
    out = []
    for boxes, pose in zip(boxes_per_frame, poses):
        b = np.ascontiguousarray(boxes[None], np.float64)
        p = np.ascontiguousarray(pose[None], np.float64)
        s = np.array([seed], np.int64)
        img = torch.empty((1, 2, rig.height, rig.width), dtype=torch.uint8, device="cuda")
        _lib.call("es_render", ctypes.byref(rs), _lib.ptr(b), b.shape[1], _lib.ptr(p), _lib.ptr(s),
                  1, ctypes.c_double(scale), 12, ctypes.c_void_p(img.data_ptr()), None,
                  ctypes.c_void_p(0))
        out.append(img.cpu().numpy()[0])
    return out


def _compare(rig, frames, motions, params=None):
    from paper_1708_06301_b200 import core, pipeline
    pipe = pipeline.DisparityPipeline(rig, params)
    orc = O.OracleStereo(rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max)
    fractions = []
    for k, (img, motion) in enumerate(zip(frames, motions)):
        res = pipe.process_frame(core.GrayImage(img[0]), core.GrayImage(img[1]), motion)
        want = orc.step(img[0], img[1], motion)
        for view, name in ((0, "left"), (1, "right")):
            iv = res.intervals_left if view == 0 else res.intervals_right
            assert np.array_equal(iv.lo, want[name + "_iv"][0]), (k, name)
            assert np.array_equal(iv.hi, want[name + "_iv"][1]), (k, name)
            meas = res.measured_left if view == 0 else res.measured_right
            var = res.measured_left_var if view == 0 else res.measured_right_var
            assert np.array_equal(meas.values, want[name + "_meas"][0]), (k, name, "wta")
            assert np.array_equal(var.values, want[name + "_meas"][1]), (k, name, "r")
            keep = res.keep_left if view == 0 else res.keep_right
            assert np.array_equal(keep, want[name + "_keep"]), (k, name, "keep")
            fd = res.fused.left if view == 0 else res.fused.right
            fp = res.fused.left_var if view == 0 else res.fused.right_var
            assert np.array_equal(fd.valid, want[name + "_fused"][2]), (k, name)
            np.testing.assert_allclose(fd.values, want[name + "_fused"][0], rtol=1e-9, atol=0)
            np.testing.assert_allclose(fp.values, want[name + "_fused"][1], rtol=1e-9, atol=0)
        fractions.append(res.search_fraction_left)
        np.testing.assert_allclose(res.search_fraction_left, want["left_fraction"], rtol=1e-15)
    return fractions


@pytest.mark.slow
def test_config4_class_d256():
    from paper_1708_06301_b200 import core, scenes
    rig = core.StereoRig(f=450.0, b=0.3, cx=319.5, cy=79.5, width=640, height=160, d_max=255)
    boxes, poses, motions = scenes.sequence_spec(seed=404, n_frames=3, step=0.4,
                                                 yaw_deg=1.0, z_range=(0.9, 8.0))
    frames = _render(rig, [boxes] * 3, poses, seed=3, scale=0.02)
    fr = _compare(rig, frames, motions)
    assert fr[0] == 1.0 and fr[-1] < 1.0


def test_config3_class_moving_boxes_and_salt_noise():
    from paper_1708_06301_b200 import core, scenes
    rig = core.StereoRig(f=180.0, b=0.54, cx=151.0, cy=46.0, width=310, height=94, d_max=40)
    n = 6
    boxes, poses, motions = scenes.sequence_spec(seed=303, n_frames=n, step=0.5,
                                                 z_range=(4.0, 30.0))
    rng = np.random.default_rng(33)
    movers = [2, 3, 4]   # three boxes move independently of the ego-motion
    vel = rng.uniform(-0.3, 0.3, (len(movers), 3)) * np.array([1.0, 0.0, 1.0])
    per_frame = []
    for k in range(n):
        b = boxes.copy()
        for i, bi in enumerate(movers):
            b[bi, 0:2] += vel[i, 0] * k
            b[bi, 4:6] += vel[i, 2] * k
        per_frame.append(b)
    frames = _render(rig, per_frame, poses, seed=5, scale=0.05)
    for img in frames:   # 2% salt noise, independent per view
        for v in range(2):
            mask = rng.random(img[v].shape) < 0.02
            img[v][mask] = 255
    fr = _compare(rig, frames, motions)
    assert fr[0] == 1.0 and min(fr[1:]) < 1.0


@pytest.mark.slow
def test_config2_full_size_sequence():
    """BASELINE config 2 at its full size (1242x375, D = 128, f = 718.9,
    b = 0.54, 1 m/frame with yaw/pitch/roll noise): the bench's device-rendered
    scene, frame 0 full range then predicted frames, bit-exact vs the oracle."""
    import bench
    from paper_1708_06301_b200 import core
    rig = core.StereoRig(**bench.RIG)
    specs = bench.sequence_specs(1, seed0=2000)
    imgs = bench.render_frames(specs, [0, 1, 2], "cuda:0").cpu().numpy()
    frames = [imgs[k, 0] for k in range(3)]
    fr = _compare(rig, frames, bench.motions_for_frames(specs, 0, 3))
    assert fr[0] == 1.0 and fr[2] < 1.0


@pytest.mark.slow
def test_config4_full_size_batched_equals_single():
    """BASELINE config 4 at its full size (2048x1024, D = 256): two sequences
    in one batched context give exactly the maps each gives alone (the
    batched launch geometry, the D = 256 kernels and the partial sums are
    per-(sequence, view) independent)."""
    import bench
    from paper_1708_06301_b200 import core, pipeline
    bench.use_config(4)
    try:
        rig = core.StereoRig(**bench.RIG)
        specs = bench.sequence_specs(2, seed0=4000)
        imgs = bench.render_frames(specs, [0, 1, 2], "cuda:0")
        bp = pipeline.BatchedPipeline(rig, 2)
        singles = [pipeline.DisparityPipeline(rig) for _ in range(2)]
        host = imgs.cpu().numpy()
        for k in range(3):
            bp.process_frames(None, bench.motions_for(specs, k), sync=True,
                              images_dev=imgs[k].data_ptr())
            for s in range(2):
                res = singles[s].process_frame(core.GrayImage(host[k, s, 0]),
                                               core.GrayImage(host[k, s, 1]),
                                               bench.motions_for(specs, k)[s])
                got = bp.result(s)
                for a, b in ((res.measured_left, got.measured_left),
                             (res.measured_right, got.measured_right),
                             (res.fused.left, got.fused.left), (res.fused.right, got.fused.right)):
                    assert np.array_equal(a.values, b.values) and np.array_equal(a.valid, b.valid)
                assert np.array_equal(res.intervals_left.lo, got.intervals_left.lo)
                assert res.search_fraction_left == got.search_fraction_left
        assert got.search_fraction_left < 1.0
    finally:
        bench.use_config(5)


@pytest.mark.slow
def test_config3_full_size_moving_boxes_and_salt_noise():
    """BASELINE config 3's features at the full 1242x375 size: three boxes
    moving independently of the ego-motion and 2% salt noise per view, over
    4 frames (fallback windows, LR rejection, adopt/drop), vs the oracle."""
    import bench
    from paper_1708_06301_b200 import core
    rig = core.StereoRig(**bench.RIG)
    n = 4
    specs = bench.sequence_specs(1, seed0=3000)
    boxes, poses, motions = specs[0][0], specs[0][1], specs[0][2]
    rng = np.random.default_rng(303)
    movers = [1, 4, 6]
    vel = rng.uniform(-0.5, 0.5, (len(movers), 3)) * np.array([1.0, 0.0, 1.0])
    per_frame = []
    for k in range(n):
        b = boxes.copy()
        for i, bi in enumerate(movers):
            b[bi, 0:2] += vel[i, 0] * k
            b[bi, 4:6] += vel[i, 2] * k
        per_frame.append(b)
    frames = _render(rig, per_frame, poses[:n], seed=17, scale=bench.TEXTURE_SCALE)
    for img in frames:
        for v in range(2):
            img[v][rng.random(img[v].shape) < 0.02] = 255
    fr = _compare(rig, frames, motions[:n])
    assert fr[0] == 1.0 and min(fr[1:]) < 1.0


@pytest.mark.parametrize("w,h,d_max", [(2, 2, 1), (3, 2, 2), (33, 2, 8), (40, 3, 39), (7, 64, 6), (64, 2, 63)])
def test_degenerate_shapes_match_oracle(w, h, d_max):
    """Edge shapes the reference accepts (at least 2x2, d_max < W): two-row
    images, narrow column bands, d_max = W - 1, widths around a warp: two
    frames (full range, then predicted under a small motion) vs the oracle."""
    from paper_1708_06301_b200 import core
    rig = core.StereoRig(f=float(max(w, 8)), b=0.5, cx=(w - 1) / 2.0, cy=(h - 1) / 2.0,
                         width=w, height=h, d_max=d_max)
    rng = np.random.default_rng(w * 100 + h)
    frames = [rng.integers(0, 256, (2, h, w)).astype(np.uint8) for _ in range(2)]
    frames[1][1] = np.roll(frames[1][0], -1, axis=1)   # some structure to match
    motions = [None, core.make_motion(t=(0.01, 0.0, -0.02))]
    _compare(rig, frames, motions)


@pytest.mark.parametrize("window,p1,p2,tau_sad", [(5, 7.0, 86.0, 900.0), (7, 7.0, 86.0, 3000.0),
                                                  (9, 10.0, 120.0, 5000.0), (3, 1.0, 1.0, 200.0)])
def test_window_and_penalty_variants_match_oracle(window, p1, p2, tau_sad):
    """Parameter edges of sgm.py:40-46: window 5 (u16 aggregation), window 7
    and 9 (the u16 sum bound fails: float32 aggregation, generic cost
    kernel), P1 == P2 (neighbour terms tie with the m + P2 term), three
    frames of a rendered scene vs the oracle."""
    from paper_1708_06301_b200 import core, pipeline, scenes, sgm
    rig = core.StereoRig(f=160.0, b=0.54, cx=79.5, cy=31.5, width=160, height=64, d_max=47)
    boxes, poses, motions = scenes.sequence_spec(seed=77 + window, n_frames=3, step=0.5,
                                                 yaw_deg=0.5, z_range=(2.5, 12.0))
    frames = _render(rig, [boxes] * 3, poses, seed=9, scale=0.05)
    params = pipeline.PipelineParams(sgm=sgm.SgmParams(window=window, p1=p1, p2=p2,
                                                       tau_sad=tau_sad))
    _compare_params(rig, frames, motions, params,
                    O.OracleParams(window=window, p1=p1, p2=p2, tau_sad=tau_sad))


@pytest.mark.parametrize("w,h,d_max", [(352, 24, 300), (520, 16, 511)])
def test_large_disparity_range_matches_oracle(w, h, d_max):
    """d_max beyond config 4's 255 up to the device limit 511 (the widest
    lane-group instances of the aggregation and WTA): full range then a
    predicted frame vs the oracle."""
    from paper_1708_06301_b200 import core
    rig = core.StereoRig(f=float(w), b=0.5, cx=(w - 1) / 2.0, cy=(h - 1) / 2.0,
                         width=w, height=h, d_max=d_max)
    rng = np.random.default_rng(d_max)
    base = rng.integers(0, 256, (h, w + d_max)).astype(np.uint8)
    shift = d_max // 3
    frames = [np.stack([base[:, shift:shift + w], base[:, :w]]) for _ in range(2)]
    motions = [None, core.make_motion(t=(0.0, 0.0, -0.05))]
    _compare(rig, frames, motions)


def _compare_params(rig, frames, motions, params, oparams):
    from paper_1708_06301_b200 import core, pipeline
    pipe = pipeline.DisparityPipeline(rig, params)
    orc = O.OracleStereo(rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max, oparams)
    for k, (img, motion) in enumerate(zip(frames, motions)):
        res = pipe.process_frame(core.GrayImage(img[0]), core.GrayImage(img[1]), motion)
        want = orc.step(img[0], img[1], motion, keep_volumes=True)
        for view, name in ((0, "left"), (1, "right")):
            assert np.array_equal(res.total_volume(view), want[name + "_total"]), (k, name)
            meas = res.measured_left if view == 0 else res.measured_right
            var = res.measured_left_var if view == 0 else res.measured_right_var
            assert np.array_equal(meas.values, want[name + "_meas"][0]), (k, name, "wta")
            assert np.array_equal(var.values, want[name + "_meas"][1]), (k, name, "r")
            keep = res.keep_left if view == 0 else res.keep_right
            assert np.array_equal(keep, want[name + "_keep"]), (k, name, "keep")
            fd = res.fused.left if view == 0 else res.fused.right
            assert np.array_equal(fd.valid, want[name + "_fused"][2]), (k, name)
            np.testing.assert_allclose(fd.values, want[name + "_fused"][0], rtol=1e-9, atol=0)
