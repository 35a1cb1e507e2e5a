"""The benchmark's own code path against the oracle: BatchedPipeline with
device-resident inputs and deferred (non-syncing) steps, B = 12 sequences
(> 8, so two concurrent partial sums as in the B = 64 bench), the device
renderer's scenes, both SGM regime kernels (frame 0 full range, later
frames reduced)."""

import ctypes

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def test_batched_deferred_path_matches_oracle():
    import torch
    from paper_1708_06301_b200 import _lib, pipeline, scenes
    from paper_1708_06301_b200.core import StereoRig
    B, n = 12, 4
    rig = StereoRig(f=180.0, b=0.54, cx=151.0, cy=46.0, width=310, height=94, d_max=40)
    specs = [scenes.sequence_spec(seed=900 + s, n_frames=n, step=0.5, z_range=(4.0, 30.0))
             for s in range(B)]
    rs = _lib.rig_struct(rig)
    boxes = np.ascontiguousarray(np.stack([sp[0] for sp in specs]), np.float64)
    seeds = np.arange(B, dtype=np.int64) + 3
    imgs = torch.empty((n, B, 2, rig.height, rig.width), dtype=torch.uint8, device="cuda")
    for k in range(n):
        poses = np.ascontiguousarray(np.stack([sp[1][k] for sp in specs]), np.float64)
        _lib.call("es_render", ctypes.byref(rs), _lib.ptr(boxes), boxes.shape[1], _lib.ptr(poses),
                  _lib.ptr(seeds), B, ctypes.c_double(0.05), 12,
                  ctypes.c_void_p(imgs[k].data_ptr()), None, ctypes.c_void_p(0))
    torch.cuda.synchronize()
    host = imgs.cpu().numpy()
    bp = pipeline.BatchedPipeline(rig, B)
    # frame 0 synced (establishes have_state), the rest deferred like the bench
    bp.process_frames(None, [sp[2][0] for sp in specs], sync=True, images_dev=imgs[0].data_ptr())
    for k in range(1, n):
        bp.process_frames(None, [sp[2][k] for sp in specs], sync=False,
                          images_dev=imgs[k].data_ptr())
    bp.sync()
    kitti = bp.fused_kitti(0)
    for s in range(B):
        orc = O.OracleStereo(rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max)
        for k in range(n):
            want = orc.step(host[k, s, 0], host[k, s, 1], specs[s][2][k])
        got = bp.result(s)
        for view, name in ((0, "left"), (1, "right")):
            meas = got.measured_left if view == 0 else got.measured_right
            assert np.array_equal(meas.values, want[name + "_meas"][0]), (s, name)
            fd = got.fused.left if view == 0 else got.fused.right
            fp = got.fused.left_var if view == 0 else got.fused.right_var
            assert np.array_equal(fd.valid, want[name + "_fused"][2]), (s, name)
            np.testing.assert_allclose(fd.values, want[name + "_fused"][0], rtol=1e-9, atol=0)
            np.testing.assert_allclose(fp.values, want[name + "_fused"][1], rtol=1e-9, atol=0)
        # the e2e result encoding (kitti_io.write_disparity_png)
        fl = want["left_fused"]
        enc = np.where(fl[2], np.maximum(np.rint(fl[0] * 256.0), 1.0), 0.0).astype(np.uint16)
        assert np.array_equal(kitti[s], enc), s
        assert got.search_fraction_left < 1.0


def test_e2e_host_inputs_async_exports_match_oracle():
    """The e2e pattern: pinned host images uploaded on the copy stream
    (double-buffered), deferred steps, one asynchronous KITTI export per step
    into its own pinned buffer, a fence and one sync at the end -- every
    step's export must equal that frame's oracle state."""
    import torch
    from paper_1708_06301_b200 import pipeline, scenes
    from paper_1708_06301_b200.core import StereoRig
    import bench
    B, n = 3, 5
    rig = StereoRig(f=180.0, b=0.54, cx=151.0, cy=46.0, width=310, height=94, d_max=40)
    specs = [scenes.sequence_spec(seed=700 + s, n_frames=n, step=0.5, z_range=(4.0, 30.0))
             for s in range(B)]
    imgs = bench.render_frames(specs, list(range(n)), "cuda:0", rig=rig)
    staged = [imgs[k].cpu().pin_memory() for k in range(n)]
    outs = [torch.empty((B, rig.height, rig.width), dtype=torch.int16, pin_memory=True)
            for _ in range(n)]
    bp = pipeline.BatchedPipeline(rig, B)
    bp.process_frames(staged[0].numpy(), [sp[2][0] for sp in specs], sync=True)
    bp.fused_kitti(0, out=outs[0].numpy().view(np.uint16), sync=True)
    for k in range(1, n):
        bp.process_frames(staged[k].numpy(), [sp[2][k] for sp in specs], sync=False)
        bp.fused_kitti(0, out=outs[k].numpy().view(np.uint16), sync=False)
    bp.fence()
    bp.sync()
    host = imgs.cpu().numpy()
    for s in range(B):
        orc = O.OracleStereo(rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max)
        for k in range(n):
            want = orc.step(host[k, s, 0], host[k, s, 1], specs[s][2][k])["left_fused"]
            enc = np.where(want[2], np.maximum(np.rint(want[0] * 256.0), 1.0), 0.0).astype(np.uint16)
            assert np.array_equal(outs[k].numpy().view(np.uint16)[s], enc), (s, k)


@pytest.mark.slow
def test_config5_full_batch_declared_subset_matches_oracle():
    """The benchmark's exact configuration -- B = 64 sequences of 1242x375,
    D = 128 in one context (two partial sums, split row sweeps, deferred
    steps) -- with sequences {0, 21, 42, 63} checked against the oracle over
    frames 0-2 (parity for config 5 on a declared subset)."""
    import bench
    from paper_1708_06301_b200 import core, pipeline
    rig = core.StereoRig(**bench.RIG)
    B, n = 64, 3
    specs = bench.sequence_specs(B, seed0=1000)
    imgs = bench.render_frames(specs, list(range(n)), "cuda:0")
    bp = pipeline.BatchedPipeline(rig, B)
    bp.process_frames(None, bench.motions_for(specs, 0), sync=True, images_dev=imgs[0].data_ptr())
    for k in range(1, n):
        bp.process_frames(None, bench.motions_for(specs, k), sync=False,
                          images_dev=imgs[k].data_ptr())
    bp.sync()
    host = imgs.cpu().numpy()
    for s in (0, 21, 42, 63):
        orc = O.OracleStereo(rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max)
        for k in range(n):
            want = orc.step(host[k, s, 0], host[k, s, 1], bench.motions_for(specs, k)[s])
        got = bp.result(s)
        for view, name in ((0, "left"), (1, "right")):
            meas = got.measured_left if view == 0 else got.measured_right
            assert np.array_equal(meas.values, want[name + "_meas"][0]), (s, name)
            keep = got.keep_left if view == 0 else got.keep_right
            assert np.array_equal(keep, want[name + "_keep"]), (s, name)
            fd = got.fused.left if view == 0 else got.fused.right
            fp = got.fused.left_var if view == 0 else got.fused.right_var
            assert np.array_equal(fd.valid, want[name + "_fused"][2]), (s, name)
            np.testing.assert_allclose(fd.values, want[name + "_fused"][0], rtol=1e-9, atol=0)
            np.testing.assert_allclose(fp.values, want[name + "_fused"][1], rtol=1e-9, atol=0)
        assert got.search_fraction_left < 1.0


@pytest.mark.parametrize("B", [1, 2, 5, 9])
def test_every_batch_schedule_equals_single_sequences(B):
    """Every aggregation schedule (4 partial sums with split row sweeps for
    B <= 8, 2 partial sums for larger batches; lanes per chain widened for
    small batches) gives each sequence exactly its single-sequence maps."""
    import bench
    from paper_1708_06301_b200 import core, pipeline, scenes
    rig = core.StereoRig(f=180.0, b=0.54, cx=151.0, cy=46.0, width=310, height=94, d_max=40)
    specs = [scenes.sequence_spec(seed=500 + s, n_frames=3, step=0.5, z_range=(4.0, 30.0))
             for s in range(B)]
    imgs = bench.render_frames(specs, [0, 1, 2], "cuda:0", rig=rig)
    host = imgs.cpu().numpy()
    bp = pipeline.BatchedPipeline(rig, B)
    singles = [pipeline.DisparityPipeline(rig) for _ in range(B)]
    for k in range(3):
        bp.process_frames(None, [sp[2][k] for sp in specs], sync=True, images_dev=imgs[k].data_ptr())
        for s in range(B):
            want = singles[s].process_frame(core.GrayImage(host[k, s, 0]), core.GrayImage(host[k, s, 1]),
                                            specs[s][2][k])
            got = bp.result(s)
            for a, b in ((want.measured_left, got.measured_left), (want.fused.right, got.fused.right)):
                assert np.array_equal(a.values, b.values) and np.array_equal(a.valid, b.valid), (B, s, k)
            assert np.array_equal(want.measured_right_var.values, got.measured_right_var.values)


def test_grouped_batch_equals_single_context():
    """BatchedPipeline groups (B >= 24 runs as contexts of ~16 sequences on their own
    streams): the same sequences through groups=2 and groups=1 give
    identical maps -- device-pointer and host-image inputs, deferred and
    synced steps, the KITTI export and the device metrics of every
    sequence (per-group pointer offsets)."""
    import torch
    from paper_1708_06301_b200 import pipeline, scenes
    from paper_1708_06301_b200.core import StereoRig
    import bench
    B, n = 6, 4
    rig = StereoRig(f=180.0, b=0.54, cx=151.0, cy=46.0, width=310, height=94, d_max=40)
    specs = [scenes.sequence_spec(seed=500 + s, n_frames=n, step=0.5, z_range=(4.0, 30.0))
             for s in range(B)]
    imgs, gts = bench.render_frames(specs, list(range(n)), "cuda:0", rig=rig, with_gt=True)
    one = pipeline.BatchedPipeline(rig, B, groups=1)
    two = pipeline.BatchedPipeline(rig, B, groups=2)
    assert two.groups == 2 and len(two.engines) == 2
    three = pipeline.BatchedPipeline(rig, B, groups=3)
    with pytest.raises(AttributeError):
        two.engine
    for k in range(n):
        mot = [sp[2][k] for sp in specs]
        one.process_frames(None, mot, sync=True, images_dev=imgs[k].data_ptr())
        if k % 2:
            two.process_frames(imgs[k].cpu().numpy(), mot, sync=True)
        else:
            two.process_frames(None, mot, sync=False, images_dev=imgs[k].data_ptr())
        three.process_frames(None, mot, sync=False, images_dev=imgs[k].data_ptr())
    two.sync()
    three.sync()
    assert np.array_equal(one.fused_kitti(0), two.fused_kitti(0))
    assert np.array_equal(one.fused_kitti(1), three.fused_kitti(1))
    for s in range(B):
        a, b = one.result(s), two.result(s)
        for name in ("measured_left", "measured_right"):
            assert np.array_equal(getattr(a, name).values, getattr(b, name).values), (s, name)
        assert np.array_equal(a.fused.left.values, b.fused.left.values), s
        assert np.array_equal(a.fused.right_var.values, b.fused.right_var.values), s
        assert a.search_fraction_left == b.search_fraction_left
    gt = gts[n - 1][:, 0].contiguous()
    gv = (gt > 0).to(torch.uint8).contiguous()
    h, w = rig.height, rig.width
    qa = one.metrics(gt.data_ptr(), gv.data_ptr(), h * w)
    qb = two.metrics(gt.data_ptr(), gv.data_ptr(), h * w)
    assert [(r.rate, d) for r, d in qa] == [(r.rate, d) for r, d in qb]
    with pytest.raises(ValueError):
        pipeline.BatchedPipeline(rig, 5, groups=2)
