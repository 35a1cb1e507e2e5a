"""Evaluation metrics and the run_sequence output tree on the B200
(metrics.py:39-117, pipeline.py:241-302) against outputs of the unmodified
reference (tests/golden/metrics.npz, run_sequence.npz) and the oracle."""

import numpy as np
import pytest

import oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_bad_pixel_metrics_match_reference():
    from paper_1708_06301_b200 import core, metrics
    g = load_golden("metrics")
    for case in range(4):
        est, ev, gt, gv = (g[f"c{case}_{k}"] for k in ("est", "ev", "gt", "gv"))
        e, t = core.DisparityMap(est, ev), core.DisparityMap(gt, gv)
        assert metrics.density(e) == float(g[f"c{case}_density"])
        for mode in ("or", "and"):
            r = metrics.bad_pixel_rate(e, t, mode)
            # exact: the rates are formed from integer counts
            assert np.array_equal(np.array([r.rate, r.rate_all, r.density]),
                                  g[f"c{case}_{mode}_rates"]), (case, mode)
            assert np.array_equal(metrics.bad_pixel_mask(e, t, mode), g[f"c{case}_{mode}_mask"])
            assert np.array_equal(metrics.error_image(e, t, mode), g[f"c{case}_{mode}_rgb"])
            assert np.array_equal(metrics.bad_pixel_mask(e, t, mode),
                                  O.bad_mask(est, ev, gt, gv, mode))


def test_metrics_errors():
    from paper_1708_06301_b200 import core, metrics
    a = core.DisparityMap(np.ones((3, 4)), np.ones((3, 4), bool))
    b = core.DisparityMap(np.ones((4, 3)), np.ones((4, 3), bool))
    with pytest.raises(ValueError):
        metrics.bad_pixel_rate(a, a, "xor")
    with pytest.raises(ValueError):
        metrics.bad_pixel_rate(a, b)
    # empty ground truth: zeros (metrics.py:57-58)
    z = core.DisparityMap(np.zeros((3, 4)), np.zeros((3, 4), bool))
    assert metrics.bad_pixel_rate(a, z) == metrics.BadPixelResult(0.0, 0.0, 0.0)


def test_run_sequence_output_tree_matches_reference(tmp_path):
    """The reference's own sequence runner, KITTI writer and metrics files
    (pipeline.py:241-302, kitti_io.py) on top of the device stages:
    install() into the unmodified package from baseline/_ref, then
    egostereo.run_sequence must write exactly the tree the reference wrote
    with its numpy stages (golden run_sequence.npz)."""
    import os
    import sys
    cv2 = pytest.importorskip("cv2")
    from conftest import ROOT
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "egostereo")):
        pytest.skip("reference not installed (tools/install_reference.sh)")
    sys.path.insert(0, ref)
    import egostereo
    from egostereo import core, pipeline
    from paper_1708_06301_b200 import install
    install.install(egostereo)
    try:
        g = load_golden("run_sequence")
        f, b, cx, cy, w, h, d_max = g["rig"]
        rig = core.StereoRig(f=f, b=b, cx=cx, cy=cy, width=int(w), height=int(h),
                             d_max=int(d_max))
        n = len([k for k in g.files if k.endswith("_left")])
        seq = pipeline.Sequence(
            rig, [core.GrayImage(g[f"f{k}_left"]) for k in range(n)],
            [core.GrayImage(g[f"f{k}_right"]) for k in range(n)],
            [g[f"f{k}_motion"] if bool(g[f"f{k}_has_motion"]) else None for k in range(n)],
            gt_left=[core.DisparityMap(g[f"f{k}_gt_d"], g[f"f{k}_gt_v"]) for k in range(n)],
            gt_right=[core.DisparityMap(g[f"f{k}_gtr_d"], g[f"f{k}_gtr_v"]) for k in range(n)])
        results = pipeline.run_sequence(seq, out_dir=str(tmp_path), metric_mode="or")
        assert pipeline.DisparityPipeline.__b200__
    finally:
        install.uninstall(egostereo)
        sys.path.remove(ref)
    assert len(results) == n
    assert open(tmp_path / "metrics.txt").read() == str(g["metrics_txt"])
    assert open(tmp_path / "summary.txt").read() == str(g["summary_txt"])
    for k in range(n):
        disp = cv2.imread(str(tmp_path / "disp_0" / f"{k:06d}.png"), cv2.IMREAD_UNCHANGED)
        assert np.array_equal(disp, g[f"f{k}_disp_png"]), k
        err = cv2.imread(str(tmp_path / "err_0" / f"{k:06d}.png"), cv2.IMREAD_UNCHANGED)
        assert np.array_equal(err, g[f"f{k}_err_png"]), k


def test_batched_device_metrics_match_host_metrics():
    """BatchedPipeline.metrics (device ground truth, one read-back) equals the
    host-map path on every sequence."""
    import torch
    import bench
    from paper_1708_06301_b200 import core, metrics, pipeline
    rig = core.StereoRig(f=180.0, b=0.54, cx=151.0, cy=46.0, width=310, height=94, d_max=40)
    B = 3
    specs = bench.sequence_specs(B, seed0=900)
    imgs, gts = bench.render_frames(specs, [0, 1, 2], "cuda:0", rig=rig, with_gt=True)
    bp = pipeline.BatchedPipeline(rig, B)
    for k in range(3):
        bp.process_frames(None, bench.motions_for(specs, k), sync=True,
                          images_dev=imgs[k].data_ptr())
    gt = gts[2][:, 0].contiguous()                       # left view, [B][H][W]
    gv = (gt > 0).to(torch.uint8).contiguous()
    hw = rig.width * rig.height
    for mode in ("or", "and"):
        dev = bp.metrics(gt.data_ptr(), gv.data_ptr(), hw, view=0, mode=mode)
        for s in range(B):
            fl = bp.result(s).fused.left
            t = core.DisparityMap(gt[s].cpu().numpy(), gv[s].cpu().numpy().astype(bool))
            assert dev[s][0] == metrics.bad_pixel_rate(fl, t, mode), (s, mode)
            assert dev[s][1] == metrics.density(fl)
