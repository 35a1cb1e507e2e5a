"""Frame-step parity on the B200: the fused device pipeline against golden
sequences from the reference, the full-size config-1 pair, and the batched
engine against single sequences."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

RTOL = 1e-9


def _rig(g):
    from paper_1708_06301_b200 import core
    f, b, cx, cy, w, h, d_max = g["rig"]
    return core.StereoRig(f=f, b=b, cx=cx, cy=cy, width=int(w), height=int(h), d_max=int(d_max))


def _check_frame(res, g, k, check_volumes=True):
    for v, view in (("l", 0), ("r", 1)):
        iv = res.intervals_left if view == 0 else res.intervals_right
        assert np.array_equal(iv.lo, g[f"f{k}_{v}_lo"]), (k, v, "lo")
        assert np.array_equal(iv.hi, g[f"f{k}_{v}_hi"]), (k, v, "hi")
        meas = res.measured_left if view == 0 else res.measured_right
        mvar = res.measured_left_var if view == 0 else res.measured_right_var
        assert np.array_equal(meas.values, g[f"f{k}_{v}_meas_d"]), (k, v, "wta")
        assert np.array_equal(meas.valid, g[f"f{k}_{v}_meas_v"]), (k, v, "valid")
        assert np.array_equal(mvar.values, g[f"f{k}_{v}_meas_r"]), (k, v, "r")
        keep = res.keep_left if view == 0 else res.keep_right
        assert np.array_equal(keep, g[f"f{k}_{v}_keep"]), (k, v, "keep")
        pred = res.predicted_left if view == 0 else res.predicted_right
        pvar = res.predicted_left_var if view == 0 else res.predicted_right_var
        assert np.array_equal(pred.valid, g[f"f{k}_{v}_pred_v"]), (k, v, "pred valid")
        np.testing.assert_allclose(pred.values, g[f"f{k}_{v}_pred_d"], rtol=RTOL, atol=0)
        np.testing.assert_allclose(pvar.values, g[f"f{k}_{v}_pred_p"], rtol=RTOL, atol=0)
        fused = res.fused
        fd = fused.left if view == 0 else fused.right
        fp = fused.left_var if view == 0 else fused.right_var
        assert np.array_equal(fd.valid, g[f"f{k}_{v}_fused_v"]), (k, v, "fused valid")
        np.testing.assert_allclose(fd.values, g[f"f{k}_{v}_fused_d"], rtol=RTOL, atol=0)
        np.testing.assert_allclose(fp.values, g[f"f{k}_{v}_fused_p"], rtol=RTOL, atol=0)
        if check_volumes and f"f{k}_{v}_cost" in g:
            assert np.array_equal(res.cost_volume(view), g[f"f{k}_{v}_cost"]), (k, v, "cost")
            assert np.array_equal(res.total_volume(view), g[f"f{k}_{v}_total"]), (k, v, "total")
    np.testing.assert_allclose([res.search_fraction_left, res.search_fraction_right],
                               g[f"f{k}_frac"], rtol=1e-15)


def _frames(g):
    k = 0
    while f"f{k}_left" in g:
        motion = g[f"f{k}_motion"] if bool(g[f"f{k}_has_motion"]) else None
        yield k, g[f"f{k}_left"], g[f"f{k}_right"], motion
        k += 1


@pytest.mark.parametrize("name,p1,p2", [("seq_small", 7.0, 86.0), ("seq_drive", 8.0, 100.0)])
def test_sequence_matches_reference(name, p1, p2):
    from paper_1708_06301_b200 import core, pipeline, sgm
    g = load_golden(name)
    params = pipeline.PipelineParams(sgm=sgm.SgmParams(p1=p1, p2=p2))
    pipe = pipeline.DisparityPipeline(_rig(g), params)
    n = 0
    for k, left, right, motion in _frames(g):
        res = pipe.process_frame(core.GrayImage(left), core.GrayImage(right), motion)
        assert res.frame == k
        _check_frame(res, g, k)
        n += 1
    assert n >= 4


def test_float_penalties_sequence_matches_oracle():
    """Non-integer P1/P2 take the float32 aggregation path; compare with the
    oracle (itself pinned to the reference) on the small sequence."""
    import oracle as O
    from paper_1708_06301_b200 import core, pipeline, sgm
    g = load_golden("seq_small")
    rig = _rig(g)
    params = pipeline.PipelineParams(sgm=sgm.SgmParams(p1=6.5, p2=80.25))
    pipe = pipeline.DisparityPipeline(rig, params)
    orc = O.OracleStereo(rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max,
                         O.OracleParams(p1=6.5, p2=80.25))
    for k, left, right, motion in _frames(g):
        res = pipe.process_frame(core.GrayImage(left), core.GrayImage(right), motion)
        out = orc.step(left, right, motion, keep_volumes=True)
        for view, name in ((0, "left"), (1, "right")):
            assert np.array_equal(res.total_volume(view), out[name + "_total"]), (k, name)
            meas = res.measured_left if view == 0 else res.measured_right
            assert np.array_equal(meas.values, out[name + "_meas"][0])
            fd = res.fused.left if view == 0 else res.fused.right
            assert np.array_equal(fd.valid, out[name + "_fused"][2])
            np.testing.assert_allclose(fd.values, out[name + "_fused"][0], rtol=RTOL, atol=0)


def test_config1_full_size_full_range():
    """Config 1 (1242x375, D=128, full range) against the reference's
    outputs: WTA, variance, keep masks, sampled rows and row/column sums of
    the cost and aggregated volumes."""
    from paper_1708_06301_b200 import core, pipeline
    g = load_golden("config1")
    rig = core.StereoRig(f=718.9, b=0.54, cx=607.0, cy=185.0, width=1242, height=375, d_max=127)
    pipe = pipeline.DisparityPipeline(rig)
    res = pipe.process_frame(core.GrayImage(g["left"]), core.GrayImage(g["right"]), None)
    rows = np.array([0, 187, 374])
    for view, name in ((0, "left"), (1, "right")):
        meas = res.measured_left if view == 0 else res.measured_right
        assert np.array_equal(meas.values.astype(np.uint8), g[f"{name}_wta"])
        r = (res.measured_left_var if view == 0 else res.measured_right_var).values
        assert np.array_equal(r.astype(np.float32), g[f"{name}_r"])
        cost = res.cost_volume(view)
        total = res.total_volume(view)
        assert np.isfinite(cost).all() and np.isfinite(total).all()
        c = cost.astype(np.int64)
        s = total.astype(np.int64)
        assert np.array_equal(c.sum(axis=(1, 2)), g[f"{name}_cost_rowsum"])
        assert np.array_equal(c.sum(axis=(0, 2)), g[f"{name}_cost_colsum"])
        assert np.array_equal(s.sum(axis=(1, 2)), g[f"{name}_total_rowsum"])
        assert np.array_equal((s * s).sum(axis=(1, 2)), g[f"{name}_total_rowsum_sq"])
        assert np.array_equal(s.sum(axis=(0, 2)), g[f"{name}_total_colsum"])
        assert np.array_equal(s.sum(axis=(0, 1)), g[f"{name}_total_dsum"])
        assert np.array_equal(total[rows].astype(np.uint16), g[f"{name}_total_rows"])
        assert np.array_equal(cost[rows].astype(np.uint16), g[f"{name}_cost_rows"])
    kl = np.unpackbits(g["keep_left"])[: rig.width * rig.height].reshape(rig.shape).astype(bool)
    kr = np.unpackbits(g["keep_right"])[: rig.width * rig.height].reshape(rig.shape).astype(bool)
    assert np.array_equal(res.keep_left, kl) and np.array_equal(res.keep_right, kr)
    assert res.search_fraction_left == 1.0


def test_batched_equals_single_sequences():
    """B sequences advanced together give exactly the per-sequence results."""
    from paper_1708_06301_b200 import core, pipeline
    g = load_golden("seq_small")
    rig = _rig(g)
    frames = list(_frames(g))
    B = 3
    # sequence s starts s frames late (empty state + motion -> full range)
    bp = pipeline.BatchedPipeline(rig, B)
    singles = [pipeline.DisparityPipeline(rig) for _ in range(B)]
    for t in range(len(frames)):
        imgs = np.empty((B, 2, rig.height, rig.width), np.uint8)
        motions = []
        for s in range(B):
            k = max(t - s, 0)
            _, left, right, motion = frames[k]
            imgs[s, 0], imgs[s, 1] = left, right
            motions.append(motion if t - s > 0 else None)
        bp.process_frames(imgs, motions)
        for s in range(B):
            want = singles[s].process_frame(core.GrayImage(imgs[s, 0]), core.GrayImage(imgs[s, 1]),
                                            motions[s])
            got = bp.result(s)
            for a, b in ((got.fused.left, want.fused.left), (got.fused.right, want.fused.right)):
                assert np.array_equal(a.valid, b.valid) and np.array_equal(a.values, b.values)
            assert np.array_equal(got.measured_left.values, want.measured_left.values)
            assert got.search_fraction_left == want.search_fraction_left


def test_reset_and_baseline_mode():
    from paper_1708_06301_b200 import core, pipeline
    g = load_golden("seq_small")
    rig = _rig(g)
    frames = list(_frames(g))
    base = pipeline.DisparityPipeline(rig, pipeline.PipelineParams(baseline=True))
    for k, left, right, motion in frames[:3]:
        res = base.process_frame(core.GrayImage(left), core.GrayImage(right), motion)
        assert res.search_fraction_left == 1.0
        assert not res.predicted_left.valid.any()
    pipe = pipeline.DisparityPipeline(rig)
    for k, left, right, motion in frames[:2]:
        pipe.process_frame(core.GrayImage(left), core.GrayImage(right), motion)
    pipe.reset()
    assert pipe.state.frame == -1
    k, left, right, motion = frames[1]
    res = pipe.process_frame(core.GrayImage(left), core.GrayImage(right), motion)
    assert res.frame == 0 and res.search_fraction_left == 1.0   # empty state -> full range
