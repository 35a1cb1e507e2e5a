"""Stage-level parity on the B200: each drop-in function against the golden
vectors the reference produced (oracle/make_golden.py).  Integer outputs
must match bit for bit; floating-point state within 1e-9 relative (the
north star allows 1e-4)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module")
def es():
    import paper_1708_06301_b200 as pkg
    from paper_1708_06301_b200 import core, fusion, prediction, sgm
    return pkg, core, sgm, prediction, fusion


def test_cost_aggregation_wta_variance(es):
    pkg, core, sgm, _, _ = es
    g = load_golden("cost_agg")
    for case in range(4):
        left, right = g[f"c{case}_left"], g[f"c{case}_right"]
        lo, hi = g[f"c{case}_lo"], g[f"c{case}_hi"]
        d_max = g[f"c{case}_w3_left_cost"].shape[2] - 1
        iv = sgm.IntervalMap(lo, hi, d_max)
        for window in (3, 5):
            prm = sgm.SgmParams(window=window)
            for view in ("left", "right"):
                key = f"c{case}_w{window}_{view}"
                vol = sgm.matching_cost(core.GrayImage(left), core.GrayImage(right), iv, prm, view)
                assert np.array_equal(vol.data, g[key + "_cost"]), key
                agg = sgm.aggregate_paths(vol, prm)
                assert np.array_equal(agg.data, g[key + "_total"]), key
                disp = sgm.select_disparity(agg)
                assert np.array_equal(disp.values, g[key + "_wta"]), key
                assert np.array_equal(disp.valid, g[key + "_valid"]), key
                r = sgm.matching_variance_map(agg, disp, prm)
                assert np.array_equal(r.values, g[key + "_r"]), key


@pytest.mark.parametrize("k", range(4))
def test_hand_volumes_integer_and_float_penalties(es, k):
    _, _, sgm, _, _ = es
    g = load_golden("cost_agg")
    C = g[f"vol{k}_cost"]
    p1, p2 = g[f"vol{k}_p"]
    iv = sgm.IntervalMap(g[f"vol{k}_lo"], g[f"vol{k}_hi"], C.shape[2] - 1)
    prm = sgm.SgmParams(p1=float(p1), p2=float(p2))
    agg = sgm.aggregate_paths(sgm.CostVolume(C, iv), prm)
    assert np.array_equal(agg.data, g[f"vol{k}_total"])
    disp = sgm.select_disparity(agg)
    assert np.array_equal(disp.values, g[f"vol{k}_wta"])
    r = sgm.matching_variance_map(agg, disp, prm)
    assert np.array_equal(r.values, g[f"vol{k}_r"])


def test_reference_hand_table(es):
    """The reference's 1x3 hand table (tests/test_sgm.py:134-150 semantics)."""
    _, _, sgm, _, _ = es
    C = np.array([[[0.0, 4.0, 8.0], [5.0, 1.0, 6.0], [2.0, 3.0, 0.0]]], np.float32)
    iv = sgm.IntervalMap(np.zeros((1, 3), np.int64), np.full((1, 3), 2, np.int64), 2)
    got = sgm.aggregate_paths(sgm.CostVolume(C, iv), sgm.SgmParams(p1=1.0, p2=2.0)).data
    want = np.array([[[1.0, 32.0, 65.0], [42.0, 10.0, 50.0], [17.0, 24.0, 1.0]]])
    assert np.array_equal(got.astype(np.float64), want)
    disp = sgm.select_disparity(sgm.CostVolume(got, iv))
    assert not disp.valid[0, 0] and disp.values[0, 1] == 1.0 and disp.values[0, 2] == 2.0


def test_matching_variance_scalar_walk(es):
    _, _, sgm, _, _ = es
    prm = sgm.SgmParams(s_max=10.0, r_min=0.25)
    assert sgm.matching_variance(np.array([13.0, 8.0, 5.0, 7.0, 14.0]), 0, 2, prm) == 2.0
    assert sgm.matching_variance(np.full(5, 9.0), 3, 3, prm) == 4.0
    assert sgm.matching_variance(np.array([100.0, 0.0, 100.0]), 0, 1, prm) == 0.25
    assert sgm.matching_variance(np.array([0.0, 10.0]), 0, 0, prm) == 0.25
    with pytest.raises(ValueError):
        sgm.matching_variance(np.array([1.0, 2.0]), 0, 9, prm)


def test_intervals_checks_fusion(es):
    _, core, sgm, _, fusion = es
    g = load_golden("intervals_checks_fusion")
    rig = core.StereoRig(f=53.0, b=0.5, cx=26.0, cy=9.5, width=53, height=20, d_max=40)
    iv = sgm.search_intervals(core.DisparityMap(g["iv_d"], g["iv_valid"]),
                              core.VarianceMap(g["iv_p"]), rig)
    assert np.array_equal(iv.lo, g["iv_lo"]) and np.array_equal(iv.hi, g["iv_hi"])
    ml = core.DisparityMap(g["chk_dl"], g["chk_vl"])
    mr = core.DisparityMap(g["chk_dr"], g["chk_vr"])
    kl, kr = sgm.lr_consistency(ml, mr, 1.0)
    assert np.array_equal(kl, g["chk_lr_l"]) and np.array_equal(kr, g["chk_lr_r"])
    L, R = core.GrayImage(g["chk_left"]), core.GrayImage(g["chk_right"])
    for window, tau in ((3, 200.0), (5, 900.0)):
        assert np.array_equal(sgm.sad_check(L, R, ml, window, tau, "left"), g[f"chk_sad_l_w{window}"])
        assert np.array_equal(sgm.sad_check(L, R, mr, window, tau, "right"), g[f"chk_sad_r_w{window}"])
    vp, vm = g["fu_vp"], g["fu_vm"]
    fd, fp = fusion.fuse_maps(core.DisparityMap(np.where(vp, g["fu_dp"], 0), vp),
                              core.VarianceMap(g["fu_pp"]),
                              core.DisparityMap(np.where(vm, g["fu_dm"], 0), vm),
                              core.VarianceMap(g["fu_rm"]), fusion.FusionParams(1.0))
    assert np.array_equal(fd.valid, g["fu_v"])
    assert np.array_equal(fd.values, g["fu_d"]) and np.array_equal(fp.values, g["fu_p"])


def test_prediction(es):
    _, core, _, prediction, _ = es
    from paper_1708_06301_b200 import geometry
    g = load_golden("prediction")
    f, b, cx, cy, w, h, d_max = g["rig"]
    rig = core.StereoRig(f=f, b=b, cx=cx, cy=cy, width=int(w), height=int(h), d_max=int(d_max))
    for t in range(10):
        T = g[f"t{t}_T"]
        assert np.array_equal(geometry.disparity_homography(rig, T), g[f"t{t}_HL"])
        dm = core.DisparityMap(g[f"t{t}_d"], g[f"t{t}_v"])
        vm = core.VarianceMap(g[f"t{t}_p"])
        assert np.array_equal(prediction.reject_edges(dm, 3.0, 1), g[f"t{t}_edges"])
        prm = prediction.PredictionParams(edge_reject=bool(g[f"t{t}_edge"]))
        state = core.FilterState(dm, vm, dm.copy(), vm.copy(), 0)
        out = prediction.predict_maps(state, T, rig, prm)
        for tag, dmap, pmap in (("pl", out.left, out.left_var), ("pr", out.right, out.right_var)):
            assert np.array_equal(dmap.valid, g[f"t{t}_{tag}_v"]), (t, tag)
            np.testing.assert_allclose(dmap.values, g[f"t{t}_{tag}_d"], rtol=RTOL, atol=0)
            np.testing.assert_allclose(pmap.values, g[f"t{t}_{tag}_p"], rtol=RTOL, atol=0)
        assert out.frame == 1
        fd, fp = prediction.fill_zoom_holes(out.left, out.left_var, 3.0, 0.5)
        assert np.array_equal(fd.valid, g[f"t{t}_fl_v"])
        np.testing.assert_allclose(fd.values, g[f"t{t}_fl_d"], rtol=RTOL, atol=0)
        np.testing.assert_allclose(fp.values, g[f"t{t}_fl_p"], rtol=RTOL, atol=0)


def test_identity_prediction_is_bit_exact_fixed_point(es):
    """Acceptance criterion 2 (reference tests/test_acceptance.py:109-143)."""
    _, core, _, prediction, _ = es
    rig = core.StereoRig(f=16.0, b=0.5, cx=7.5, cy=3.5, width=16, height=8, d_max=6)
    rng = np.random.default_rng(0)
    prm = prediction.PredictionParams(q=0.0, edge_reject=False, fill_holes=False)
    for _ in range(20):
        valid = rng.random(rig.shape) < 0.6
        values = np.where(valid, rng.uniform(0.5, 6.0, rig.shape), 0.0)
        var = np.where(valid, rng.uniform(0.1, 4.0, rig.shape), 0.0)
        d = core.DisparityMap(values, valid)
        p = core.VarianceMap(var)
        out = prediction.predict_maps(core.FilterState(d, p, d.copy(), p.copy()), np.eye(4), rig, prm)
        assert np.array_equal(out.left.values, values) and np.array_equal(out.left.valid, valid)
        assert np.array_equal(out.left_var.values, var)


def test_point_at_infinity_raises(es):
    pkg, core, _, prediction, _ = es
    from paper_1708_06301_b200 import geometry
    H = np.eye(4)
    H[3] = [0.0, 0.0, 0.0, 0.0]
    with pytest.raises(pkg.PointAtInfinityError):
        geometry.warp_point(H, np.array([1.0, 2.0, 3.0]))
    out = geometry.warp_point(np.eye(4), np.array([[1.0, 2.0, 3.0], [4.0, 5.0, 6.0]]))
    assert np.array_equal(out, [[1.0, 2.0, 3.0], [4.0, 5.0, 6.0]])
