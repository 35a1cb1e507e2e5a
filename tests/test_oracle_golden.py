"""Pin the CPU oracle against golden vectors produced by the reference itself
(oracle/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle as O
from conftest import load_golden


def _views():
    return ("left", "right")


def test_cost_aggregation_wta_variance():
    g = load_golden("cost_agg")
    for case in range(4):
        left, right = g[f"c{case}_left"], g[f"c{case}_right"]
        lo, hi = g[f"c{case}_lo"], g[f"c{case}_hi"]
        d_max = g[f"c{case}_w3_left_cost"].shape[2] - 1
        for window in (3, 5):
            prm = O.OracleParams(window=window)
            for view in _views():
                key = f"c{case}_w{window}_{view}"
                cost = O.sad_volume(left, right, lo, hi, d_max, window, view)
                assert np.array_equal(cost, g[key + "_cost"]), key
                total = O.sgm_total(cost, prm.p1, prm.p2)
                assert np.array_equal(total, g[key + "_total"]), key
                d, v = O.wta(total)
                assert np.array_equal(d, g[key + "_wta"]) and np.array_equal(v, g[key + "_valid"])
                r = O.variance_counts(total, lo, hi, d, prm.s_max, prm.r_min)
                assert np.array_equal(r, g[key + "_r"]), key


@pytest.mark.parametrize("k", range(4))
def test_hand_volumes_float_and_integer(k):
    g = load_golden("cost_agg")
    C = g[f"vol{k}_cost"]
    p1, p2 = g[f"vol{k}_p"]
    total = O.sgm_total(C, float(p1), float(p2))
    assert np.array_equal(total, g[f"vol{k}_total"])
    d, _ = O.wta(total)
    assert np.array_equal(d, g[f"vol{k}_wta"])
    r = O.variance_counts(total, g[f"vol{k}_lo"], g[f"vol{k}_hi"], d, 10.0, 0.25)
    assert np.array_equal(r, g[f"vol{k}_r"])


def test_intervals_checks_fusion():
    g = load_golden("intervals_checks_fusion")
    lo, hi = O.predicted_intervals(g["iv_d"], g["iv_p"], g["iv_valid"], 40)
    assert np.array_equal(lo, g["iv_lo"]) and np.array_equal(hi, g["iv_hi"])
    kl, kr = O.lr_masks(g["chk_dl"], g["chk_vl"], g["chk_dr"], g["chk_vr"], 1.0)
    assert np.array_equal(kl, g["chk_lr_l"]) and np.array_equal(kr, g["chk_lr_r"])
    for window, tau in ((3, 200.0), (5, 900.0)):
        sl = O.sad_masks(g["chk_left"], g["chk_right"], g["chk_dl"], g["chk_vl"], window, tau, "left")
        sr = O.sad_masks(g["chk_left"], g["chk_right"], g["chk_dr"], g["chk_vr"], window, tau, "right")
        assert np.array_equal(sl, g[f"chk_sad_l_w{window}"])
        assert np.array_equal(sr, g[f"chk_sad_r_w{window}"])
    vp, vm = g["fu_vp"], g["fu_vm"]
    d, p, v = O.kalman_fuse(np.where(vp, g["fu_dp"], 0), g["fu_pp"], vp,
                            np.where(vm, g["fu_dm"], 0), g["fu_rm"], vm, 1.0)
    assert np.array_equal(v, g["fu_v"])
    assert np.array_equal(d, g["fu_d"]) and np.array_equal(p, g["fu_p"])


def test_prediction():
    g = load_golden("prediction")
    f, b, cx, cy, w, h, d_max = g["rig"]
    for t in range(10):
        T = g[f"t{t}_T"]
        HL = O.homography(f, b, T)
        HR = O.homography(f, b, O.right_view_motion(b, T))
        assert np.array_equal(HL, g[f"t{t}_HL"]) and np.array_equal(HR, g[f"t{t}_HR"])
        d, p, v = g[f"t{t}_d"], g[f"t{t}_p"], g[f"t{t}_v"]
        edge = bool(g[f"t{t}_edge"])
        assert np.array_equal(O.edge_mask(d, v, 3.0, 1), g[f"t{t}_edges"])
        for tag, H in (("pl", HL), ("pr", HR)):
            od, op, ov = O.warp_view(d, p, v, H, cx, cy, d_max, 0.5, 3.0, 1, edge)
            assert np.array_equal(ov, g[f"t{t}_{tag}_v"]), (t, tag)
            np.testing.assert_allclose(od, g[f"t{t}_{tag}_d"], rtol=1e-12, atol=0)
            np.testing.assert_allclose(op, g[f"t{t}_{tag}_p"], rtol=1e-12, atol=0)
            if tag == "pl":
                fd, fp, fv = O.fill_holes(od, op, ov, 3.0, 0.5)
                assert np.array_equal(fv, g[f"t{t}_fl_v"])
                np.testing.assert_allclose(fd, g[f"t{t}_fl_d"], rtol=1e-12, atol=0)
                np.testing.assert_allclose(fp, g[f"t{t}_fl_p"], rtol=1e-12, atol=0)


def _check_sequence(name, params):
    g = load_golden(name)
    f, b, cx, cy, w, h, d_max = g["rig"]
    orc = O.OracleStereo(f, b, cx, cy, int(w), int(h), int(d_max), params)
    k = 0
    while f"f{k}_left" in g:
        motion = g[f"f{k}_motion"] if bool(g[f"f{k}_has_motion"]) else None
        out = orc.step(g[f"f{k}_left"], g[f"f{k}_right"], motion, keep_volumes=True)
        for v in ("l", "r"):
            view = "left" if v == "l" else "right"
            lo, hi = out[view + "_iv"]
            assert np.array_equal(lo, g[f"f{k}_{v}_lo"]) and np.array_equal(hi, g[f"f{k}_{v}_hi"])
            if f"f{k}_{v}_total" in g:
                assert np.array_equal(out[view + "_cost"], g[f"f{k}_{v}_cost"])
                assert np.array_equal(out[view + "_total"], g[f"f{k}_{v}_total"])
            dm, r, vm = out[view + "_meas"]
            assert np.array_equal(dm, g[f"f{k}_{v}_meas_d"])
            assert np.array_equal(vm, g[f"f{k}_{v}_meas_v"])
            assert np.array_equal(r, g[f"f{k}_{v}_meas_r"])
            assert np.array_equal(out[view + "_keep"], g[f"f{k}_{v}_keep"])
            for tag, got in (("pred", out[view + "_pred"]), ("fused", out[view + "_fused"])):
                assert np.array_equal(got[2], g[f"f{k}_{v}_{tag}_v"]), (k, v, tag)
                np.testing.assert_allclose(got[0], g[f"f{k}_{v}_{tag}_d"], rtol=1e-10, atol=0)
                np.testing.assert_allclose(got[1], g[f"f{k}_{v}_{tag}_p"], rtol=1e-10, atol=0)
        np.testing.assert_allclose([out["left_fraction"], out["right_fraction"]],
                                   g[f"f{k}_frac"], rtol=1e-15)
        k += 1
    assert k >= 2


def test_sequence_small():
    _check_sequence("seq_small", O.OracleParams())


def test_sequence_drive():
    _check_sequence("seq_drive", O.OracleParams(p1=8.0, p2=100.0))


def test_metrics():
    """metrics.py:39-117 restated, against the reference's own outputs
    (including exact |err| == 3 and |err| == 5 % threshold ties)."""
    g = load_golden("metrics")
    for case in range(4):
        est, ev, gt, gv = (g[f"c{case}_{k}"] for k in ("est", "ev", "gt", "gv"))
        assert float(ev.mean()) == float(g[f"c{case}_density"])
        for mode in ("or", "and"):
            assert np.array_equal(np.array(O.bad_rate(est, ev, gt, gv, mode)),
                                  g[f"c{case}_{mode}_rates"]), (case, mode)
            assert np.array_equal(O.bad_mask(est, ev, gt, gv, mode), g[f"c{case}_{mode}_mask"])
            assert np.array_equal(O.error_rgb(est, ev, gt, gv, mode), g[f"c{case}_{mode}_rgb"])


def test_render_boxes_matches_reference_synth():
    """The oracle's restated ray caster (the bench's port-fallback inputs)
    against synth.render_frame's own output (golden render.npz)."""
    from types import SimpleNamespace
    g = load_golden("render")
    f, b, cx, cy, w, h, d_max = g["rig"]
    cs = SimpleNamespace(rig=dict(f=f, b=b, cx=cx, cy=cy, width=int(w), height=int(h)),
                         poses=[g["pose0"], g["pose1"]], boxes=[g["boxes"]] * 2,
                         texture_scale=float(g["texture_scale"]),
                         texture_seed=int(g["texture_seed"]), background=int(g["background"]))
    for k in range(2):
        img = O.render_boxes(cs, k)
        assert np.array_equal(img[0], g[f"img{k}_l"]) and np.array_equal(img[1], g[f"img{k}_r"])
