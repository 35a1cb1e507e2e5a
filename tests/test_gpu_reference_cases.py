"""The reference's own known-answer cases for prediction and fusion
(pkg/tests/test_prediction.py, test_fusion.py, test_acceptance.py
criterion 2), restated as scenarios and run through the device stage
functions.  Expected values follow from the reference's semantics:
warp (x, y, d) -> (x - d, y, d) for a camera step of +b along x, the
largest warped disparity wins a collision, predicted variance = p + q under
a pure translation, strict hole-fill threshold, and the Kalman update's
adopt / blend / drop table."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rig(w, h, d_max, f=None):
    from paper_1708_06301_b200 import core
    f = float(w) if f is None else f
    return core.StereoRig(f=f, b=0.5, cx=(w - 1) / 2.0, cy=(h - 1) / 2.0, width=w, height=h,
                          d_max=d_max)


def _state(values, valid, var):
    from paper_1708_06301_b200 import core
    d = core.DisparityMap(np.where(valid, values, 0.0), valid)
    p = core.VarianceMap(np.where(valid, var, 0.0))
    return core.FilterState(d, p, d.copy(), p.copy())


def _predict(state, T, rig, **kw):
    from paper_1708_06301_b200 import prediction
    return prediction.predict_maps(state, T, rig, prediction.PredictionParams(**kw))


def test_translation_by_baseline_shifts_left_by_disparity():
    from paper_1708_06301_b200 import core
    rig = _rig(16, 4, 6)
    shp = (rig.height, rig.width)
    out = _predict(_state(np.full(shp, 4.0), np.ones(shp, bool), np.ones(shp)),
                   core.make_motion(t=(-rig.b, 0.0, 0.0)), rig, q=0.5, edge_reject=False,
                   fill_holes=False)
    assert out.left.valid[:, :12].all() and not out.left.valid[:, 12:].any()
    np.testing.assert_allclose(out.left.values[:, :12], 4.0, atol=1e-12)
    np.testing.assert_allclose(out.left_var.values[:, :12], 1.5, atol=1e-12)


def test_collision_keeps_the_nearer_source():
    from paper_1708_06301_b200 import core
    rig = _rig(16, 4, 6)
    shp = (rig.height, rig.width)
    values, valid, var = np.zeros(shp), np.zeros(shp, bool), np.zeros(shp)
    values[1, 3], var[1, 3], valid[1, 3] = 3.0, 1.0, True    # lands on x = 0
    values[1, 4], var[1, 4], valid[1, 4] = 4.0, 2.0, True    # lands on x = 0, nearer
    out = _predict(_state(values, valid, var), core.make_motion(t=(-rig.b, 0.0, 0.0)), rig,
                   q=0.5, edge_reject=False, fill_holes=False)
    assert out.left.valid[1, 0]
    assert abs(out.left.values[1, 0] - 4.0) < 1e-12 and abs(out.left_var.values[1, 0] - 2.5) < 1e-12


def test_targets_outside_the_image_are_dropped():
    from paper_1708_06301_b200 import core
    rig = _rig(16, 4, 8)
    shp = (rig.height, rig.width)
    out = _predict(_state(np.full(shp, 8.0), np.ones(shp, bool), np.ones(shp)),
                   core.make_motion(t=(-rig.b, 0.0, 0.0)), rig, edge_reject=False,
                   fill_holes=False)
    assert out.left.valid[:, :8].all() and not out.left.valid[:, 8:].any()


def test_edge_rejection_before_warping_and_edge_map():
    from paper_1708_06301_b200 import core, prediction
    rig = _rig(16, 4, 8)
    shp = (rig.height, rig.width)
    values = np.full(shp, 2.0)
    values[:, 8:] = 7.0
    out = _predict(_state(values, np.ones(shp, bool), np.ones(shp)), np.eye(4), rig, q=0.0,
                   gamma_e=3.0, edge_window=1, edge_reject=True, fill_holes=False)
    assert not out.left.valid[:, 7:9].any()
    assert out.left.valid[:, :7].all() and out.left.valid[:, 9:].all()
    # a 10-high step between columns 2 and 3: exactly those two columns
    v = np.full((3, 7), 10.0)
    v[:, 3:] = 20.0
    want = np.zeros((3, 7), bool)
    want[:, 2:4] = True
    assert np.array_equal(prediction.reject_edges(core.DisparityMap(v, np.ones((3, 7), bool)), 3.0, 1), want)
    # an invalid neighbour does not count
    v = np.full((3, 5), 10.0)
    ok = np.ones((3, 5), bool)
    ok[1, 2] = False
    rej = prediction.reject_edges(core.DisparityMap(np.where(ok, v, 0.0), ok), 3.0, 1)
    assert not rej[ok].any()


def test_zoom_hole_fill_known_answer():
    from paper_1708_06301_b200 import core, prediction
    d, p, v = np.zeros((5, 7)), np.zeros((5, 7)), np.zeros((5, 7), bool)
    for (y, x, val, var) in ((0, 2, 10.0, 1.0), (0, 3, 8.0, 1.0), (0, 6, 8.0, 1.0),
                             (2, 1, 10.0, 1.0), (2, 3, 11.0, 2.0), (4, 0, 5.0, 1.0),
                             (4, 2, 15.0, 1.0)):
        d[y, x], p[y, x], v[y, x] = val, var, True
    disp, var = prediction.fill_zoom_holes(core.DisparityMap(d, v), core.VarianceMap(p), 3.0, 0.5)
    # horizontal pass fills (2,2) = (10 + 11)/2 with max variance + q; the
    # vertical pass then sees it: (1,2) = (10 + 10.5)/2, variance 2.5 + q
    assert disp.valid[2, 2] and disp.values[2, 2] == 10.5 and var.values[2, 2] == 2.5
    assert disp.valid[1, 2] and disp.values[1, 2] == 10.25 and var.values[1, 2] == 3.0
    # |8 - 11| == gamma_f is not filled (strict); wide and steep gaps stay open
    assert not disp.valid[1, 3] and not disp.valid[0, 4] and not disp.valid[0, 5]
    assert not disp.valid[4, 1] and not disp.valid[3, 2]
    assert disp.values[0, 2] == 10.0 and var.values[0, 2] == 1.0
    assert disp.valid.sum() == 9


def test_identity_motion_is_a_fixed_point_over_100_fuzzed_states():
    from paper_1708_06301_b200 import core, prediction
    rig = _rig(24, 12, 10)
    rng = np.random.default_rng(42)
    prm = prediction.PredictionParams(q=0.0, edge_reject=False, fill_holes=False)
    for _ in range(100):
        valid = rng.random(rig.shape) < rng.uniform(0.2, 0.95)
        values = np.where(valid, rng.uniform(0.5, 10.0, rig.shape), 0.0)
        var = np.where(valid, rng.uniform(0.01, 9.0, rig.shape), 0.0)
        st = _state(values, valid, var)
        out = prediction.predict_maps(st, np.eye(4), rig, prm)
        for a, b in ((out.left, st.left), (out.right, st.right)):
            assert np.array_equal(a.values, b.values) and np.array_equal(a.valid, b.valid)
        assert np.array_equal(out.left_var.values, var) and np.array_equal(out.right_var.values, var)


def test_kalman_update_case_table_contraction_and_convergence():
    from paper_1708_06301_b200 import core, fusion
    m = lambda v, ok: core.DisparityMap(np.asarray([v], float), np.asarray([ok], bool))   # noqa: E731
    r = lambda v: core.VarianceMap(np.asarray([v], float))                              # noqa: E731
    fd, fp = fusion.fuse_maps(m([10.0, 0.0, 9.0, 0.0], [1, 0, 1, 0]), r([4.0, 0.0, 1.0, 0.0]),
                              m([12.0, 7.0, 0.0, 0.0], [1, 1, 0, 0]), r([4.0, 2.0, 0.0, 0.0]),
                              fusion.FusionParams(p_init=1.0))
    assert fd.valid.tolist() == [[True, True, False, False]]
    assert fd.values[0, 0] == 11.0 and fp.values[0, 0] == 2.0        # blended
    assert fd.values[0, 1] == 7.0 and fp.values[0, 1] == 1.0         # adopted at p_init
    rng = np.random.default_rng(17)
    n = 500
    p, rv = rng.uniform(0.01, 10.0, (1, n)), rng.uniform(0.01, 10.0, (1, n))
    dp, dm = rng.uniform(1.0, 50.0, (1, n)), rng.uniform(1.0, 50.0, (1, n))
    ones = np.ones((1, n), bool)
    fd, fp = fusion.fuse_maps(core.DisparityMap(dp, ones), core.VarianceMap(p),
                              core.DisparityMap(dm, ones), core.VarianceMap(rv), fusion.FusionParams())
    assert (fp.values <= np.minimum(p, rv)).all()
    assert (fd.values >= np.minimum(dp, dm)).all() and (fd.values <= np.maximum(dp, dm)).all()
    d, pv = np.array([[10.0]]), np.array([[4.0]])
    for _ in range(50):
        fd, fp = fusion.fuse_maps(core.DisparityMap(d, np.ones((1, 1), bool)), core.VarianceMap(pv),
                                  core.DisparityMap(np.array([[14.0]]), np.ones((1, 1), bool)),
                                  core.VarianceMap(np.array([[1.0]])), fusion.FusionParams())
        d, pv = fd.values, fp.values
    assert abs(d[0, 0] - 14.0) < 0.05 and pv[0, 0] < 0.05
