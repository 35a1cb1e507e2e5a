"""Generate golden vectors from the UNMODIFIED reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python oracle/make_golden.py

Imports ``egostereo`` from ``/root/reference/pkg/src`` (read-only), runs its
hot-path functions on seeded inputs and writes ``tests/golden/*.npz``.  The
reference cannot travel to the GPU box; these fixtures do.  Nothing here is
imported by the product or by the tests -- the tests only read the .npz files.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from egostereo import core, fusion, geometry, pipeline, prediction, sgm, synth  # noqa: E402
from paper_1708_06301_b200 import scenes  # noqa: E402


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB)")


def rig_small(width, height, d_max, f=None, b=0.5):
    f = f if f is not None else float(width)
    return core.StereoRig(f=f, b=b, cx=(width - 1) / 2.0, cy=(height - 1) / 2.0,
                          width=width, height=height, d_max=d_max)


def gen_cost_agg():
    """Cost, aggregation, WTA and variance on random inputs, both views."""
    out = {}
    rng = np.random.default_rng(7)
    for case, (h, w, d_max) in enumerate([(8, 12, 4), (13, 29, 11), (2, 40, 7), (24, 4, 2)]):
        left = rng.integers(0, 256, (h, w)).astype(np.uint8)
        right = rng.integers(0, 256, (h, w)).astype(np.uint8)
        lo = rng.integers(0, d_max, (h, w)).astype(np.int64)
        hi = np.minimum(lo + rng.integers(0, d_max + 1, (h, w)), d_max).astype(np.int64)
        if case == 0:
            lo[:] = 0
            hi[:] = d_max
        iv = sgm.IntervalMap(lo, hi, d_max)
        for window in (3, 5):
            prm = sgm.SgmParams(window=window)
            for view in ("left", "right"):
                vol = sgm.matching_cost(core.GrayImage(left), core.GrayImage(right), iv, prm, view)
                agg = sgm.aggregate_paths(vol, prm)
                disp = sgm.select_disparity(agg)
                var = sgm.matching_variance_map(agg, disp, prm)
                key = f"c{case}_w{window}_{view}"
                out[key + "_cost"] = vol.data
                out[key + "_total"] = agg.data
                out[key + "_wta"] = disp.values
                out[key + "_valid"] = disp.valid
                out[key + "_r"] = var.values
        out[f"c{case}_left"] = left
        out[f"c{case}_right"] = right
        out[f"c{case}_lo"] = lo
        out[f"c{case}_hi"] = hi
    # hand-built float volumes: integer and non-integer penalties
    for k, (p1, p2, D, integral) in enumerate([(1.0, 2.0, 3, True), (7.0, 86.0, 6, True),
                                               (1.5, 7.25, 5, False), (3.0, 40.0, 9, False)]):
        h, w = 6, 7
        if integral:
            C = rng.integers(0, 2000, (h, w, D)).astype(np.float32)
        else:
            C = (rng.random((h, w, D)) * 50.0).astype(np.float32)
        lo = rng.integers(0, D // 2 + 1, (h, w)).astype(np.int64)
        hi = np.minimum(lo + rng.integers(0, D, (h, w)), D - 1).astype(np.int64)
        ds = np.arange(D)
        C[(ds < lo[..., None]) | (ds > hi[..., None])] = np.inf
        prm = sgm.SgmParams(p1=p1, p2=p2)
        agg = sgm.aggregate_paths(sgm.CostVolume(C, sgm.IntervalMap(lo, hi, D - 1)), prm)
        disp = sgm.select_disparity(agg)
        var = sgm.matching_variance_map(agg, disp, prm)
        out[f"vol{k}_cost"] = C
        out[f"vol{k}_lo"] = lo
        out[f"vol{k}_hi"] = hi
        out[f"vol{k}_p"] = np.array([p1, p2])
        out[f"vol{k}_total"] = agg.data
        out[f"vol{k}_wta"] = disp.values
        out[f"vol{k}_r"] = var.values
    save("cost_agg", **out)


def gen_intervals_checks_fusion():
    out = {}
    rng = np.random.default_rng(11)
    h, w, d_max = 20, 53, 40
    rig = rig_small(w, h, d_max)
    d = rng.uniform(-2.0, d_max + 3.0, (h, w))
    mask = rng.random((h, w)) < 0.1
    d[mask] = np.round(d[mask]) + 0.5 * (rng.random(mask.sum()) < 0.5)
    p = rng.uniform(-0.5, 30.0, (h, w)) ** 2 / 30.0
    p[rng.random((h, w)) < 0.2] = 0.0
    valid = rng.random((h, w)) < 0.8
    iv = sgm.search_intervals(core.DisparityMap(d, valid), core.VarianceMap(p), rig)
    out.update(iv_d=d, iv_p=p, iv_valid=valid, iv_lo=iv.lo, iv_hi=iv.hi)

    # LR and SAD checks on random integer and fractional maps
    left = rng.integers(0, 256, (h, w)).astype(np.uint8)
    right = np.roll(left, -5, axis=1)
    right[:, -5:] = rng.integers(0, 256, (h, 5))
    dl = rng.integers(0, 12, (h, w)).astype(np.float64)
    dr = rng.integers(0, 12, (h, w)).astype(np.float64)
    dl[rng.random((h, w)) < 0.5] = 5.0
    dr[rng.random((h, w)) < 0.5] = 5.0
    dr += np.where(rng.random((h, w)) < 0.3, rng.uniform(-1.5, 1.5, (h, w)), 0.0)
    vl = (dl > 0) & (rng.random((h, w)) < 0.9)
    vr = (dr > 0) & (rng.random((h, w)) < 0.9)
    ml, mr = core.DisparityMap(dl, vl), core.DisparityMap(dr, vr)
    kl, kr = sgm.lr_consistency(ml, mr, 1.0)
    out.update(chk_left=left, chk_right=right, chk_dl=dl, chk_dr=dr, chk_vl=vl,
               chk_vr=vr, chk_lr_l=kl, chk_lr_r=kr)
    for window, tau in ((3, 200.0), (5, 900.0)):
        out[f"chk_sad_l_w{window}"] = sgm.sad_check(core.GrayImage(left), core.GrayImage(right),
                                                    ml, window, tau, "left")
        out[f"chk_sad_r_w{window}"] = sgm.sad_check(core.GrayImage(left), core.GrayImage(right),
                                                    mr, window, tau, "right")

    # Kalman update
    dp = rng.uniform(0.5, 60.0, (h, w))
    pp = rng.uniform(0.01, 9.0, (h, w))
    vp = rng.random((h, w)) < 0.6
    dm = rng.integers(1, 64, (h, w)).astype(np.float64)
    rm = np.maximum(rng.integers(0, 6, (h, w)).astype(np.float64), 0.25)
    vm = rng.random((h, w)) < 0.6
    fd, fp = fusion.fuse_maps(core.DisparityMap(np.where(vp, dp, 0), vp), core.VarianceMap(pp),
                              core.DisparityMap(np.where(vm, dm, 0), vm), core.VarianceMap(rm),
                              fusion.FusionParams(p_init=1.0))
    out.update(fu_dp=dp, fu_pp=pp, fu_vp=vp, fu_dm=dm, fu_rm=rm, fu_vm=vm,
               fu_d=fd.values, fu_p=fp.values, fu_v=fd.valid)
    save("intervals_checks_fusion", **out)


def gen_prediction():
    """predict_maps (+ fill) on random states under random rigid motions."""
    from scipy.spatial.transform import Rotation
    out = {}
    rng = np.random.default_rng(42)
    rig = rig_small(48, 24, 20, f=48.0, b=0.5)
    out["rig"] = np.array([rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max])
    for t in range(10):
        h, w = rig.shape
        valid = rng.random((h, w)) < 0.75
        base = rng.uniform(1.0, 16.0)
        vals = base + 0.05 * np.arange(w)[None, :] + rng.normal(0, 0.3, (h, w))
        # add a couple of depth discontinuities for edge rejection
        vals[:, w // 3: w // 2] += 6.0
        vals = np.clip(vals, 0.6, rig.d_max - 0.5)
        vals = np.where(valid, vals, 0.0)
        var = np.where(valid, rng.uniform(0.05, 3.0, (h, w)), 0.0)
        if t == 0:
            T = np.eye(4)
        else:
            R = Rotation.from_rotvec(rng.normal(0, 0.02, 3)).as_matrix()
            T = core.make_motion(R, rng.normal(0, 0.15, 3) + np.array([0, 0, -0.2 * (t % 3)]))
        prm = prediction.PredictionParams(edge_reject=(t % 4 != 3))
        dm = core.DisparityMap(vals, valid)
        vm = core.VarianceMap(var)
        state = core.FilterState(dm, vm, dm.copy(), vm.copy(), 0)
        pr = prediction.predict_maps(state, T, rig, prm)
        fl_d, fl_p = prediction.fill_zoom_holes(pr.left, pr.left_var, prm.gamma_f, prm.q)
        out[f"t{t}_d"] = vals
        out[f"t{t}_p"] = var
        out[f"t{t}_v"] = valid
        out[f"t{t}_T"] = T
        out[f"t{t}_edge"] = np.array(prm.edge_reject)
        out[f"t{t}_HL"] = geometry.disparity_homography(rig, T)
        out[f"t{t}_HR"] = geometry.disparity_homography(rig, geometry.right_motion(rig, T))
        out[f"t{t}_pl_d"] = pr.left.values
        out[f"t{t}_pl_p"] = pr.left_var.values
        out[f"t{t}_pl_v"] = pr.left.valid
        out[f"t{t}_pr_d"] = pr.right.values
        out[f"t{t}_pr_p"] = pr.right_var.values
        out[f"t{t}_pr_v"] = pr.right.valid
        out[f"t{t}_fl_d"] = fl_d.values
        out[f"t{t}_fl_p"] = fl_p.values
        out[f"t{t}_fl_v"] = fl_d.valid
        out[f"t{t}_edges"] = prediction.reject_edges(dm, prm.gamma_e, prm.edge_window)
    save("prediction", **out)


def _run_sequence_golden(name, rig, frames, motions, params, vol_frames=()):
    pipe = pipeline.DisparityPipeline(rig, params)
    out = {"rig": np.array([rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max])}
    for k, (left, right) in enumerate(frames):
        t0 = time.time()
        res = pipe.process_frame(core.GrayImage(left), core.GrayImage(right), motions[k])
        out[f"f{k}_left"] = left
        out[f"f{k}_right"] = right
        out[f"f{k}_motion"] = np.eye(4) if motions[k] is None else motions[k]
        out[f"f{k}_has_motion"] = np.array(motions[k] is not None)
        for v, pd, pv, iv, md, mv, kp, fd, fv in (
            ("l", res.predicted_left, res.predicted_left_var, res.intervals_left,
             res.measured_left, res.measured_left_var, res.keep_left, res.fused.left,
             res.fused.left_var),
            ("r", res.predicted_right, res.predicted_right_var, res.intervals_right,
             res.measured_right, res.measured_right_var, res.keep_right, res.fused.right,
             res.fused.right_var),
        ):
            out[f"f{k}_{v}_pred_d"] = pd.values
            out[f"f{k}_{v}_pred_p"] = pv.values
            out[f"f{k}_{v}_pred_v"] = pd.valid
            out[f"f{k}_{v}_lo"] = iv.lo.astype(np.int16)
            out[f"f{k}_{v}_hi"] = iv.hi.astype(np.int16)
            out[f"f{k}_{v}_meas_d"] = md.values
            out[f"f{k}_{v}_meas_v"] = md.valid
            out[f"f{k}_{v}_meas_r"] = mv.values
            out[f"f{k}_{v}_keep"] = kp
            out[f"f{k}_{v}_fused_d"] = fd.values
            out[f"f{k}_{v}_fused_p"] = fv.values
            out[f"f{k}_{v}_fused_v"] = fd.valid
        out[f"f{k}_frac"] = np.array([res.search_fraction_left, res.search_fraction_right])
        if k in vol_frames:
            for v in ("left", "right"):
                iv = res.intervals_left if v == "left" else res.intervals_right
                vol = sgm.matching_cost(core.GrayImage(left), core.GrayImage(right), iv,
                                        params.sgm, v)
                agg = sgm.aggregate_paths(vol, params.sgm)
                out[f"f{k}_{v[0]}_cost"] = vol.data
                out[f"f{k}_{v[0]}_total"] = agg.data
        print(f"  {name} frame {k}: {time.time() - t0:.1f}s "
              f"frac=({res.search_fraction_left:.3f},{res.search_fraction_right:.3f})")
    save(name, **out)


def gen_sequences():
    # small rendered sequence (reference synth) with noisy ego-motion
    rig = rig_small(96, 48, 24, f=64.0, b=0.5)
    scene = synth.SceneSpec(
        rig=rig,
        primitives=(synth.Plane(z=5.0),
                    synth.Plane(z=3.0, x0=-1.2, x1=0.1, y0=-0.9, y1=0.3),
                    synth.Box(x0=0.2, x1=1.0, y0=-0.2, y1=0.7, z0=1.9, z1=2.4)),
        texture_seed=3,
    )
    traj = synth.dolly_trajectory(5, -0.08)
    frames = synth.make_sequence(scene, traj, sigma_rot_deg=0.05, sigma_trans=0.005, seed=5)
    _run_sequence_golden(
        "seq_small", rig, [(f.left.data, f.right.data) for f in frames],
        [f.motion_noisy for f in frames], pipeline.PipelineParams(), vol_frames=(0, 1, 3))

    # forward-driving sequence with the bench scene model, smaller rig
    rig = core.StereoRig(f=180.0, b=0.54, cx=151.0, cy=46.0, width=310, height=94, d_max=40)
    boxes, poses, motions = scenes.sequence_spec(seed=77, n_frames=4, step=0.5,
                                                 z_range=(4.0, 30.0))
    prims = [synth.Box(*map(float, bx)) for bx in boxes]
    scene = synth.SceneSpec(rig=rig, primitives=prims, texture_seed=9, texture_scale=0.05)
    imgs = []
    for pose in poses:
        l, r, _, _ = synth.render_frame(scene, pose)
        imgs.append((l.data, r.data))
    params = pipeline.PipelineParams(sgm=sgm.SgmParams(p1=8.0, p2=100.0))
    _run_sequence_golden("seq_drive", rig, imgs, motions, params)
    # record the scene so the device renderer can be pinned against synth
    out = {"rig": np.array([rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max]),
           "boxes": boxes, "texture_seed": np.array(9), "texture_scale": np.array(0.05),
           "background": np.array(12)}
    for k, pose in enumerate(poses[:2]):
        l, r, gl, gr = synth.render_frame(scene, pose)
        out[f"pose{k}"] = pose
        out[f"img{k}_l"] = l.data
        out[f"img{k}_r"] = r.data
        out[f"gt{k}_l"] = gl.values
        out[f"gt{k}_r"] = gr.values
    save("render", **out)


def prim_records(primitives):
    """synth primitives -> the device renderer's [n][8] records
    (include/egostereo_b200.h es_render_prims)."""
    out = []
    for p in primitives:
        if isinstance(p, synth.Plane):
            flags = sum(1 << i for i, b in enumerate((p.x0, p.x1, p.y0, p.y1)) if b is not None)
            out.append([1.0, p.z] + [0.0 if b is None else b for b in (p.x0, p.x1, p.y0, p.y1)]
                       + [0.0, float(flags)])
        else:
            out.append([0.0, p.x0, p.x1, p.y0, p.y1, p.z0, p.z1, 0.0])
    return np.asarray(out, np.float64)


def gen_render_planes():
    """synth.render_frame on scenes mixing bounded / unbounded fronto-parallel
    planes and boxes, under rotated poses, both views: the device renderer
    must reproduce the images and ground truth bit for bit."""
    from scipy.spatial.transform import Rotation
    out = {}
    rng = np.random.default_rng(23)
    for case, (w, h, f) in enumerate([(96, 48, 64.0), (161, 77, 120.0), (310, 94, 180.0)]):
        rig = rig_small(w, h, min(w - 1, 60), f=f, b=0.5)
        prims = [synth.Plane(z=9.0),
                 synth.Plane(z=4.0, x0=-1.0, x1=0.4, y0=None, y1=0.6),
                 synth.Plane(z=3.0, x0=None, x1=-0.5, y0=-0.8, y1=None),
                 synth.Box(x0=0.2, x1=1.1, y0=-0.3, y1=0.7, z0=2.2, z1=2.9),
                 synth.Box(x0=-2.0, x1=2.0, y0=0.9, y1=1.0, z0=1.0, z1=8.0)]
        scene = synth.SceneSpec(rig=rig, primitives=prims, texture_seed=40 + case,
                                texture_scale=[None, 0.03, 0.05][case])
        for k in range(2):
            R = Rotation.from_rotvec(rng.normal(0, 0.03, 3)).as_matrix()
            pose = core.make_motion(R, rng.normal(0, 0.1, 3))
            l, r, gl, gr = synth.render_frame(scene, pose)
            out[f"c{case}_f{k}_pose"] = pose
            out[f"c{case}_f{k}_img"] = np.stack([l.data, r.data])
            out[f"c{case}_f{k}_gt"] = np.stack([gl.values, gr.values])
        out[f"c{case}_rig"] = np.array([rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height,
                                        rig.d_max])
        out[f"c{case}_prims"] = prim_records(prims)
        out[f"c{case}_seed"] = np.array(scene.texture_seed)
        out[f"c{case}_scale"] = np.array(scene.texture_scale)
    save("render_planes", **out)


def gen_config1():
    """Config 1 at full size (1242x375, D=128): compact reference outputs."""
    left, right, gt = scenes.config1_pair(seed=1000)
    rig = core.StereoRig(f=718.9, b=0.54, cx=607.0, cy=185.0, width=1242, height=375,
                         d_max=127)
    prm = sgm.SgmParams()
    iv = sgm.full_range_intervals(rig)
    out = {"left": left, "right": right}
    meas = {}
    for v in ("left", "right"):
        t0 = time.time()
        vol = sgm.matching_cost(core.GrayImage(left), core.GrayImage(right), iv, prm, v)
        agg = sgm.aggregate_paths(vol, prm)
        disp = sgm.select_disparity(agg)
        var = sgm.matching_variance_map(agg, disp, prm)
        c = vol.data.astype(np.int64)
        s = agg.data.astype(np.int64)
        out[f"{v}_cost_rowsum"] = c.sum(axis=(1, 2))
        out[f"{v}_total_rowsum"] = s.sum(axis=(1, 2))
        out[f"{v}_total_rowsum_sq"] = (s * s).sum(axis=(1, 2))
        out[f"{v}_cost_colsum"] = c.sum(axis=(0, 2))
        out[f"{v}_total_colsum"] = s.sum(axis=(0, 2))
        out[f"{v}_total_dsum"] = s.sum(axis=(0, 1))
        rows = np.array([0, 187, 374])
        out[f"{v}_total_rows"] = agg.data[rows].astype(np.uint16)
        out[f"{v}_cost_rows"] = vol.data[rows].astype(np.uint16)
        out[f"{v}_wta"] = disp.values.astype(np.uint8)
        out[f"{v}_r"] = var.values.astype(np.float32)
        meas[v] = disp
        print(f"  config1 {v}: {time.time() - t0:.1f}s")
    kl, kr = sgm.lr_consistency(meas["left"], meas["right"], prm.tau_lr)
    kl &= sgm.sad_check(core.GrayImage(left), core.GrayImage(right), meas["left"], 3, 200.0, "left")
    kr &= sgm.sad_check(core.GrayImage(left), core.GrayImage(right), meas["right"], 3, 200.0, "right")
    out["keep_left"] = np.packbits(kl)
    out["keep_right"] = np.packbits(kr)
    save("config1", **out)


def gen_metrics():
    """Evaluation metrics (metrics.py) on seeded maps, and the reference's
    run_sequence output tree (metrics.txt, summary.txt, disp_0 / err_0
    arrays) for a small rendered sequence with ground truth."""
    from egostereo import metrics
    import tempfile

    import cv2
    out = {}
    rng = np.random.default_rng(11)
    for case, (h, w) in enumerate([(7, 9), (31, 45), (64, 3), (5, 5)]):
        gt = rng.uniform(0.5, 60.0, (h, w))
        gv = rng.random((h, w)) < 0.7
        est = gt + rng.normal(0.0, 2.5, (h, w)) * (rng.random((h, w)) < 0.6)
        # exact threshold ties: |err| == 3 and |err| == 0.05 * gt
        est.flat[::7] = gt.flat[::7] + 3.0
        est.flat[1::11] = gt.flat[1::11] * 1.05
        ev = rng.random((h, w)) < 0.8
        if case == 3:
            gv[:] = False
        gt = np.where(gv, gt, 0.0)
        est = np.where(ev, est, 0.0)
        e, t = core.DisparityMap(est, ev), core.DisparityMap(gt, gv)
        out[f"c{case}_est"], out[f"c{case}_ev"] = est, ev
        out[f"c{case}_gt"], out[f"c{case}_gv"] = gt, gv
        out[f"c{case}_density"] = np.array(metrics.density(e))
        for mode in ("or", "and"):
            r = metrics.bad_pixel_rate(e, t, mode)
            out[f"c{case}_{mode}_rates"] = np.array([r.rate, r.rate_all, r.density])
            out[f"c{case}_{mode}_mask"] = metrics.bad_pixel_mask(e, t, mode)
            out[f"c{case}_{mode}_rgb"] = metrics.error_image(e, t, mode)
    save("metrics", **out)

    # run_sequence over a small rendered sequence with ground truth
    rig = rig_small(64, 40, 16, f=48.0, b=0.5)
    scene = synth.SceneSpec(
        rig=rig,
        primitives=(synth.Plane(z=4.0),
                    synth.Box(x0=-0.6, x1=0.3, y0=-0.4, y1=0.5, z0=2.0, z1=2.5)),
        texture_seed=4,
    )
    traj = synth.dolly_trajectory(3, -0.06)
    frames = synth.make_sequence(scene, traj, sigma_rot_deg=0.05, sigma_trans=0.005, seed=6)
    seq = pipeline.Sequence(rig, [f.left for f in frames], [f.right for f in frames],
                            [f.motion_noisy for f in frames],
                            gt_left=[f.gt_left for f in frames],
                            gt_right=[f.gt_right for f in frames])
    out = {"rig": np.array([rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max])}
    for k, f in enumerate(frames):
        out[f"f{k}_left"], out[f"f{k}_right"] = f.left.data, f.right.data
        out[f"f{k}_motion"] = np.eye(4) if f.motion_noisy is None else f.motion_noisy
        out[f"f{k}_has_motion"] = np.array(f.motion_noisy is not None)
        out[f"f{k}_gt_d"], out[f"f{k}_gt_v"] = f.gt_left.values, f.gt_left.valid
        out[f"f{k}_gtr_d"], out[f"f{k}_gtr_v"] = f.gt_right.values, f.gt_right.valid
    with tempfile.TemporaryDirectory() as tmp:
        pipeline.run_sequence(seq, out_dir=tmp, metric_mode="or")
        out["metrics_txt"] = np.array(open(os.path.join(tmp, "metrics.txt")).read())
        out["summary_txt"] = np.array(open(os.path.join(tmp, "summary.txt")).read())
        for k in range(len(frames)):
            out[f"f{k}_disp_png"] = cv2.imread(os.path.join(tmp, "disp_0", f"{k:06d}.png"),
                                               cv2.IMREAD_UNCHANGED)
            out[f"f{k}_err_png"] = cv2.imread(os.path.join(tmp, "err_0", f"{k:06d}.png"),
                                              cv2.IMREAD_UNCHANGED)
    save("run_sequence", **out)


def gen_acceptance():
    """Reference acceptance criteria on their own scenes: criterion 3 (10
    rendered 32x32 scenes, full-range matcher == the independent brute-force
    SGM of tests/reference_sgm.py) and criterion 4 (a 256x128 dolly-out
    sequence: per-frame search fractions and the fused maps)."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    import helpers
    import reference_sgm
    out = {}
    rig = helpers.make_rig(width=32, height=32, f=64.0, b=0.5, d_max=16)
    prm = sgm.SgmParams()
    for seed in range(10):
        left, right, _, _ = synth.render_frame(helpers.small_scene(rig, texture_seed=seed), np.eye(4))
        w, v = reference_sgm.match(left.data, right.data, rig.d_max, prm.window, prm.p1, prm.p2)
        disp = sgm.select_disparity(sgm.aggregate_paths(
            sgm.matching_cost(left, right, sgm.full_range_intervals(rig), prm), prm))
        assert np.array_equal(disp.valid, v)
        out[f"c3_{seed}_left"], out[f"c3_{seed}_right"] = left.data, right.data
        out[f"c3_{seed}_winners"], out[f"c3_{seed}_valid"] = np.asarray(w), np.asarray(v)
    rig = helpers.make_rig()   # 256x128, d_max = 64
    frames = helpers.recede_sequence(rig, 10, step=0.1, texture_seed=7)
    seq = pipeline.Sequence(rig=rig, lefts=[f.left for f in frames],
                            rights=[f.right for f in frames],
                            motions=[f.motion_exact for f in frames])
    res = pipeline.run_sequence(seq, pipeline.PipelineParams())
    for k, f in enumerate(frames):
        out[f"c4_{k}_left"], out[f"c4_{k}_right"] = f.left.data, f.right.data
        out[f"c4_{k}_motion"] = np.eye(4) if f.motion_exact is None else f.motion_exact
        out[f"c4_{k}_fused_d"] = res[k].fused.left.values
        out[f"c4_{k}_fused_v"] = res[k].fused.left.valid
        for v, gt in (("l", f.gt_left), ("r", f.gt_right)):
            out[f"c4_{k}_gt{v}_d"], out[f"c4_{k}_gt{v}_v"] = gt.values, gt.valid
    out["c4_fractions"] = np.array([r.search_fraction_left for r in res])
    save("acceptance", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["cost_agg", "misc", "prediction", "sequences", "config1", "metrics", "acceptance", "render_planes"]
    if "cost_agg" in which:
        gen_cost_agg()
    if "misc" in which:
        gen_intervals_checks_fusion()
    if "prediction" in which:
        gen_prediction()
    if "sequences" in which:
        gen_sequences()
    if "config1" in which:
        gen_config1()
    if "metrics" in which:
        gen_metrics()
    if "acceptance" in which:
        gen_acceptance()
    if "render_planes" in which:
        gen_render_planes()
