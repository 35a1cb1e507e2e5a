"""Full-size golden digests of BASELINE.json configs 2-5 from the UNMODIFIED
reference (build container only; test infrastructure, never imported by the
product).

    python oracle/make_golden_configs.py [2] [3] [4] [5]

For every config the scenes come from ``paper_1708_06301_b200.scenes.
config_sequence`` (boxes, poses, motions, texture seed; config 3 adds three
independently moving boxes and 2% salt noise).  Each frame is rendered with
the reference's own ``synth.render_frame`` (/root/reference/pkg/src/egostereo/
synth.py:195-218) and fed to the reference's ``DisparityPipeline.
process_frame`` (pipeline.py:108-170) at the config's full size and length:

    config 2: 1242x375, D=128, 10 frames
    config 3: 1242x375, D=128, 100 frames, moving boxes + salt noise
    config 4: 2048x1024, D=256, frames 0-2 (a numpy frame takes minutes, ~10 GB)
    config 5: 1242x375, D=128, sequences 0, 9, ..., 63 of the 64-sequence batch,
              frames 0-4

A full FrameResult is ~14 maps per view per frame (GBs over a sequence), so
the fixture keeps compact digests: a SHA-256 of every map in a canonical dtype
(images, intervals, WTA disparities, validity / keep masks, matching
variance, predicted and fused float64 state), float64 row sums of the float
maps (a tolerance check if a hash ever differs), the search fractions, and at
a few frames the finite row / column / plane sums and hashes of the dense
cost and aggregated volumes.  The GPU tests (tests/test_gpu_full_configs.py)
render the same scenes on the device -- the image hashes prove the bytes are
identical -- and compare the device pipeline's digests with these.
"""

from __future__ import annotations

import hashlib
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")

# the jobs: config -> (sequences, frames, frames whose dense volumes are digested)
JOBS = {
    2: ([0], 10, (0, 1, 9)),
    3: ([0], 100, (1, 50, 99)),
    4: ([0], 3, (0, 1)),
    5: (list(range(0, 64, 9)), 5, (1,)),
}


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def canonical_maps(res_maps):
    """{name: canonical array} of one view; shared definition with the tests
    (tests/test_gpu_full_configs.py:_canonical)."""
    out = {}
    for name, a in res_maps.items():
        if name in ("lo", "hi"):
            out[name] = np.asarray(a).astype(np.int16)
        elif name == "meas_d":
            out[name] = np.asarray(a).astype(np.uint16)
        elif name.endswith("_v") or name == "keep":
            out[name] = np.asarray(a).astype(np.uint8)
        else:
            out[name] = np.asarray(a, dtype=np.float64)
    return out


FLOAT_MAPS = ("pred_d", "pred_p", "meas_r", "fused_d", "fused_p")


def view_maps(res, v):
    from egostereo import core  # noqa: F401
    L = v == "l"
    return {
        "pred_d": (res.predicted_left if L else res.predicted_right).values,
        "pred_v": (res.predicted_left if L else res.predicted_right).valid,
        "pred_p": (res.predicted_left_var if L else res.predicted_right_var).values,
        "lo": (res.intervals_left if L else res.intervals_right).lo,
        "hi": (res.intervals_left if L else res.intervals_right).hi,
        "meas_d": (res.measured_left if L else res.measured_right).values,
        "meas_v": (res.measured_left if L else res.measured_right).valid,
        "meas_r": (res.measured_left_var if L else res.measured_right_var).values,
        "keep": res.keep_left if L else res.keep_right,
        "fused_d": (res.fused.left if L else res.fused.right).values,
        "fused_v": (res.fused.left if L else res.fused.right).valid,
        "fused_p": (res.fused.left_var if L else res.fused.right_var).values,
    }


def volume_digest(data):
    fin = np.isfinite(data)
    c = np.where(fin, data, 0).astype(np.int64)
    return {"hash": digest(data.astype(np.float32)), "rowsum": c.sum(axis=(1, 2)),
            "colsum": c.sum(axis=(0, 2)), "dsum": c.sum(axis=(0, 1)),
            "finite": np.array(int(fin.sum()))}


def run_job(args):
    config, seq, n_frames, vol_frames = args
    sys.path.insert(0, REF)
    sys.path.insert(0, ROOT)
    from egostereo import core, pipeline, sgm, synth
    from paper_1708_06301_b200 import scenes
    cs = scenes.config_sequence(config, seq, n_frames=n_frames)
    rig = core.StereoRig(**cs.rig)
    pipe = pipeline.DisparityPipeline(rig)
    params = pipeline.PipelineParams()
    out = {"rig": np.array([rig.f, rig.b, rig.cx, rig.cy, rig.width, rig.height, rig.d_max]),
           "n_frames": np.array(n_frames), "seq": np.array(seq)}
    t_all = time.time()
    for k in range(n_frames):
        t0 = time.time()
        scene = synth.SceneSpec(rig=rig, primitives=[synth.Box(*map(float, b)) for b in cs.boxes[k]],
                                texture_seed=cs.texture_seed, texture_scale=cs.texture_scale,
                                background=cs.background)
        l, r, _, _ = synth.render_frame(scene, cs.poses[k])
        pair = np.stack([l.data, r.data])
        out[f"f{k}_img_hash"] = np.array(digest(pair))
        scenes.apply_salt(pair, cs, k)
        out[f"f{k}_in_hash"] = np.array(digest(pair))
        res = pipe.process_frame(core.GrayImage(pair[0]), core.GrayImage(pair[1]), cs.motions[k])
        out[f"f{k}_frac"] = np.array([res.search_fraction_left, res.search_fraction_right])
        for v in ("l", "r"):
            maps = canonical_maps(view_maps(res, v))
            for name, a in maps.items():
                out[f"f{k}_{v}_{name}_hash"] = np.array(digest(a))
            for name in FLOAT_MAPS:
                out[f"f{k}_{v}_{name}_rowsum"] = maps[name].sum(axis=1)
            out[f"f{k}_{v}_counts"] = np.array([int(maps["pred_v"].sum()), int(maps["meas_v"].sum()),
                                                int(maps["keep"].sum()), int(maps["fused_v"].sum())])
        if k in vol_frames:
            for v, iv in (("l", res.intervals_left), ("r", res.intervals_right)):
                view = "left" if v == "l" else "right"
                vol = sgm.matching_cost(core.GrayImage(pair[0]), core.GrayImage(pair[1]), iv,
                                        params.sgm, view)
                agg = sgm.aggregate_paths(vol, params.sgm)
                for tag, data in (("cost", vol.data), ("total", agg.data)):
                    for key, val in volume_digest(data).items():
                        out[f"f{k}_{v}_{tag}_{key}"] = val
                del vol, agg
        print(f"config {config} seq {seq} frame {k}: {time.time() - t0:.1f}s "
              f"frac=({res.search_fraction_left:.3f},{res.search_fraction_right:.3f})", flush=True)
    out["ref_seconds"] = np.array(time.time() - t_all)
    path = os.path.join(OUT, f"cfg{config}_s{seq}.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB)", flush=True)
    return path


if __name__ == "__main__":
    which = [int(a) for a in sys.argv[1:]] or [3, 4, 2, 5]
    jobs = []
    for c in which:
        seqs, n, vols = JOBS[c]
        jobs += [(c, s, n, vols) for s in seqs]
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    procs = int(os.environ.get("GOLDEN_PROCS", "7"))
    with mp.get_context("spawn").Pool(procs) as pool:
        for p in pool.imap_unordered(run_job, jobs):
            print("done", p, flush=True)
