"""Child process of tests/test_gpu_vd.py: with the aggregation schedule
chosen by ES_SGM_VD (read once per process), run a batch of sequences and
compare every sequence's aggregated cost volume (the sum of the partial
sums, both views) and WTA maps with the oracle (keep_volumes)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402


def main(width, height, d_max, B, frames):
    import bench
    from paper_1708_06301_b200 import core, pipeline, scenes
    rig = core.StereoRig(f=width * 0.6, b=0.54, cx=(width - 1) / 2.0, cy=height / 2.0,
                         width=width, height=height, d_max=d_max)
    specs = [scenes.sequence_spec(seed=700 + s, n_frames=frames, step=0.5, z_range=(4.0, 30.0))
             for s in range(B)]
    imgs = bench.render_frames(specs, list(range(frames)), "cuda:0", rig=rig)
    host = imgs.cpu().numpy()
    bp = pipeline.BatchedPipeline(rig, B)
    check = [0, B // 2, B - 1]
    orcs = {s: O.OracleStereo(rig.f, rig.b, rig.cx, rig.cy, width, height, d_max) for s in check}
    for k in range(frames):
        bp.process_frames(None, [sp[2][k] for sp in specs], sync=True, images_dev=imgs[k].data_ptr())
        for s in check:
            motion = specs[s][2][k]
            want = orcs[s].step(host[k, s, 0], host[k, s, 1], motion, keep_volumes=True)
            got = bp.result(s)
            for view, name in ((0, "left"), (1, "right")):
                assert np.array_equal(got.total_volume(view), want[name + "_total"]), (k, s, name)
                meas = got.measured_left if view == 0 else got.measured_right
                assert np.array_equal(meas.values, want[name + "_meas"][0]), (k, s, name)
    print("volumes ok", width, height, d_max, B, frames)


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:6]])
