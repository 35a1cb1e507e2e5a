"""Dump the search intervals (lo, hi) of a few bench-scene frames (both
views of sequence 0..n-1) to gpurun_out/meta.npz for offline analysis of the
aggregation's work distribution (lanes per chain, union waste)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
from paper_1708_06301_b200 import pipeline
from paper_1708_06301_b200.core import StereoRig

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
bench.use_config(cfg)
rig = StereoRig(**bench.RIG)
B = 2
specs = bench.sequence_specs(B, seed0=1000 * cfg)
frames = list(range(8))
imgs = bench.render_frames(specs, frames, "cuda:0")
bp = pipeline.BatchedPipeline(rig, B)
out = {}
for k in frames:
    bp.process_frames(None, bench.motions_for(specs, k), sync=True, images_dev=imgs[k].data_ptr())
    if k in (0, 3, 7):
        for s in range(B):
            r = bp.result(s)
            for v, iv in (("L", r.intervals_left), ("R", r.intervals_right)):
                out[f"f{k}_s{s}_{v}_lo"] = iv.lo.astype(np.int16)
                out[f"f{k}_s{s}_{v}_hi"] = iv.hi.astype(np.int16)
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed(f"gpurun_out/meta_c{cfg}.npz", **out)
print("saved", len(out))
