"""Experiment: the B=64 step as one context vs two B=32 contexts stepped
alternately on their own streams (does stage overlap between independent
sub-batches help?).  Host wall clock around a device sync; A/B only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1708_06301_b200 import pipeline
from paper_1708_06301_b200.core import StereoRig

rig = StereoRig(**bench.RIG)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
K, Wm = 8, 3
nctx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
specs = bench.sequence_specs(B, seed0=1000)
imgs = bench.render_frames(specs, list(range(Wm + K)), "cuda:0")
per = B // nctx
bps = [pipeline.BatchedPipeline(rig, per) for _ in range(nctx)]
sub = [specs[i * per:(i + 1) * per] for i in range(nctx)]
for k in range(Wm):
    for i, bp in enumerate(bps):
        bp.process_frames(None, bench.motions_for(sub[i], k), sync=True,
                          images_dev=imgs[k, i * per].data_ptr())
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(K):
    k = Wm + s
    for i, bp in enumerate(bps):
        bp.process_frames(None, bench.motions_for(sub[i], k), sync=False,
                          images_dev=imgs[k, i * per].data_ptr())
for bp in bps:
    bp.sync()
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"contexts={nctx} B={B}: {B * K / dt:.1f} frames/s ({dt / K * 1e3:.2f} ms/step)")
