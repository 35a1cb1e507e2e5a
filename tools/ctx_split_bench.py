"""Experiment: a batch stepped as contexts of the given (possibly unequal)
sizes, each told the whole batch (es_ctx_shared_batch); host wall clock
around a device sync, A/B only.  usage: ctx_split_bench.py 16,16,16,16"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1708_06301_b200 import _lib, pipeline
from paper_1708_06301_b200.core import StereoRig

rig = StereoRig(**bench.RIG)
sizes = [int(x) for x in sys.argv[1].split(",")]
B = sum(sizes)
K, Wm = 8, 3
specs = bench.sequence_specs(B, seed0=1000)
imgs = bench.render_frames(specs, list(range(Wm + K)), "cuda:0")
offs = [sum(sizes[:i]) for i in range(len(sizes))]
bps = [pipeline.BatchedPipeline(rig, n, groups=1) for n in sizes]
for bp in bps:
    _lib.call("es_ctx_shared_batch", bp.engines[0]._h, B)
sub = [specs[o:o + n] for o, n in zip(offs, sizes)]


def step(k, sync):
    for i, bp in enumerate(bps):
        bp.process_frames(None, bench.motions_for(sub[i], k), sync=sync,
                          images_dev=imgs[k, offs[i]].data_ptr())


for k in range(Wm):
    step(k, True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(K):
    step(Wm + s, False)
for bp in bps:
    bp.sync()
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"contexts={sizes} B={B}: {B * K / dt:.1f} frames/s ({dt / K * 1e3:.2f} ms/step)")
