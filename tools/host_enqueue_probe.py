import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1708_06301_b200 import pipeline
from paper_1708_06301_b200.core import StereoRig
rig = StereoRig(**bench.RIG)
B, K, Wm = 64, 10, 3
specs = bench.sequence_specs(B, seed0=1000)
imgs = bench.render_frames(specs, list(range(Wm + K)), "cuda:0")
bp = pipeline.BatchedPipeline(rig, B)
for k in range(Wm):
    bp.process_frames(None, bench.motions_for(specs, k), sync=True, images_dev=imgs[k].data_ptr())
staged = [imgs[Wm + i].cpu().pin_memory() for i in range(K)]
outs = [torch.empty((B, rig.height, rig.width), dtype=torch.int16, pin_memory=True) for _ in range(K)]
torch.cuda.synchronize()
t0 = time.perf_counter(); th = []
for i in range(K):
    a = time.perf_counter()
    bp.process_frames(staged[i].numpy(), bench.motions_for(specs, Wm + i), sync=False)
    b = time.perf_counter()
    bp.fused_kitti(0, out=outs[i].numpy().view(np.uint16), sync=False)
    th.append((b - a, time.perf_counter() - b))
t1 = time.perf_counter()
bp.sync(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("host enqueue per step ms (step, export):", [(round(x*1e3,2), round(y*1e3,2)) for x, y in th])
print("enqueue total %.1f ms, wall total %.1f ms, per step %.2f ms" % ((t1-t0)*1e3, (t2-t0)*1e3, (t2-t0)*1e3/K))
