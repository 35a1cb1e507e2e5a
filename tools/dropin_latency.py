"""Per-frame latency of the single-sequence drop-in API
(DisparityPipeline.process_frame + reading the fused left map), config 5
shape, host images in, host maps out -- what a reference user sees."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1708_06301_b200 import core, pipeline

rig = core.StereoRig(**bench.RIG)
specs = bench.sequence_specs(1, seed0=1000)
n = 20
imgs = bench.render_frames(specs, list(range(n)), "cuda:0").cpu().numpy()
pipe = pipeline.DisparityPipeline(rig)
times, parts = [], []
for k in range(n):
    t0 = time.perf_counter()
    res = pipe.process_frame(core.GrayImage(imgs[k, 0, 0]), core.GrayImage(imgs[k, 0, 1]),
                             bench.motions_for(specs, k)[0])
    t1 = time.perf_counter()
    fl = res.fused.left          # host map, as the reference returns it
    times.append(time.perf_counter() - t0)
    parts.append((t1 - t0, time.perf_counter() - t1))
    del res, fl
steady = times[3:]
print("step / map read ms:", [(round(a * 1e3, 2), round(b * 1e3, 2)) for a, b in parts[3:8]])
print(f"drop-in process_frame + fused map read: median {1e3 * sorted(steady)[len(steady) // 2]:.2f} ms "
      f"per frame ({len(steady)} frames after 3 warm-up), first frame {1e3 * times[0]:.0f} ms")
