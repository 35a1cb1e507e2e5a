"""Per-call latency of stage-level drop-in functions on config-5-sized
inputs (host arrays in / out, as the reference API passes them):
matching_cost and aggregate_paths (dense 375x1242x128 float32 volume).  A/B of library builds via ES_LIB_PATH."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1708_06301_b200 import core, sgm

H, W, D = 375, 1242, 128
rig = core.StereoRig(f=718.9, b=0.54, cx=607.0, cy=185.0, width=W, height=H, d_max=D - 1)
rng = np.random.default_rng(3)
left = core.GrayImage(rng.integers(0, 256, (H, W), dtype=np.uint8))
right = core.GrayImage(rng.integers(0, 256, (H, W), dtype=np.uint8))
params = sgm.SgmParams()
iv = sgm.full_range_intervals(rig)


def timed(f, n=5):
    f()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e3 * sorted(ts)[len(ts) // 2]


vol = sgm.matching_cost(left, right, iv, params, "left")
print(f"matching_cost   {timed(lambda: sgm.matching_cost(left, right, iv, params, 'left')):8.2f} ms")
print(f"aggregate_paths {timed(lambda: sgm.aggregate_paths(vol, params)):8.2f} ms")
