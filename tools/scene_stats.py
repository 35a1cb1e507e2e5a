"""Per-frame search fraction / validity of the bench scene for a few texture
scales (scene-model sanity check; not a benchmark)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_1708_06301_b200 import pipeline
from paper_1708_06301_b200.core import StereoRig

rig = StereoRig(**bench.RIG)
for ts in [float(x) for x in sys.argv[1:]] or [0.05]:
    bench.TEXTURE_SCALE = ts
    specs = bench.sequence_specs(2, seed0=1000)
    imgs = bench.render_frames(specs, list(range(8)), "cuda:0")
    bp = pipeline.BatchedPipeline(rig, 2)
    fr = []
    for k in range(8):
        bp.process_frames(None, bench.motions_for(specs, k), sync=True, images_dev=imgs[k].data_ptr())
        r = bp.result(0)
        fr.append((round(r.search_fraction_left, 3), round(float(r.fused.left.valid.mean()), 3),
                   round(float(r.measured_left.valid.mean()), 3), round(float(r.keep_left.mean()), 3)))
    print(f"texture_scale={ts}: (fraction, fused valid, measured valid, kept) per frame:", fr)
