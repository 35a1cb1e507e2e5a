import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_1708_06301_b200 import core, pipeline
g = np.load("tests/golden/seq_small.npz")
f, b, cx, cy, w, h, d_max = g["rig"]
rig = core.StereoRig(f=f, b=b, cx=cx, cy=cy, width=int(w), height=int(h), d_max=int(d_max))
pipe = pipeline.DisparityPipeline(rig)
try:
    for k in range(3):
        m = g[f"f{k}_motion"] if bool(g[f"f{k}_has_motion"]) else None
        r = pipe.process_frame(core.GrayImage(g[f"f{k}_left"]), core.GrayImage(g[f"f{k}_right"]), m)
        ok = np.array_equal(r.measured_left.values, g[f"f{k}_l_meas_d"])
        print(os.environ.get("ES_SGM_VAR"), "frame", k, "wta ok" if ok else "WTA MISMATCH")
except Exception as e:
    print(os.environ.get("ES_SGM_VAR"), "ERROR", str(e)[:100])
