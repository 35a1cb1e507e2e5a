"""The device renderer (bench input generator) against the reference's own
synth.render_frame output stored in tests/golden/render.npz."""

import ctypes

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_render_matches_reference_synth():
    import torch
    from paper_1708_06301_b200 import _lib, core
    g = load_golden("render")
    f, b, cx, cy, w, h, d_max = g["rig"]
    rig = core.StereoRig(f=f, b=b, cx=cx, cy=cy, width=int(w), height=int(h), d_max=int(d_max))
    boxes = np.ascontiguousarray(g["boxes"][None], np.float64)
    seeds = np.array([int(g["texture_seed"])], np.int64)
    rs = _lib.rig_struct(rig)
    for k in range(2):
        pose = np.ascontiguousarray(g[f"pose{k}"][None], np.float64)
        img = torch.empty((1, 2, rig.height, rig.width), dtype=torch.uint8, device="cuda")
        gt = torch.empty((1, 2, rig.height, rig.width), dtype=torch.float64, device="cuda")
        _lib.call("es_render", ctypes.byref(rs), _lib.ptr(boxes), boxes.shape[1], _lib.ptr(pose),
                  _lib.ptr(seeds), 1, ctypes.c_double(float(g["texture_scale"])),
                  int(g["background"]), ctypes.c_void_p(img.data_ptr()),
                  ctypes.c_void_p(gt.data_ptr()), ctypes.c_void_p(0))
        im = img.cpu().numpy()[0]
        gd = gt.cpu().numpy()[0]
        for v, tag in ((0, "l"), (1, "r")):
            ref = g[f"img{k}_{tag}"]
            # value-noise texture in float64: allow last-ulp rint flips only
            diff = np.abs(im[v].astype(int) - ref.astype(int))
            assert (diff <= 1).all() and (diff > 0).mean() < 1e-3, (k, tag, (diff > 0).mean())
            np.testing.assert_allclose(gd[v], g[f"gt{k}_{tag}"], rtol=1e-12, atol=0)
