"""The device renderer (bench / parity input generator) against the
reference's own synth.render_frame output: bit-exact images and ground truth
(tests/golden/render.npz: boxes; render_planes.npz: bounded and unbounded
planes plus boxes under rotated poses, both views)."""

import ctypes

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _rig(a):
    from paper_1708_06301_b200 import core
    f, b, cx, cy, w, h, d_max = a
    return core.StereoRig(f=f, b=b, cx=cx, cy=cy, width=int(w), height=int(h), d_max=int(d_max))


def _render(rig, entry, recs, n, pose, seed, scale, background=12):
    import torch
    from paper_1708_06301_b200 import _lib
    rs = _lib.rig_struct(rig)
    recs = np.ascontiguousarray(recs[None], np.float64)
    pose = np.ascontiguousarray(pose[None], np.float64)
    seeds = np.array([seed], np.int64)
    img = torch.empty((1, 2, rig.height, rig.width), dtype=torch.uint8, device="cuda")
    gt = torch.empty((1, 2, rig.height, rig.width), dtype=torch.float64, device="cuda")
    _lib.call(entry, ctypes.byref(rs), _lib.ptr(recs), n, _lib.ptr(pose), _lib.ptr(seeds), 1,
              ctypes.c_double(scale), background, ctypes.c_void_p(img.data_ptr()),
              ctypes.c_void_p(gt.data_ptr()), ctypes.c_void_p(0))
    return img.cpu().numpy()[0], gt.cpu().numpy()[0]


def test_render_boxes_bit_exact_vs_reference_synth():
    g = load_golden("render")
    rig = _rig(g["rig"])
    for k in range(2):
        im, gd = _render(rig, "es_render", g["boxes"], g["boxes"].shape[0], g[f"pose{k}"],
                         int(g["texture_seed"]), float(g["texture_scale"]), int(g["background"]))
        for v, tag in ((0, "l"), (1, "r")):
            assert np.array_equal(im[v], g[f"img{k}_{tag}"]), (k, tag)
            assert np.array_equal(gd[v], g[f"gt{k}_{tag}"]), (k, tag)


@pytest.mark.parametrize("case", [0, 1, 2])
def test_render_planes_bit_exact_vs_reference_synth(case):
    g = load_golden("render_planes")
    rig = _rig(g[f"c{case}_rig"])
    prims = g[f"c{case}_prims"]
    for k in range(2):
        im, gd = _render(rig, "es_render_prims", prims, prims.shape[0], g[f"c{case}_f{k}_pose"],
                         int(g[f"c{case}_seed"]), float(g[f"c{case}_scale"]))
        assert np.array_equal(im, g[f"c{case}_f{k}_img"]), (case, k)
        assert np.array_equal(gd, g[f"c{case}_f{k}_gt"]), (case, k)
