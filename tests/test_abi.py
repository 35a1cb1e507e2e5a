"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/egostereo_b200.h declares, the ctypes table
matches the header, and the host types keep the reference's validation."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "egostereo_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(es_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_1708_06301_b200 import _lib, build
    path = build.build()
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a_with_static_cudart():
    import subprocess
    from paper_1708_06301_b200 import build
    path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", path], capture_output=True, text=True).stdout
    assert "libcudart" not in ldd


def test_version_and_error_string_without_gpu():
    from paper_1708_06301_b200 import _lib
    lib = _lib.load()
    assert lib.es_version() == 1
    assert isinstance(lib.es_last_error(), bytes)


def test_host_types_validate_like_reference():
    from paper_1708_06301_b200 import core, prediction, sgm, fusion
    with pytest.raises(ValueError):
        core.StereoRig(f=1.0, b=0.5, cx=0, cy=0, width=10, height=10, d_max=10)
    with pytest.raises(ValueError):
        sgm.SgmParams(window=4)
    with pytest.raises(ValueError):
        sgm.SgmParams(p1=10.0, p2=5.0)
    with pytest.raises(ValueError):
        sgm.IntervalMap(np.array([[2]]), np.array([[1]]), 4)
    with pytest.raises(ValueError):
        prediction.PredictionParams(q=-1.0)
    with pytest.raises(ValueError):
        fusion.FusionParams(p_init=0.0)
    with pytest.raises(ValueError):
        core.validate_rigid_motion(np.diag([1.0, 1.0, -1.0, 1.0]))
    assert sgm.SgmParams().border_cost == 9 * 255
    img = core.GrayImage(np.full((3, 3), 7, np.int32))
    assert img.data.dtype == np.uint8


def test_homography_bit_identical_to_golden():
    from paper_1708_06301_b200 import core, geometry
    from conftest import load_golden
    g = load_golden("prediction")
    f, b, cx, cy, w, h, d_max = g["rig"]
    rig = core.StereoRig(f=f, b=b, cx=cx, cy=cy, width=int(w), height=int(h), d_max=int(d_max))
    for t in range(10):
        T = g[f"t{t}_T"]
        assert np.array_equal(geometry.disparity_homography(rig, T), g[f"t{t}_HL"])
        assert np.array_equal(geometry.disparity_homography(rig, geometry.right_motion(rig, T)),
                              g[f"t{t}_HR"])


def test_device_calls_fail_loudly_without_gpu():
    """No CPU fallback: with no CUDA device a stage call raises."""
    from conftest import has_gpu
    if has_gpu():
        pytest.skip("GPU present")
    from paper_1708_06301_b200 import core, sgm
    rig = core.StereoRig(f=8.0, b=0.5, cx=3.5, cy=1.5, width=8, height=4, d_max=3)
    with pytest.raises(RuntimeError):
        sgm.search_intervals(core.DisparityMap(np.zeros(rig.shape), np.zeros(rig.shape, bool)),
                             core.VarianceMap(np.zeros(rig.shape)), rig)


def test_batched_pipeline_groups_validate_before_device_work():
    """BatchedPipeline's context groups (B >= 24 runs as contexts of ~16 sequences): a
    batch that does not split raises ValueError before any device call."""
    from paper_1708_06301_b200 import core, pipeline
    rig = core.StereoRig(f=100.0, b=0.5, cx=15.0, cy=10.0, width=32, height=20, d_max=8)
    with pytest.raises(ValueError, match="groups"):
        pipeline.BatchedPipeline(rig, 5, groups=2)
    with pytest.raises(ValueError, match="groups"):
        pipeline.BatchedPipeline(rig, 4, groups=0)


def test_bench_launch_count_by_path():
    """bench.py's gpu_launches claim: 13 kernels per context step with the
    fused sweeps (>= 64 views per context), 19 with per-direction jobs."""
    import bench
    assert bench.kernels_per_step(64) == 13 and bench.kernels_per_step(128) == 13
    assert bench.kernels_per_step(32) == 19 and bench.kernels_per_step(2) == 19
    # contexts of 32 views sharing a batch of >= 128 views keep the fused sweeps
    assert bench.kernels_per_step(32, 128) == 13 and bench.kernels_per_step(16, 128) == 19
    assert bench.kernels_per_step(24, 48) == 13 and bench.kernels_per_step(32, 0) == 19
    from paper_1708_06301_b200 import pipeline
    assert [pipeline.default_groups(b) for b in (1, 8, 16, 20, 24, 32, 48, 63, 64, 96, 128)] == \
        [1, 1, 1, 1, 2, 2, 3, 3, 4, 6, 8]
