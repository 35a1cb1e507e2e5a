"""KITTI-layout I/O (kitti_io.py, pipeline.load_sequence / write_sequence)
against a tree written and read back by the unmodified reference
(tests/golden/kitti.npz), plus the reference tests' error cases.  CPU only."""

import os

import numpy as np
import pytest

from conftest import load_golden

cv2 = pytest.importorskip("cv2")


def _materialise(g, root):
    os.makedirs(root, exist_ok=True)
    for rel in ("calib.txt", "poses.txt"):
        open(os.path.join(root, rel), "wb").write(g["file_" + rel.replace(".", "_")].tobytes())
    n = len([k for k in g.files if k.startswith("left_")])
    for sub in ("image_0", "image_1", "gt_disp_0", "gt_disp_1"):
        os.makedirs(os.path.join(root, sub), exist_ok=True)
        for k in range(n):
            open(os.path.join(root, sub, f"{k:06d}.png"), "wb").write(g[f"file_{sub}_{k}"].tobytes())
    return n


def test_load_sequence_matches_reference(tmp_path):
    from paper_1708_06301_b200 import pipeline
    g = load_golden("kitti")
    n = _materialise(g, str(tmp_path))
    seq = pipeline.load_sequence(str(tmp_path), d_max=8)
    r = seq.rig
    assert np.array_equal(np.array([r.f, r.b, r.cx, r.cy, r.width, r.height, r.d_max]), g["rig"])
    assert len(seq) == n
    for k in range(n):
        assert np.array_equal(seq.lefts[k].data, g[f"left_{k}"])
        assert np.array_equal(seq.rights[k].data, g[f"right_{k}"])
        m = np.eye(4) if seq.motions[k] is None else seq.motions[k]
        assert np.array_equal(m, g[f"motion_{k}"])
        assert np.array_equal(seq.gt_left[k].values, g[f"gtl_d_{k}"])
        assert np.array_equal(seq.gt_left[k].valid, g[f"gtl_v_{k}"])
        assert np.array_equal(seq.gt_right[k].values, g[f"gtr_d_{k}"])
    assert seq.motions[0] is None


def test_write_sequence_matches_reference(tmp_path):
    from paper_1708_06301_b200 import core, kitti_io, pipeline
    g = load_golden("kitti")
    n = _materialise(g, str(tmp_path / "ref"))
    seq = pipeline.load_sequence(str(tmp_path / "ref"), d_max=8)
    # write the in-memory maps the reference wrote, through our writer
    seq.gt_left = [core.DisparityMap(g[f"src_gtl_d_{k}"], g[f"src_gtl_v_{k}"]) for k in range(n)]
    seq.gt_right = None
    pipeline.write_sequence(str(tmp_path / "ours"), seq, list(g["poses"]))
    for rel in ("calib.txt", "poses.txt"):
        assert open(tmp_path / "ours" / rel, "rb").read() == g["file_" + rel.replace(".", "_")].tobytes()
    for k in range(n):
        for sub in ("image_0", "gt_disp_0"):
            ours = cv2.imread(str(tmp_path / "ours" / sub / f"{k:06d}.png"), cv2.IMREAD_UNCHANGED)
            ref = cv2.imdecode(g[f"file_{sub}_{k}"], cv2.IMREAD_UNCHANGED)
            assert np.array_equal(ours, ref), (sub, k)
    assert not (tmp_path / "ours" / "gt_disp_1").exists()
    again = kitti_io.read_disparity_png(str(tmp_path / "ours" / "gt_disp_0" / "000000.png"))
    assert np.array_equal(again.values, g["gtl_d_0"])


def test_disparity_png_round_trip_and_errors(tmp_path):
    from paper_1708_06301_b200 import core, kitti_io
    vals = np.array([[0.0, 1 / 256, 12.5], [100.0, 255.99, 0.001]])
    valid = np.array([[False, True, True], [True, True, True]])
    p = str(tmp_path / "d.png")
    kitti_io.write_disparity_png(p, core.DisparityMap(np.where(valid, vals, 0.0), valid))
    back = kitti_io.read_disparity_png(p)
    assert np.array_equal(back.valid, valid)               # a tiny valid value stays valid (>= 1)
    assert back.values[1, 2] == 1 / 256
    with pytest.raises(ValueError):
        kitti_io.write_disparity_png(p, core.DisparityMap(np.full((2, 2), 300.0), np.ones((2, 2), bool)))
    cv2.imwrite(str(tmp_path / "g8.png"), np.zeros((3, 3), np.uint8))
    with pytest.raises(kitti_io.FileFormatError):
        kitti_io.read_disparity_png(str(tmp_path / "g8.png"))
    with pytest.raises(kitti_io.FileFormatError):
        kitti_io.read_disparity_png(str(tmp_path / "missing.png"))


def test_pose_and_calib_validation(tmp_path):
    from paper_1708_06301_b200 import kitti_io
    p = str(tmp_path / "poses.txt")
    open(p, "w").write("1 0 0 0 0 1 0 0 0 0 1 0\n2 0 0 0 0 1 0 0 0 0 1 0\n")
    with pytest.raises(kitti_io.FileFormatError, match=":2:"):
        kitti_io.read_pose_file(p)
    open(p, "w").write("1 0 0 0 0 1 0 0 0 0 1\n")
    with pytest.raises(kitti_io.FileFormatError, match="expected 12"):
        kitti_io.read_pose_file(p)
    open(p, "w").write("\n")
    with pytest.raises(kitti_io.FileFormatError, match="no poses"):
        kitti_io.read_pose_file(p)
    c = str(tmp_path / "calib.txt")
    kitti_io.write_calib_file(c, kitti_io.CalibData(f=700.0, cx=600.0, cy=180.0, b=0.5))
    assert kitti_io.read_calib_file(c) == kitti_io.CalibData(f=700.0, cx=600.0, cy=180.0, b=0.5)
    open(c, "w").write("P0: 700 0 600 0 0 700 180 0 0 0 1 0\n")
    with pytest.raises(kitti_io.FileFormatError, match="missing P1"):
        kitti_io.read_calib_file(c)
    open(c, "w").write("P0: 700 0 600 0 0 700 180 0 0 0 1 0\nP1: 710 0 600 -350 0 700 180 0 0 0 1 0\n")
    with pytest.raises(kitti_io.FileFormatError, match="disagree"):
        kitti_io.read_calib_file(c)
    open(c, "w").write("P0: 700 0 600 0 0 700 180 0 0 0 1 0\nP1: 700 0 600 350 0 700 180 0 0 0 1 0\n")
    with pytest.raises(kitti_io.FileFormatError, match="baseline"):
        kitti_io.read_calib_file(c)
