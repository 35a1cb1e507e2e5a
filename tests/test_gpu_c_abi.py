"""The C ABI used natively (no Python between the caller and the library):
tests/c/abi_smoke.c is compiled against include/egostereo_b200.h, linked
with libegostereo_b200.so and run."""

import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_against_the_library(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    libdir = os.path.join(ROOT, "paper_1708_06301_b200")
    exe = str(tmp_path / "abi_smoke")
    subprocess.run([cc, "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-o", exe,
                    "-L", libdir, "-l:libegostereo_b200.so", "-Wl,-rpath," + libdir, "-lm"],
                   check=True)
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "brute-force SAD" in res.stdout
