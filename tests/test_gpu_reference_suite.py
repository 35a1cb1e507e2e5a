"""Drop-in proof: the reference's OWN test suite (119 tests, shipped next to
the unmodified package in baseline/_ref by tools/install_reference.sh) run
with install.install() applied, i.e. every hot-path function the suite
imports from egostereo executes on the B200 through the C ABI."""

import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")


def test_reference_suite_passes_on_the_device_path():
    tests = os.path.join(REF, "egostereo_tests")
    if not os.path.isdir(tests):
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]))
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "-p", "paper_1708_06301_b200._pytest_install", "egostereo_tests"],
                       cwd=REF, env=env, capture_output=True, text=True, timeout=1800)
    tail = p.stdout[-4000:]
    assert "device implementations installed" in p.stdout, tail
    m = re.search(r"(\d+) passed", p.stdout)
    assert p.returncode == 0 and m and int(m.group(1)) == 119, tail
