"""install() rebinding into the unmodified reference package (baseline/_ref,
tools/install_reference.sh): every hot-path name the reference binds -- in
its defining modules, again in pipeline.py:38-50 and in __init__.py:30-47 --
points at a device adapter afterwards, and uninstall() restores them.  CPU
only (no device call is made); the device run of the reference's own suite
is tests/test_gpu_reference_suite.py."""

import os
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture()
def egostereo():
    if not os.path.isdir(os.path.join(REF, "egostereo")):
        pytest.skip("reference not installed (tools/install_reference.sh)")
    sys.path.insert(0, REF)
    try:
        import egostereo as eg
        yield eg
    finally:
        sys.path.remove(REF)


def test_install_rebinds_every_bound_name_and_uninstall_restores(egostereo):
    from paper_1708_06301_b200 import install
    import egostereo.pipeline as rp
    import egostereo.sgm as rs
    before = {(m, n): getattr(getattr(egostereo, m), n)
              for m, names in install.REBOUND.items() for n in names}
    before_pipe = {n: getattr(rp, n) for n in install.PIPELINE_NAMES}
    ref_dp = rp.DisparityPipeline
    install.install(egostereo)
    try:
        assert install.installed(egostereo)
        for (m, n), old in before.items():
            new = getattr(getattr(egostereo, m), n)
            assert new is not old and getattr(new, "__b200__", False), (m, n)
        for n in install.PIPELINE_NAMES:
            assert getattr(rp, n) is getattr(getattr(egostereo, _home(install, n)), n), n
        for n in install.ROOT_NAMES:
            assert getattr(getattr(egostereo, n), "__b200__", False), n
        assert issubclass(rp.DisparityPipeline, ref_dp) and rp.DisparityPipeline.__b200__
        assert egostereo.DisparityPipeline is rp.DisparityPipeline
        assert rs.matching_cost.__name__ == "<lambda>" or rs.matching_cost.__b200__
        install.install(egostereo)          # idempotent
    finally:
        install.uninstall(egostereo)
    assert not install.installed(egostereo)
    for (m, n), old in before.items():
        assert getattr(getattr(egostereo, m), n) is old
    for n, old in before_pipe.items():
        assert getattr(rp, n) is old
    assert rp.DisparityPipeline is ref_dp


def _home(install, name):
    for m, names in install.REBOUND.items():
        if name in names:
            return m
    raise KeyError(name)
