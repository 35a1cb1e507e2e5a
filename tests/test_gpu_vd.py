"""The opt-in fused column + diagonal aggregation (es_sgm_vd.cu, one
thread-block cluster per view) against the same oracle and single-sequence
checks as the default path.  The schedule is chosen once per process from
ES_SGM_VD, so each mode runs the bench-path tests in a child process."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.mark.parametrize("mode,tests", [
    ("1", ["test_every_batch_schedule_equals_single_sequences",
           "test_config5_full_batch_declared_subset_matches_oracle"]),
    ("2", ["test_every_batch_schedule_equals_single_sequences"]),
])
def test_fused_cluster_pass_matches(mode, tests):
    env = dict(os.environ, ES_SGM_VD=mode)
    sel = " or ".join(tests)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(HERE, "test_gpu_bench_path.py"), "-k", sel],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("mode", ["1", "2", "3"])
@pytest.mark.parametrize("shape", [(310, 94, 40), (1242, 40, 127), (96, 32, 31)])
def test_fused_cluster_pass_total_volumes(mode, shape):
    """The aggregated volumes themselves (not only the winners) of a batch of
    9 sequences, three of them checked against the oracle, for image widths
    that leave trailing CTAs of a cluster without columns (310, 96) and the
    full config width (1242)."""
    w, h, d = shape
    env = dict(os.environ, ES_SGM_VD=mode)
    if mode == "3":   # the cluster pass into a third partial sum, concurrent with grp4 jobs
        env["ES_SGM_PARTS"] = "4"
    r = subprocess.run([sys.executable, os.path.join(HERE, "vd_volume_check.py"), str(w), str(h),
                        str(d), "9", "3"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0 and "volumes ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
