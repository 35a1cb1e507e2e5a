"""The fused vertical + diagonal sweep (csrc/es_sgm_sweep.cu) forced on for
every batch size (by default it runs for contexts of >= 64 views, or >= 24
views in a batch split over several contexts): the batched / deferred bench
path, every partial-sum schedule (2 and 4 partial sums: read-modify-write
and initialising sweeps), degenerate shapes, window / penalty variants,
D = 256 (8 lanes per chain) and config 4 at full size bit-exact against the
reference -- the same tests as the default path, in a subprocess with
ES_SGM_SWEEP=1 (the switch is read once per process)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_parity_suite_with_the_sweep_forced_on():
    env = dict(os.environ, ES_SGM_SWEEP="1")
    tests = ["tests/test_gpu_bench_path.py", "tests/test_gpu_pipeline.py",
             "tests/test_gpu_configs.py::test_config4_class_d256",
             "tests/test_gpu_configs.py::test_degenerate_shapes_match_oracle",
             "tests/test_gpu_configs.py::test_window_and_penalty_variants_match_oracle",
             "tests/test_gpu_configs.py::test_config3_class_moving_boxes_and_salt_noise",
             "tests/test_gpu_full_configs.py::test_full_size_sequence_matches_reference[4]",
             "tests/test_gpu_full_configs.py::test_full_size_sequence_matches_reference[2]"]
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *tests],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=2400)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]


def test_row_kernel_read_modify_write_schedule():
    """ES_SGM_SWEEP_ORDER=2 runs both sweeps BEFORE the row jobs, so the row
    kernel (k_sgm_row, the cp.async operand ring) runs its partial-sum
    read-modify-write variant -- by default only batches of >= 64 sequences
    per context do that -- and ES_SGM_ROW=0 runs the same tests with the
    grp4 row jobs it replaced (the A/B fallback)."""
    tests = ["tests/test_gpu_pipeline.py",
             "tests/test_gpu_configs.py::test_degenerate_shapes_match_oracle",
             "tests/test_gpu_configs.py::test_window_and_penalty_variants_match_oracle",
             "tests/test_gpu_configs.py::test_config3_class_moving_boxes_and_salt_noise"]
    for extra in ({"ES_SGM_SWEEP": "1", "ES_SGM_SWEEP_ORDER": "2"}, {"ES_SGM_ROW": "0"}):
        env = dict(os.environ, **extra)
        p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *tests],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=2400)
        assert p.returncode == 0, str(extra) + p.stdout[-4000:] + p.stderr[-2000:]
