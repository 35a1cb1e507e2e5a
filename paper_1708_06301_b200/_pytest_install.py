"""pytest plugin: run the reference's OWN test suite with the device
implementations installed (install.install, INTEGRATION.md Option B).

    PYTHONPATH=baseline/_ref:. python -m pytest \
        -p paper_1708_06301_b200._pytest_install baseline/_ref/egostereo_tests

The plugin is loaded before the test modules import ``egostereo``'s names,
so every ``from egostereo.sgm import matching_cost`` in the suite binds the
device adapter.  tests/test_gpu_reference_suite.py drives it.
"""


def pytest_configure(config):
    import egostereo

    from paper_1708_06301_b200 import install
    install.install(egostereo)
    print("egostereo hot path: paper_1708_06301_b200 device implementations installed",
          flush=True)
    config.addinivalue_line("markers", "b200: reference suite run on the device path")


def pytest_report_header(config):
    return "egostereo hot path: paper_1708_06301_b200 device implementations installed"
