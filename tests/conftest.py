import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_runtest_logreport(report):
    """BNF_DURATIONS_FILE=path: append every test's call duration as it finishes (survives a killed run)."""
    path = os.environ.get("BNF_DURATIONS_FILE")
    if path and report.when == "call":
        with open(path, "a") as f:
            f.write("%8.2f %s %s\n" % (report.duration, report.outcome, report.nodeid))


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
