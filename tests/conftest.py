"""pytest configuration: `gpu` marker, oracle build, shared fixtures.

The oracle (oracle/, test infrastructure only) is the CPU restatement of the
reference hot path; it is built on first use with `make -C oracle`.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU case")


def _build_oracle():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


@pytest.fixture(scope="session")
def oracle():
    _build_oracle()
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_build"))
    import mb_oracle

    return mb_oracle
