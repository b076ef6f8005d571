"""pytest configuration: `gpu` marker, checker builds, shared fixtures.

Two CPU checkers (oracle/, test infrastructure only):
  * `ref`    the reference itself: /root/reference/proj/core/src compiled
             verbatim against the Eigen-subset shim (`make -C oracle ref`,
             oracle/_ref/mb_ref*.so). Built here when /root/reference exists;
             on the GPU box the prebuilt module travels with the repo.
  * `oracle` the line-by-line restatement (`make -C oracle`, oracle/_build).
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


REFERENCE = "/root/reference/proj"


def _build_ref():
    if os.path.isdir(REFERENCE):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)


@pytest.fixture(scope="session")
def ref():
    _build_ref()
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    import mb_ref  # fails loudly when neither the reference nor the prebuilt module is present

    return mb_ref


@pytest.fixture(scope="session")
def oracle():
    _build_oracle()
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_build"))
    import mb_oracle

    return mb_oracle
