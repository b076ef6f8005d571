"""Builds and runs the C++ host-API test (tests/cpp/test_cpp_api.cpp) that
exercises include/manybeam_b200.hpp the way the reference's doctest suites
exercise the C++ library."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2306_00271_b200")


def _build(tmp_path):
    exe = str(tmp_path / "test_cpp_api")
    subprocess.run(["g++", "-O2", "-std=c++17", os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"),
                    f"-L{LIBDIR}", "-lmanybeam_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_api_host_only(tmp_path):
    r = subprocess.run([_build(tmp_path), "--no-device"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_api_device(tmp_path):
    r = subprocess.run([_build(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
