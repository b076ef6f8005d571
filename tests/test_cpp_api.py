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


def test_curve_csv_python_cpp_bytes(tmp_path):
    """Two independent writers of the reference's wire format (csvio.cpp:65-149)
    agree byte for byte: Python writes, C++ reads and rewrites."""
    import numpy as np
    import paper_2306_00271_b200 as mb
    rng = np.random.default_rng(7)
    eta = rng.random((5, 4)) ** 6
    eta[0, 1] = 0.0
    c = mb.RockingCurve(list(np.linspace(0.5, 2.5, 5)), [0.0] * 5, eta, ["(0;0)", "(1;0)", "(0;-1)", "(-1;1)"],
                        "sp6", 0.0125, 1000.0)
    a = tmp_path / "a.csv"
    b = tmp_path / "b.csv"
    mb.write_curve_csv(a, c)
    r = subprocess.run([_build(tmp_path), "--rewrite", str(a), str(b)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert a.read_bytes() == b.read_bytes()
    back = mb.read_curve_csv(b)
    assert back.rod_labels == c.rod_labels and back.method == "sp6" and back.rhst_threshold == 1000.0
    assert mb.curve_error(back, c) <= 1e-15
    assert mb.compare_curve_files(a, b) == 0.0
    (tmp_path / "bad.csv").write_text("theta0,theta1,eta(0;0)\n1.0,2.0\n")
    with pytest.raises(mb.IoError):
        mb.read_curve_csv(tmp_path / "bad.csv")
