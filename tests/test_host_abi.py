"""CPU-side tests of the product boundary: the C-ABI library loads, exports
every symbol include/manybeam_b200.h declares, and its host logic (rods,
first-N truncation, stepper tables, energy conversion, validation) agrees
with the oracle restatement bit for bit. No compute calls here (no GPU)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2306_00271_b200 as mb
from paper_2306_00271_b200 import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "manybeam_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(mb_\w+)\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(mb.library_path())
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s


def test_library_targets_sm100a():
    out = os.popen(f"cuobjdump --list-elf {mb.library_path()} 2>&1").read()
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    if mb.device_available():
        pytest.skip("a device is present")
    with pytest.raises(mb.CudaError):
        mb.Context(0)


@pytest.mark.parametrize("cell,n", [(("hex", 3.84), 13), (("hex", 3.84), 15), (("hex", 3.84), 63),
                                    (("rect", 7.68, 3.84), 61), (("hex", 19.2), 199), (("hex", 3.84), 255)])
def test_rods_match_oracle_bitwise(oracle, cell, n):
    lat = mb.Lattice2D.hexagonal(cell[1]) if cell[0] == "hex" else mb.Lattice2D.rectangular(cell[1], cell[2])
    r = mb.RodSet.build_first(lat, n)
    o = oracle.RodSet.build_first(oracle.Lattice2D(lat.a1, lat.a2), n)
    assert np.array_equal(r.k, o.k) and np.array_equal(r.m, o.m)
    assert np.array_equal(r.diff, o.diff) and np.array_equal(r.diff_m, o.diff_m)
    assert np.array_equal(r.diff_index, o.diff_index)


@pytest.mark.parametrize("cell,n", [(("hex", 3.84), 13), (("hex", 3.84), 63), (("rect", 7.68, 3.84), 61),
                                    (("hex", 19.2), 199), (("hex", 3.84), 255)])
def test_rods_match_reference_bitwise(ref, cell, n):
    """The product's host rod tables against the reference's own RodSet::build
    (oracle/_ref; first-N by truncating the reference's total order)."""
    lat = mb.Lattice2D.hexagonal(cell[1]) if cell[0] == "hex" else mb.Lattice2D.rectangular(cell[1], cell[2])
    r = mb.RodSet.build_first(lat, n)
    o = ref.RodSet.build_first(ref.Lattice2D(lat.a1, lat.a2), n)
    assert np.array_equal(r.k, o.k) and np.array_equal(r.m, o.m)
    assert np.array_equal(r.diff_m, o.diff_m) and np.array_equal(r.diff_index, o.diff_index)


def test_rods_cutoff_build_matches_reference(ref):
    lat = mb.Lattice2D((2.0, 0.0), (0.0, 2.6))
    r = mb.RodSet.build(lat, 5.0)
    o = ref.RodSet.build(ref.Lattice2D(lat.a1, lat.a2), 5.0)
    assert r.size() == 11 and np.array_equal(r.k, o.k) and np.array_equal(r.diff_index, o.diff_index)


def test_rods_cutoff_build_matches_oracle(oracle):
    lat = mb.Lattice2D((2.0, 0.0), (0.0, 2.6))
    r = mb.RodSet.build(lat, 5.0)
    o = oracle.RodSet.build(oracle.Lattice2D(lat.a1, lat.a2), 5.0)
    assert r.size() == 11 and np.array_equal(r.k, o.k) and np.array_equal(r.diff_index, o.diff_index)


def test_rods_validation():
    with pytest.raises(mb.ConfigError):
        mb.RodSet.build(mb.Lattice2D((1.0, 2.0), (2.0, 4.0)), 3.0)
    with pytest.raises(mb.ConfigError):
        mb.RodSet.build(mb.Lattice2D((1.0, 0.0), (0.0, 1.0)), -1.0)


def test_stepper_tables_match_oracle(oracle):
    for name in ("sp4", "sp6"):
        a, b = mb.StepperSpec.by_name(name), oracle.StepperSpec.by_name(name)
        assert list(a.drift) == list(b.drift) and list(a.kick) == list(b.kick)
    with pytest.raises(mb.ConfigError):
        mb.StepperSpec.by_name("magnus9")


def test_energy_conversion_matches_oracle(oracle):
    for e in (10000.0, 15000.0, 30000.0):
        assert mb.beam_from_energy(e) == oracle.beam_from_energy(e)
        assert configs.relativistic(e) == pytest.approx(oracle.beam_from_energy(e), rel=1e-15)


def test_angle_grid_validation():
    with pytest.raises(mb.ConfigError):
        mb.AngleGrid.validated([], [0.0])
    with pytest.raises(mb.ConfigError):
        mb.AngleGrid.validated([2.0, 1.0], [0.0])
    with pytest.raises(mb.ConfigError):
        mb.AngleGrid.validated([0.0], [0.0])
    assert mb.AngleGrid.validated([1.0, 2.0], [0.0, 30.0]).rows() == 4


def test_workload_shapes():
    assert configs.config0().points() == 31
    assert configs.config1().points() == 121
    assert configs.config2().points() == 1024 * 61
    assert configs.config3().points() == 61
    assert configs.config4(255).points() == 4096
    w = configs.config1()
    assert w.flops_per_point() == pytest.approx(11.98e9, rel=2e-3)
