"""Oracle pinning: rods, geometry, first-N extension, energy conversion.
Ports proj/tests/test_rods_geometry.cpp:10-131."""
import math

import numpy as np
import pytest

import fields


def test_reciprocal_basis_dual(oracle):  # :10-19
    lat = oracle.Lattice2D((2.1, 0.3), (-0.5, 2.9))
    b1, b2 = np.array(lat.b1()), np.array(lat.b2())
    tau = 2 * math.pi
    assert b1 @ np.array([2.1, 0.3]) == pytest.approx(tau, rel=1e-13)
    assert abs(b1 @ np.array([-0.5, 2.9])) < 1e-13
    assert abs(b2 @ np.array([2.1, 0.3])) < 1e-13
    assert b2 @ np.array([-0.5, 2.9]) == pytest.approx(tau, rel=1e-13)


def test_degenerate_lattice_rejected(oracle):  # :21-26
    with pytest.raises(oracle.ConfigError):
        oracle.Lattice2D((1.0, 2.0), (2.0, 4.0)).validate()


def test_square_shells(oracle):  # :28-37
    lat = oracle.Lattice2D((2.0, 0.0), (0.0, 2.0))
    b = math.pi
    assert [oracle.RodSet.build(lat, f * b).size() for f in (0.5, 1.1, 1.5, 2.1)] == [1, 5, 9, 13]


def test_canonical_11(oracle):  # :39-45
    rods = fields.rods11(oracle)
    assert rods.size() == 11
    assert tuple(rods.m[0]) == (0, 0)
    norms = np.linalg.norm(rods.k, axis=1)
    assert norms[0] == 0.0 and np.all(np.diff(norms) >= 0)


def test_difference_table(oracle):  # :47-59
    rods = fields.rods11(oracle)
    di, k, m = rods.diff_index, rods.k, rods.m
    for j in range(rods.size()):
        for kk in range(rods.size()):
            d = di[j, kk]
            assert 0 <= d < rods.diff_count()
            assert np.linalg.norm(rods.diff[d] - (k[j] - k[kk])) <= 1e-14
            assert tuple(rods.diff_m[d]) == tuple(m[j] - m[kk])
    assert rods.diff_count() < rods.size() ** 2


def b0_by_rotation(gamma, t0, t1):  # oracles.hpp:113-119
    d = math.pi / 180
    v = np.array([math.cos(t0 * d), 0.0, -math.sin(t0 * d)])
    c, s = math.cos(t1 * d), math.sin(t1 * d)
    v = np.array([c * v[0] - s * v[1], s * v[0] + c * v[1], v[2]])
    return gamma * v[:2]


def test_incident_matches_rotation(oracle):  # :61-71
    rng = np.random.default_rng(5)
    for _ in range(50):
        g, t0, t1 = rng.uniform(0.5, 40), rng.uniform(1, 89), rng.uniform(-180, 180)
        beam = oracle.BeamGeometry(g, t0, t1)
        assert np.linalg.norm(np.array(beam.b0) - b0_by_rotation(g, t0, t1)) <= 1e-12 * g
        assert beam.sin_theta0 == pytest.approx(math.sin(t0 * math.pi / 180), rel=1e-14)


@pytest.mark.parametrize("args", [(1.0, 0.0), (1.0, 90.0), (1.0, -5.0), (0.0, 10.0), (-2.0, 10.0)])
def test_angle_gamma_validation(oracle, args):  # :73-79
    with pytest.raises(oracle.ConfigError):
        oracle.BeamGeometry(args[0], args[1], 0.0)


def test_gamma_squares_back(oracle):  # :81-106
    rng = np.random.default_rng(9)
    rods = fields.rods11(oracle)
    for _ in range(40):
        beam = oracle.BeamGeometry(rng.uniform(1, 20), rng.uniform(1, 60), rng.uniform(-90, 90))
        gm = oracle.GammaMatrix.build(rods, beam)
        b0 = np.array(beam.b0)
        for i in range(rods.size()):
            exp = beam.gamma ** 2 - np.sum((b0 + rods.k[i]) ** 2)
            assert abs(gm.diag[i] ** 2 - exp) <= 1e-13 * max(1.0, abs(exp))
            assert gm.gamma2[i] == pytest.approx(exp, rel=1e-13)
            if exp > 0:
                assert gm.propagating[i] and gm.diag[i].real > 0 and gm.diag[i].imag == 0
            else:
                assert not gm.propagating[i] and gm.diag[i].real == 0 and gm.diag[i].imag > 0
            assert abs(gm.diag[i] * gm.inv_diag[i] - 1.0) <= 1e-14


def test_specular_propagates(oracle):  # :108-115
    rods = fields.rods1(oracle)
    for t0 in (0.5, 5.0, 45.0, 89.0):
        gm = fields.scalar_gamma(oracle, 3.0, t0, rods)
        assert gm.propagating[0]
        assert gm.diag[0].real == pytest.approx(3.0 * math.sin(t0 * math.pi / 180), rel=1e-13)


def test_grazing_rejected(oracle):  # :117-127
    lat = fields.rect_lattice(oracle)
    b2 = np.linalg.norm(lat.b2())
    t0 = 40.0
    gamma = b2 / (1.0 - math.cos(t0 * math.pi / 180))
    rods = oracle.RodSet.build(lat, 1.05 * b2)
    with pytest.raises(oracle.ConfigError):
        oracle.GammaMatrix.build(rods, oracle.BeamGeometry(gamma, t0, 90.0))


# ---- EXTENSION: first-N truncation (SURVEY.md finding 4)
@pytest.mark.parametrize("a", [3.84, 19.2])
def test_first_n_is_prefix_of_reference_order(oracle, a):
    lat = oracle.Lattice2D((a, 0.0), (a * math.cos(2 * math.pi / 3), a * math.sin(2 * math.pi / 3)))
    big = oracle.RodSet.build(lat, 2 * math.pi / a * 12)
    for n in (1, 13, 15, 31, 63, 127):
        r = oracle.RodSet.build_first(lat, n)
        assert r.size() == n
        assert np.array_equal(r.m, big.m[:n])
        assert np.array_equal(r.k, big.k[:n])


def test_first_n_equals_cutoff_build_on_shells(oracle):
    a = 3.84
    lat = oracle.Lattice2D((a, 0.0), (a * math.cos(2 * math.pi / 3), a * math.sin(2 * math.pi / 3)))
    for n in (13, 31, 127):
        first = oracle.RodSet.build_first(lat, n)
        shell = oracle.RodSet.build(lat, first.cutoff * (1 + 1e-9))
        assert shell.size() == n
        assert np.array_equal(shell.diff_index, first.diff_index)
        assert np.array_equal(shell.diff_m, first.diff_m)


def test_beam_from_energy(oracle):
    g, gl = oracle.beam_from_energy(10000.0)
    assert g == pytest.approx(51.4817, abs=2e-4)
    assert gl == pytest.approx(1.019569, abs=1e-6)
    g, gl = oracle.beam_from_energy(15000.0)
    assert g == pytest.approx(63.2045, abs=2e-4)
