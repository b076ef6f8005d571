"""Oracle pinning: potential fields, atom-potential extension, slicing and
node tables. Ports proj/tests/test_potential.cpp:11-105 and
proj/tests/test_slicing_stages.cpp:10-70."""
import math

import numpy as np
import pytest

import fields


def test_field_validation(oracle):  # test_potential.cpp:11-27
    PF = oracle.PotentialField
    with pytest.raises(oracle.ConfigError):
        PF.zero(0.0)
    with pytest.raises(oracle.ConfigError):
        PF.zero(1.0)
    with pytest.raises(oracle.ConfigError):
        PF.gaussian_layers(-5.0, [(-1.0, 0.3, 0.0, 1.0, 0.0)])
    with pytest.raises(oracle.ConfigError):
        PF.gaussian_layers(-5.0, [(-1.0, 0.3, 1.0, 1.0, -0.1)])
    with pytest.raises(oracle.ConfigError):
        PF.gaussian_layers(-5.0, [(-1.0, 0.3, 1.0, 1.0, 0.0)], 6.0)
    with pytest.raises(oracle.ConfigError):
        PF.tabulated(-5.0, [0.0, -5.0], [((0, 0), [1, 1])])
    with pytest.raises(oracle.ConfigError):
        PF.tabulated(-5.0, [-4.0, 0.0], [((0, 0), [1, 1])])
    with pytest.raises(oracle.ConfigError):
        PF.tabulated(-5.0, [-5.0, 0.0], [((0, 0), [1])])


def test_gaussian_layer_formula(oracle):  # test_potential.cpp:29-49
    rods = fields.rods11(oracle)
    layer = (-2.0, -0.4, 1.7, 0.9, 0.12)
    u = oracle.BoundPotential(oracle.PotentialField.gaussian_layers(-8.0, [layer]), rods)
    z = -3.3
    U = u.eval(z)
    k = rods.k
    for j in range(rods.size()):
        for kk in range(rods.size()):
            dk2 = np.sum((k[j] - k[kk]) ** 2)
            exp = complex(layer[1], layer[1] * layer[4]) * math.exp(-dk2 / (2 * layer[2] ** 2)) * math.exp(
                -((z - layer[0]) ** 2) / (2 * layer[3] ** 2))
            assert abs(U[j, kk] - exp) <= 1e-15
    assert U[1, 0] == U[0, 2]


def test_zero_field(oracle):  # :51-56
    u = oracle.BoundPotential(oracle.PotentialField.zero(-4.0), fields.rods1(oracle))
    assert np.linalg.norm(u.eval(-1.0)) == 0.0


def test_tabulated_linear_exact(oracle):  # :58-71
    grid = [-6.0, -4.5, -2.0, -0.5, 0.0]
    vals = [complex(0.3 + 0.1 * z, -0.05 * z) for z in grid]
    u = oracle.BoundPotential(oracle.PotentialField.tabulated(-6.0, grid, [((0, 0), vals)]), fields.rods1(oracle))
    for z in (-6.0, -5.1, -4.5, -3.3, -2.0, -1.7, -0.25, 0.0):
        assert abs(u.eval(z)[0, 0] - complex(0.3 + 0.1 * z, -0.05 * z)) <= 1e-13


def test_tabulated_needs_all_differences(oracle):  # :73-80
    f = oracle.PotentialField.tabulated(-5.0, [-5.0, 0.0], [((0, 0), [1, 1])])
    with pytest.raises(oracle.ConfigError):
        oracle.BoundPotential(f, fields.rods11(oracle))


def test_domain_and_periodic_extension(oracle):  # :82-95
    rods = fields.rods1(oracle)
    layer = (-1.0, -0.5, 1.5, 0.4, 0.0)
    u = oracle.BoundPotential(oracle.PotentialField.gaussian_layers(-4.0, [layer], 2.0), rods)
    with pytest.raises(oracle.DomainError):
        u.eval(0.5)
    assert abs(u.eval(-5.0)[0, 0] - u.eval(-3.0)[0, 0]) <= 1e-15
    assert abs(u.eval(-9.0)[0, 0] - u.eval(-3.0)[0, 0]) <= 1e-15
    ub = oracle.BoundPotential(oracle.PotentialField.gaussian_layers(-4.0, [layer]), rods)
    with pytest.raises(oracle.DomainError):
        ub.eval(-4.5)


def test_layered_field_absorbing(oracle):  # :97-105
    u = oracle.BoundPotential(fields.layered_field(oracle), fields.rods11(oracle))
    for z in np.arange(-9.5, -0.5, 0.37):
        c = u.eval(z)[0, 0]
        if abs(c) > 1e-6:
            assert c.imag < 0.0


# ---- EXTENSION: atom potential
def _atom_field(oracle, sign, absorption=0.1):
    a = 3.84
    xyz = np.array([[0.0, 0.0, -2.0], [a / 2, a * math.sqrt(3) / 6, -2.8], [0.3, 0.1, -5.1]])
    ff_a = np.array([[0.5, 1.2, 0.8, 0.3], [1.9, 0.4, 0.2, 1.1]])
    ff_b = np.array([[0.7, 4.0, 12.0, 35.0], [1.0, 2.0, 9.0, 30.0]])
    area = a * a * math.sin(2 * math.pi / 3)
    f = oracle.PotentialField.atoms(-8.0, xyz, np.array([0, 1, 0], np.int32), np.array([0.5, 0.7, 0.3]), ff_a, ff_b,
                                    area, 1.0195, sign, absorption)
    lat = oracle.Lattice2D((a, 0.0), (a * math.cos(2 * math.pi / 3), a * math.sin(2 * math.pi / 3)))
    return f, oracle.RodSet.build_first(lat, 13), (xyz, ff_a, ff_b, area)


@pytest.mark.parametrize("sign", [1.0, -1.0])
def test_atom_potential_formula(oracle, sign):
    f, rods, (xyz, ff_a, ff_b, area) = _atom_field(oracle, sign)
    u = oracle.BoundPotential(f, rods)
    B = [0.5, 0.7, 0.3]
    spc = [0, 1, 0]
    for z in (-7.9, -5.0, -2.4, -0.1):
        c = u.eval_coeffs(z)
        for d, g in enumerate(rods.diff):
            V = 0j
            for ia in range(3):
                for i in range(4):
                    bp = ff_b[spc[ia], i] + B[ia]
                    V += (ff_a[spc[ia], i] * 2 * math.sqrt(math.pi) / math.sqrt(bp)
                          * math.exp(-bp * (g @ g) / (16 * math.pi ** 2))
                          * np.exp(-1j * (g @ xyz[ia, :2]))
                          * math.exp(-4 * math.pi ** 2 * (z - xyz[ia, 2]) ** 2 / bp))
            exp = complex(sign, -0.1) * 1.0195 * 4 * math.pi / area * V
            assert abs(c[d] - exp) <= 1e-13 * max(1.0, abs(exp))


def test_atom_potential_hermitian_and_absorbing(oracle):
    f, rods, _ = _atom_field(oracle, 1.0, absorption=0.0)
    U = oracle.BoundPotential(f, rods).eval(-2.5)
    assert np.allclose(U, U.conj().T, atol=1e-14)  # u(-g) = conj u(g) without absorption
    for sign in (1.0, -1.0):
        f, rods, _ = _atom_field(oracle, sign)
        u = oracle.BoundPotential(f, rods)
        for z in (-5.0, -2.8, -2.0):
            assert u.eval(z)[0, 0].imag < 0.0  # Im U < 0 absorbing (potential.hpp:15-16)


# ---- slicing / stages (test_slicing_stages.cpp)
def test_slicing_endpoints(oracle):  # :10-20
    plan = oracle.SlicingPlan.with_target_dz(-9.7, 0.013)
    assert plan.z(0) == -9.7 and plan.z(plan.count) == 0.0
    assert plan.count == 746
    assert plan.h * plan.count == pytest.approx(9.7, rel=1e-15)
    p2 = oracle.SlicingPlan.with_count(-5.0, 10)
    assert p2.h == 0.5
    assert all(p2.z(i) < p2.z(i + 1) for i in range(1, 10))


def test_node_schedules(oracle):  # :22-31
    s = oracle.schedule_from_fracs([1.0 - 1e-15, 0.5, 0.0, 0.5 + 1e-14, 1e-16])
    assert s.frac == [0.0, 0.5, 1.0] and s.endpoint_pair()
    assert not oracle.midpoint_schedule().endpoint_pair()
    assert oracle.rk4_schedule().endpoint_pair()


def test_shared_endpoints_bitwise(oracle):  # :33-40
    w = oracle.StepWindow.over(-7.3, 0.0, 613)
    s = oracle.rk4_schedule()
    for i in range(0, w.count - 1, 61):
        assert oracle.node_z(w, i, 2, s) == oracle.node_z(w, i + 1, 0, s)
    assert oracle.node_z(w, 0, 0, s) == -7.3
    assert oracle.node_z(w, w.count - 1, 2, s) == 0.0


def test_table_equals_direct(oracle):  # :42-59
    u = oracle.BoundPotential(fields.layered_field(oracle), fields.rods11(oracle))
    w = oracle.StepWindow.over(-10.0, 0.0, 157)
    for s in (oracle.midpoint_schedule(), oracle.rk4_schedule(), oracle.schedule_from_fracs([0.0, 0.21, 0.58, 1.0])):
        t = oracle.UTable(u, w, s)
        for i in (0, 1, 77, 155, 156):
            for m in range(s.nodes()):
                assert np.array_equal(t.at(i, m), u.eval(oracle.node_z(w, i, m, s)))


def test_table_bytes(oracle):  # :61-70
    mid = oracle.midpoint_schedule()
    one = oracle.UTable.bytes_estimate(11, 1, mid)
    assert one >= 11 * 11 * 16
    assert oracle.UTable.bytes_estimate(11, 100, mid) >= 100 * one
    assert oracle.UTable.bytes_estimate(11, 100, oracle.rk4_schedule()) <= 201 * one + one
