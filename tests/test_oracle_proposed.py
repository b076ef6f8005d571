"""Oracle pinning: the proposed (matrix-ODE) solver. Ports
proj/tests/test_proposed.cpp:29-298 and acceptance c01/c02/c03/c05/c07
(proj/tests/acceptance.cpp:69-271). Closed forms: Fresnel slab/interface
(oracles.hpp:38-49)."""
import math

import numpy as np
import pytest

import fields

INF = float("inf")


def rand_c(rng, n, m=None, scale=1.0):
    m = n if m is None else m
    return scale * (rng.uniform(-1, 1, (n, m)) + 1j * rng.uniform(-1, 1, (n, m)))


def test_coefficient_tables(oracle):  # :29-43
    S = oracle.StepperSpec
    for s in (S.rk4(), S.sp4(), S.sp6()):
        s.validate()
    assert len(S.sp4().drift) == 6 and len(S.sp4().kick) == 7
    assert len(S.sp6().drift) == 11 and len(S.sp6().kick) == 12
    with pytest.raises(oracle.ConfigError):
        S.by_name("magnus9")
    bad = S.splitting("sp4", oracle.SplitVariant.BAB, S.sp4().drift, S.sp4().kick)
    k = list(bad.kick)
    k[0] += 0.01
    bad.kick = k
    with pytest.raises(oracle.ConfigError):
        bad.validate()


def test_kick_schedules(oracle):  # proposed.cpp:62-100 (SPEC: kick heights = accumulated drifts)
    for name, nodes in (("sp4", 7), ("sp6", 12)):
        spec = oracle.StepperSpec.by_name(name)
        ks = oracle.kick_schedule(spec)
        assert ks.nodes.nodes() == nodes and ks.nodes.endpoint_pair()
        assert len(ks.occ2node) == len(spec.kick)
        acc = np.concatenate([[0.0], np.cumsum(spec.drift)])
        for occ, node in enumerate(ks.occ2node):
            assert abs(ks.nodes.frac[node] - acc[occ]) < 1e-12


def test_tau_rho_round_trip(oracle):  # :45-59
    rng = np.random.default_rng(41)
    rods = fields.rods11(oracle)
    gm = fields.scalar_gamma(oracle, fields.K_GAMMA11, 12.0, rods)
    st = oracle.PropagationState(rand_c(rng, 11), rand_c(rng, 11), -1.0)
    T, R = oracle.to_tau_rho(gm, st)
    back = oracle.from_tau_rho(gm, T, R, st.z)
    assert np.linalg.norm(back.Q - st.Q) <= 1e-13 * np.linalg.norm(st.Q)
    assert np.linalg.norm(back.P - st.P) <= 1e-13 * np.linalg.norm(st.P)


def test_initial_state(oracle):  # :61-77
    rng = np.random.default_rng(43)
    rods = fields.rods11(oracle)
    gm = fields.scalar_gamma(oracle, fields.K_GAMMA11, 12.0, rods)
    R0 = rand_c(rng, 11, scale=0.3)
    st = oracle.initial_state(gm, R0, -10.0)
    assert st.z == -10.0
    T, R = oracle.to_tau_rho(gm, st)
    assert np.linalg.norm(T - np.eye(11)) <= 1e-13
    assert np.linalg.norm(R - R0) <= 1e-13 * max(1.0, np.linalg.norm(R0))
    assert np.linalg.norm(oracle.extract_reflection(gm, st) - R0) <= 1e-12 * max(1.0, np.linalg.norm(R0))
    v = oracle.initial_state(gm, np.zeros(0, complex), -10.0)
    assert np.linalg.norm(oracle.extract_reflection(gm, v)) <= 1e-14


def test_rhst_invariance_unit(oracle):  # :79-97
    rng = np.random.default_rng(47)
    rods = fields.rods11(oracle)
    gm = fields.scalar_gamma(oracle, fields.K_GAMMA11, 12.0, rods)
    Q = rand_c(rng, 11) + 2.5 * np.eye(11)
    P = rand_c(rng, 11)
    before = oracle.extract_reflection(gm, oracle.PropagationState(Q, P))
    tr = oracle.PropagationState(Q, P)
    assert oracle.apply_rhst(tr, 0.0)
    assert np.linalg.norm(tr.Q - np.eye(11)) == 0.0
    assert np.linalg.norm(oracle.extract_reflection(gm, tr) - before) <= 1e-12 * np.linalg.norm(before)
    Q2 = Q.copy()
    Q2[0, 0] = 1e9
    off = oracle.PropagationState(Q2, P)
    assert not oracle.apply_rhst(off, INF)
    assert off.Q[0, 0] == 1e9


def test_steppers_linear(oracle):  # :99-138
    rng = np.random.default_rng(53)
    rods = fields.rods11(oracle)
    gm = fields.scalar_gamma(oracle, fields.K_GAMMA11, 12.0, rods)
    u = oracle.BoundPotential(fields.layered_field(oracle), rods)
    M = rand_c(rng, 11)
    h, z0 = 0.05, -4.0
    Q, P = rand_c(rng, 11), rand_c(rng, 11)
    g2 = list(gm.gamma2)
    a = oracle.PropagationState(Q, P, z0)
    b = oracle.PropagationState(Q @ M, P @ M, z0)
    U0, Um, U1 = u.eval(z0), u.eval(z0 + h / 2), u.eval(z0 + h)
    oracle.rk4_step(a, h, U0, Um, U1, g2)
    oracle.rk4_step(b, h, U0, Um, U1, g2)
    assert np.linalg.norm(a.Q @ M - b.Q) <= 1e-12 * np.linalg.norm(b.Q)
    assert np.linalg.norm(a.P @ M - b.P) <= 1e-12 * np.linalg.norm(b.P)
    for name in ("sp4", "sp6"):
        spec = oracle.StepperSpec.by_name(name)
        ks = oracle.kick_schedule(spec)
        mats = [u.eval(z0 + h * f) for f in ks.nodes.frac]
        Us = [mats[o] for o in ks.occ2node]
        aa = oracle.PropagationState(Q, P, z0)
        bb = oracle.PropagationState(Q @ M, P @ M, z0)
        oracle.splitting_step(aa, h, spec, Us, g2)
        oracle.splitting_step(bb, h, spec, Us, g2)
        assert np.linalg.norm(aa.Q @ M - bb.Q) <= 1e-12 * np.linalg.norm(bb.Q)
        assert np.linalg.norm(aa.P @ M - bb.P) <= 1e-12 * np.linalg.norm(bb.P)


def _const_setup(oracle, u0):
    gamma, theta0, z_e = 2.0, 30.0, -7.0
    g = gamma * math.sin(theta0 * math.pi / 180)
    rods = fields.rods1(oracle)
    gm = fields.scalar_gamma(oracle, gamma, theta0, rods)
    u = oracle.BoundPotential(fields.constant_field(oracle, u0, z_e), rods)
    return u, gm, z_e, fields.fresnel_slab_rho0(g, u0, z_e)


def test_constant_potential_closed_form(oracle):  # :140-158
    u, gm, z_e, exp = _const_setup(oracle, complex(-0.8, -0.2))
    plan = oracle.SlicingPlan.with_target_dz(z_e, 0.01)
    S = oracle.StepperSpec
    r6, _ = oracle.solve_proposed(u, gm, plan, S.sp6())
    assert abs(r6[0] - exp) <= 1e-6 * abs(exp)
    for s in (S.sp4(), S.rk4()):
        r, _ = oracle.solve_proposed(u, gm, plan, s)
        assert abs(r[0] - exp) <= 1e-4 * abs(exp)


def test_empirical_orders(oracle):  # :160-187
    u, gm, z_e, exp = _const_setup(oracle, complex(-0.9, -0.25))

    def orders(spec, ladder, lo, hi):
        hs, errs = [], []
        for n in ladder:
            r, _ = oracle.solve_proposed(u, gm, oracle.SlicingPlan.with_count(z_e, n), spec)
            hs.append(-z_e / n)
            errs.append(abs(r[0] - exp) / abs(exp))
        return fields.fit_order(hs, errs, lo, hi, 4)

    fine = [10, 14, 20, 28, 40, 56, 80, 112, 160, 224, 320]
    coarse = [6, 8, 10, 14, 20, 28, 40]
    S = oracle.StepperSpec
    assert orders(S.rk4(), fine, 1e-12, 1e-3) == pytest.approx(4.0, rel=0.12)
    assert orders(S.sp4(), fine, 1e-12, 1e-3) == pytest.approx(4.0, rel=0.12)
    assert orders(S.sp6(), coarse, 1e-13, 1e-2) == pytest.approx(6.0, rel=0.12)


def test_thresholds_agree_short_domain(oracle):  # :189-209 and acceptance c05 (:183-200)
    rods = fields.rods11(oracle)
    u = oracle.BoundPotential(oracle.PotentialField.gaussian_layers(-2.0, [(-1.0, -0.35, 1.8, 0.4, 0.1)]), rods)
    plan = oracle.SlicingPlan.with_target_dz(-2.0, 0.005)
    for theta0 in (12.0, 20.0):
        gm = fields.scalar_gamma(oracle, fields.K_GAMMA11, theta0, rods)
        sols = []
        for th in (0.0, 1000.0, INF):
            r, n = oracle.solve_proposed(u, gm, plan, oracle.StepperSpec.sp6(), th)
            sols.append(r)
            if th == 0.0:
                assert n == plan.count
            if th == INF:
                assert n == 0
        scale = np.linalg.norm(sols[1])
        for i in range(3):
            for j in range(i + 1, 3):
                assert np.linalg.norm(sols[i] - sols[j]) <= 1e-10 * scale


def test_deep_domain(oracle):  # :211-238 and acceptance c07 (:238-271)
    rods = fields.rods11(oracle)
    gm = fields.scalar_gamma(oracle, fields.K_GAMMA11, 5.0, rods)
    u = oracle.BoundPotential(fields.deep_field(oracle), rods)
    S = oracle.StepperSpec
    ref, _ = oracle.solve_proposed(u, gm, oracle.SlicingPlan.with_target_dz(-50.0, 0.002), S.sp6(), 1000.0)
    plan = oracle.SlicingPlan.with_target_dz(-50.0, 0.02)
    good, n = oracle.solve_proposed(u, gm, plan, S.sp6(), 1000.0)
    assert n > 0
    assert np.linalg.norm(good - ref) <= 1e-6 * np.linalg.norm(ref)
    failed = False
    try:
        raw, _ = oracle.solve_proposed(u, gm, plan, S.sp6(), INF)
        failed = (not np.all(np.isfinite(raw))) or np.linalg.norm(raw - ref) > 1e-3 * np.linalg.norm(ref)
    except oracle.SolverError:
        failed = True
    assert failed


def test_table_vs_direct_bitwise(oracle):  # :240-252
    rods = fields.rods11(oracle)
    gm = fields.scalar_gamma(oracle, fields.K_GAMMA11, 9.0, rods)
    u = oracle.BoundPotential(fields.layered_field(oracle), rods)
    plan = oracle.SlicingPlan.with_target_dz(-10.0, 0.05)
    for name in ("rk4", "sp4", "sp6"):
        spec = oracle.StepperSpec.by_name(name)
        a, _ = oracle.solve_proposed(u, gm, plan, spec, use_table=True)
        b, _ = oracle.solve_proposed(u, gm, plan, spec, use_table=False)
        assert np.array_equal(a, b)


def test_bulk_vs_fresnel_interface(oracle):  # :281-298 (proposed side)
    gamma, theta0 = 2.0, 30.0
    g = gamma * math.sin(theta0 * math.pi / 180)
    u0 = complex(-0.6, -0.3)
    rods = fields.rods1(oracle)
    gm = fields.scalar_gamma(oracle, gamma, theta0, rods)
    f = oracle.PotentialField.tabulated(-2.0, [-2.0, 0.0], [((0, 0), [u0, u0])], 1.0)
    u = oracle.BoundPotential(f, rods)
    Rp = oracle.compute_bulk_reflection_proposed(u, gm, 0.01, oracle.StepperSpec.sp6())
    exp = fields.fresnel_interface_r(g, u0)
    assert abs(Rp[0, 0] - exp) <= 1e-8 * abs(exp)


def test_acceptance_c01_zero_potential(oracle):  # acceptance.cpp:69-94 (stepper methods)
    rods = fields.rods1(oracle)
    u = oracle.BoundPotential(oracle.PotentialField.zero(-1.0), rods)
    plan = oracle.SlicingPlan.with_target_dz(-1.0, 5e-4)
    worst_rho = worst_eta = 0.0
    for t0 in range(1, 70):
        gm = oracle.GammaMatrix.build(rods, oracle.BeamGeometry(1.0, float(t0), 0.0))
        for m in ("rk4", "sp4", "sp6"):
            r, _ = oracle.solve_proposed(u, gm, plan, oracle.StepperSpec.by_name(m))
            worst_rho = max(worst_rho, np.abs(r).max())
            worst_eta = max(worst_eta, np.abs(oracle.intensity(r, gm)).max())
    assert worst_rho <= 1e-12 and worst_eta <= 1e-24


def test_acceptance_c02_fresnel_step(oracle):  # acceptance.cpp:99-118 (sp6 side)
    theta0 = math.asin(0.1) * 180 / math.pi
    u0 = complex(-2.0, 0.0)
    rods = fields.rods1(oracle)
    gm = oracle.GammaMatrix.build(rods, oracle.BeamGeometry(10.0, theta0, 0.0))
    g = gm.diag[0].real
    target = abs(fields.fresnel_interface_r(g, u0))
    u = oracle.BoundPotential(fields.constant_field(oracle, u0, -12.0), rods)
    r, _ = oracle.solve_proposed(u, gm, oracle.SlicingPlan.with_target_dz(-12.0, 0.01), oracle.StepperSpec.sp6())
    assert abs(abs(r[0]) - target) <= 1e-6


@pytest.mark.slow
def test_acceptance_c03_orders(oracle):  # acceptance.cpp:123-159 (stepper methods)
    rods = fields.rods11(oracle)
    field = fields.smooth_field(oracle)
    u = oracle.BoundPotential(field, rods)
    gm = oracle.GammaMatrix.build(rods, oracle.BeamGeometry(fields.K_GAMMA11, 30.0, 0.0))
    ref, _ = oracle.solve_proposed(u, gm, oracle.SlicingPlan.with_target_dz(-10.0, 0.001), oracle.StepperSpec.sp6())
    dzs = [0.010, 0.015, 0.022, 0.033, 0.047, 0.068, 0.10, 0.15, 0.22, 0.33, 0.47, 0.68]  # driver.cpp:10-11
    want = {"rk4": 4.0, "sp4": 4.0, "sp6": 6.0}
    for m, order in want.items():
        hs, errs = [], []
        for dz in dzs:
            plan = oracle.SlicingPlan.with_target_dz(-10.0, dz)
            r, _ = oracle.solve_proposed(u, gm, plan, oracle.StepperSpec.by_name(m))
            hs.append(plan.h)
            errs.append(np.linalg.norm(r - ref) / np.linalg.norm(ref))
        slope = fields.fit_order(hs, errs, 1e-13, 5e-5) if m == "sp6" else fields.fit_order(hs, errs)
        assert abs(slope - order) <= 0.5, (m, slope)
