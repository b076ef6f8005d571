"""GPU parity: the device path (C-ABI -> sm_100a kernels) against the
reference itself (oracle/_ref: the reference's hot-path sources compiled
verbatim, fixture `ref`) on identical seeded inputs, plus the reference's own
known-answer tests run through the device path. Tolerance (BASELINE.json
north_star): curve_error <= 1e-9 and per-entry relative error
<= 1e-9 on entries above 1e-12 * max eta, complex128 throughout. The one
exception is N = 199 (cfg3), where two correct CPU builds at the same RHST
schedule (the reference vs the restatement) already differ by 8.6e-9 per
entry: see test_config3_subset_parity."""
import math

import numpy as np
import pytest

import fields as F
import harness as H
import paper_2306_00271_b200 as mb
from paper_2306_00271_b200 import configs

pytestmark = pytest.mark.gpu
TOL = 1e-9


def dev_layered_field():
    return mb.PotentialField.gaussian_layers(-10.0, F.LAYERED_LAYERS)


def dev_rods11():
    return mb.RodSet.build(mb.Lattice2D(*F.RECT), 5.0)


def dev_rods1():
    return mb.RodSet.build(mb.Lattice2D(*F.RECT), 0.5)


def oracle_curve(o, field, rods, gamma, t0, method, dz, threshold=1000.0, threads=4):
    opts = o.SweepOptions()
    opts.method, opts.dz, opts.threads, opts.rhst_threshold = method, dz, threads, threshold
    return o.rocking_curve(field, rods, gamma, o.AngleGrid.validated(t0, [0.0]), opts)


@pytest.mark.parametrize("method", ["rk4", "sp4", "sp6"])
@pytest.mark.parametrize("fsal", [False, True])
def test_layered_field_parity(ref, method, fsal):
    t0 = [2.0, 5.0, 9.0, 12.0, 17.0, 25.0]
    rc = oracle_curve(ref, F.layered_field(ref), F.rods11(ref), F.K_GAMMA11, t0, method, 0.02)
    c = mb.rocking_curve(dev_layered_field(), dev_rods11(), F.K_GAMMA11, mb.AngleGrid.validated(t0, [0.0]),
                         mb.SweepOptions(method=method, dz=0.02, fsal=fsal))
    assert H.curve_err(c.eta, rc.eta) <= TOL
    assert H.entry_rel_err(c.eta, rc.eta) <= TOL
    assert H.entry_abs_err(c.eta, rc.eta) <= 1e-11
    assert np.abs(c.rho - rc.rho).max() <= 1e-10 * np.abs(rc.rho).max()


def test_deep_field_rhst_parity(ref):  # test_proposed.cpp:211-238 domain
    t0 = [3.0, 5.0, 7.0]
    rc = oracle_curve(ref, F.deep_field(ref), F.rods11(ref), F.K_GAMMA11, t0, "sp6", 0.02)
    field = mb.PotentialField.gaussian_layers(-50.0, F.DEEP_LAYERS)
    c = mb.rocking_curve(field, dev_rods11(), F.K_GAMMA11, mb.AngleGrid.validated(t0, [0.0]),
                         mb.SweepOptions(method="sp6", dz=0.02))
    assert (c.status["rhst"] > 0).all()
    assert np.array_equal(c.status["rhst"], rc.rhst)
    assert H.curve_err(c.eta, rc.eta) <= TOL


@pytest.mark.parametrize("threshold", [0.0, 1000.0, math.inf])
def test_threshold_invariance(ref, threshold):  # test_proposed.cpp:189-209
    field = mb.PotentialField.gaussian_layers(-2.0, [(-1.0, -0.35, 1.8, 0.4, 0.1)])
    grid = mb.AngleGrid.validated([12.0, 20.0], [0.0])
    c = mb.rocking_curve(field, dev_rods11(), F.K_GAMMA11, grid,
                         mb.SweepOptions(method="sp6", dz=0.005, rhst_threshold=threshold))
    base = mb.rocking_curve(field, dev_rods11(), F.K_GAMMA11, grid, mb.SweepOptions(method="sp6", dz=0.005))
    assert np.linalg.norm(c.rho - base.rho) <= 1e-10 * np.linalg.norm(base.rho)
    if threshold == 0.0:
        assert (c.status["rhst"] == 400).all()
    if math.isinf(threshold):
        assert (c.status["rhst"] == 0).all()


def test_fresnel_slab_closed_form():  # test_proposed.cpp:140-158
    gamma, theta0, z_e, u0 = 2.0, 30.0, -7.0, complex(-0.8, -0.2)
    g = gamma * math.sin(math.radians(theta0))
    exp = F.fresnel_slab_rho0(g, u0, z_e)
    field = mb.PotentialField.tabulated(z_e, [z_e, 0.0], [((0, 0), [u0, u0])])
    grid = mb.AngleGrid.validated([theta0], [0.0])
    for method, tol in (("sp6", 1e-6), ("sp4", 1e-4), ("rk4", 1e-4)):
        c = mb.rocking_curve(field, dev_rods1(), gamma, grid, mb.SweepOptions(method=method, dz=0.01))
        assert abs(c.rho[0, 0] - exp) <= tol * abs(exp)


def test_empirical_order_sp6():  # test_proposed.cpp:160-187 (sp6 ladder)
    gamma, theta0, z_e, u0 = 2.0, 30.0, -7.0, complex(-0.9, -0.25)
    g = gamma * math.sin(math.radians(theta0))
    exp = F.fresnel_slab_rho0(g, u0, z_e)
    field = mb.PotentialField.tabulated(z_e, [z_e, 0.0], [((0, 0), [u0, u0])])
    grid = mb.AngleGrid.validated([theta0], [0.0])
    hs, errs = [], []
    for n in (6, 8, 10, 14, 20, 28, 40):
        c = mb.rocking_curve(field, dev_rods1(), gamma, grid, mb.SweepOptions(method="sp6", slices=n))
        hs.append(-z_e / n)
        errs.append(abs(c.rho[0, 0] - exp) / abs(exp))
    assert F.fit_order(hs, errs, 1e-13, 1e-2, 4) == pytest.approx(6.0, rel=0.12)


def test_zero_potential():  # acceptance.cpp:69-94
    field = mb.PotentialField.zero(-1.0)
    grid = mb.AngleGrid.validated([float(t) for t in range(1, 70)], [0.0])
    for m in ("rk4", "sp4", "sp6"):
        c = mb.rocking_curve(field, dev_rods1(), 1.0, grid, mb.SweepOptions(method=m, dz=5e-4))
        assert np.abs(c.rho).max() <= 1e-12 and np.abs(c.eta).max() <= 1e-24


def test_breakdown_surfaces_with_step(ref):  # test_sweep.cpp:90-105
    layers = [(-1.0 - 2.0 * i, -0.22, 2.2, 0.7, 0.08) for i in range(75)]
    field = mb.PotentialField.gaussian_layers(-150.0, layers)
    grid = mb.AngleGrid.validated([3.0, 5.0], [0.0])
    with pytest.raises(mb.BreakdownError) as ei:
        mb.rocking_curve(field, dev_rods11(), F.K_GAMMA11, grid,
                         mb.SweepOptions(method="sp6", dz=0.02, rhst_threshold=math.inf))
    assert ei.value.step is not None and 0 < ei.value.step < 7500
    with pytest.raises(ref.BreakdownError) as eo:
        ref.rocking_curve(ref.PotentialField.gaussian_layers(-150.0, layers), F.rods11(ref), F.K_GAMMA11,
                          ref.AngleGrid.validated([3.0], [0.0]), _opts(ref, "sp6", 0.02, math.inf))
    assert ei.value.step == eo.value.step


def _opts(o, method, dz, thr):
    s = o.SweepOptions()
    s.method, s.dz, s.rhst_threshold = method, dz, thr
    return s


def test_flux_bound():  # acceptance.cpp:308-319
    grid = mb.AngleGrid.validated([float(t) for t in range(1, 70)], [0.0])
    c = mb.rocking_curve(dev_layered_field(), dev_rods11(), F.K_GAMMA11, grid, mb.SweepOptions(method="sp4", dz=0.02))
    assert c.eta.sum(axis=1).max() <= 1.0 + 1e-8


def test_custom_aba_stepper_parity(ref):
    # a symmetric ABA splitting (Strang-type 2-stage) through both paths
    drift, kick = [0.25, 0.5, 0.25], [0.5, 0.5]
    t0 = [4.0, 11.0]
    o = ref.SweepOptions()
    o.dz, o.threads = 0.02, 2
    o.set_splitting("aba2", "ABA", drift, kick)  # StepperSpec::splitting, proposed.hpp:35-36
    refs = ref.rocking_curve(F.layered_field(ref), F.rods11(ref), F.K_GAMMA11, ref.AngleGrid.validated(t0, [0.0]),
                             o).rho
    spec = mb.StepperSpec.splitting("aba2", mb.StepperSpec.ABA, drift, kick)
    c = mb.rocking_curve(dev_layered_field(), dev_rods11(), F.K_GAMMA11, mb.AngleGrid.validated(t0, [0.0]),
                         mb.SweepOptions(dz=0.02, stepper=spec))
    assert np.abs(c.rho - np.array(refs)).max() <= 1e-10 * np.abs(np.array(refs)).max()


def test_deterministic_bitwise():
    grid = mb.AngleGrid.validated([2.0, 5.0, 8.0, 11.0], [0.0])
    args = (dev_layered_field(), dev_rods11(), F.K_GAMMA11, grid, mb.SweepOptions(method="sp4", dz=0.02))
    a, b = mb.rocking_curve(*args), mb.rocking_curve(*args)
    assert np.array_equal(a.eta, b.eta)
    # a row solved alone equals the same row inside a batch (fixed per-pair arithmetic)
    one = mb.rocking_curve(dev_layered_field(), dev_rods11(), F.K_GAMMA11, mb.AngleGrid.validated([8.0], [0.0]),
                           mb.SweepOptions(method="sp4", dz=0.02))
    assert np.array_equal(one.eta[0], a.eta[2])


# ---------------------------------------------------------------- atom configs
def test_config0_full_parity(ref, oracle):
    w = configs.config0()
    want, rref, rh = H.run_oracle(ref, w)
    eta, rho, st = H.run_device(w)
    assert (st["code"] == 0).all()
    assert np.array_equal(st["rhst"], rh)
    H.assert_parity(eta, want, H.run_oracle(oracle, w)[0])


def test_config1_subset_parity(ref, oracle):
    w = configs.config1().subset(theta0=[0.1, 1.0, 2.5, 6.1])
    want, rref, rh = H.run_oracle(ref, w, threads=4)
    alt = H.run_oracle(oracle, w, threads=4)[0]
    for fsal in (False, True):
        eta, rho, st = H.run_device(w, fsal=fsal)
        assert np.array_equal(st["rhst"], rh), fsal
        H.assert_parity(eta, want, alt)


def test_config2_subset_parity(ref, oracle):
    w = configs.config2(n_structures=3).subset(theta0=[0.5, 2.0, 4.4, 6.5])
    want, _, rh = H.run_oracle(ref, w, threads=4)
    eta, _, st = H.run_device(w)
    assert np.array_equal(st["rhst"], rh)
    H.assert_parity(eta, want, H.run_oracle(oracle, w, threads=4)[0])


@pytest.mark.parametrize("n,method", [(15, "rk4"), (15, "sp6"), (31, "sp6"), (63, "sp6")])
def test_config4_subset_parity(ref, oracle, n, method):
    w = configs.config4(n, method, n_structures=2).subset(theta0=[0.5, 3.3, 6.8], slices=100)
    want, _, rh = H.run_oracle(ref, w, threads=4)
    eta, _, st = H.run_device(w)
    assert np.array_equal(st["rhst"], rh)
    H.assert_parity(eta, want, H.run_oracle(oracle, w, threads=4)[0])


# ---------------------------------------------------------------- large-N batched path
# Thinner slabs at the configs' own step (h = 0.016 A for cfg4, 0.01 for cfg3)
# keep the oracle cheap; a coarse h breaks both paths down by design.
@pytest.mark.parametrize("n,method,path", [(63, "rk4", 0), (31, "rk4", 2), (61, "sp6", 2), (127, "sp6", 2),
                                           (127, "rk4", 2), (127, "sp6", 3), (127, "rk4", 3), (81, "sp6", 3),
                                           (143, "sp6", 3), (143, "rk4", 2)])
def test_large_path_parity(ref, oracle, n, method, path):
    w = configs.config4(n, method, n_structures=2).subset(theta0=[0.5, 4.1], slices=150, z_bottom=-2.4)
    want, _, rh = H.run_oracle(ref, w, threads=4)
    eta, _, st = H.run_device(w, path=path)
    assert (st["code"] == 0).all()
    assert np.array_equal(st["rhst"], rh)
    H.assert_parity(eta, want, H.run_oracle(oracle, w, threads=4)[0])


@pytest.mark.parametrize("cfg,method", [(1, "sp6"), (4, "rk4")])
def test_large_path_matches_resident(cfg, method):
    if cfg == 1:
        w = configs.config1().subset(theta0=[0.3, 2.0, 5.5], slices=120)
    else:
        w = configs.config4(31, "rk4", n_structures=2).subset(theta0=[0.5, 2.5, 6.0], slices=200, z_bottom=-3.2)
    a, _, sa = H.run_device(w, method=method, fsal=True, path=1)
    b, _, sb = H.run_device(w, method=method, fsal=True, path=2)
    assert H.curve_err(b, a) <= 1e-11
    assert np.array_equal(sa["rhst"], sb["rhst"])


@pytest.mark.parametrize("path", [2, 3, 4])
def test_config3_subset_parity(ref, oracle, path):
    w = configs.config3().subset(theta0=[0.5, 3.5], slices=300, z_bottom=-3.0)
    want, _, rh = H.run_oracle(ref, w, threads=2)
    eta, _, st = H.run_device(w, path=path)
    assert (st["code"] == 0).all()
    assert np.array_equal(st["rhst"], rh)
    # N=199: the restatement against the reference build at the same RHST
    # schedule differs by 8.6e-9 per entry above 1e-10 max eta (curve_error
    # 1.9e-11), the case's conditioning; assert_parity takes that floor
    H.assert_parity(eta, want, H.run_oracle(oracle, w, threads=2)[0], abs_tol=1e-10)


@pytest.mark.parametrize("method,path", [("rk4", 2), ("sp6", 3)])
def test_n255_parity(ref, oracle, method, path):
    w = configs.config4(255, method, n_structures=1).subset(theta0=[1.7], slices=60, z_bottom=-0.96)
    want, _, rh = H.run_oracle(ref, w, threads=1)
    eta, _, st = H.run_device(w, path=path)
    assert (st["code"] == 0).all()
    assert np.array_equal(st["rhst"], rh)
    H.assert_parity(eta, want, H.run_oracle(oracle, w, threads=1)[0])


@pytest.mark.parametrize("n,method", [(127, "sp6"), (199, "sp6"), (127, "rk4")])
def test_cluster_matches_batched(n, method):
    """Two independent large-N designs (state resident in a CTA cluster vs in
    HBM) on the same batch; the RHST schedules coincide."""
    w = configs.config4(n, method, n_structures=2).subset(theta0=[0.5, 2.5, 6.0], slices=200, z_bottom=-3.2)
    a, _, sa = H.run_device(w, path=3)
    b, _, sb = H.run_device(w, path=2)
    assert (sa["code"] == 0).all() and (sb["code"] == 0).all()
    assert np.array_equal(sa["rhst"], sb["rhst"])
    assert H.curve_err(a, b) <= 1e-9


@pytest.mark.parametrize("n,method", [(127, "sp6"), (199, "sp6"), (127, "rk4"), (81, "sp6")])
def test_cooperative_groups_match_clusters(n, method):
    """The cluster kernel as persistent cooperative CTA groups (path 4: L2
    exchange, counter barriers, several pairs per group) computes exactly what
    the thread-block clusters compute (path 3): same arithmetic, same
    reduction orders. 26 pairs: more than one round of groups at every N.""" 
    w = configs.config4(n, method, n_structures=2).subset(theta0=[0.5 + 0.45 * i for i in range(13)], slices=60,
                                                         z_bottom=-0.96)
    a, ra, sa = H.run_device(w, path=3)
    b, rb, sb = H.run_device(w, path=4)
    assert (sa["code"] == 0).all() and (sb["code"] == 0).all()
    assert np.array_equal(sa["rhst"], sb["rhst"])
    # two instantiations: the compiler may contract a few products into FMAs
    # differently, so roundoff-level agreement, and each bitwise deterministic
    assert H.curve_err(b, a) <= 1e-13
    c, rc, sc = H.run_device(w, path=4)
    assert np.array_equal(b, c) and np.array_equal(rb, rc)


# ---------------------------------------------------------------- bulk seed
def test_bulk_fresnel_interface():  # test_proposed.cpp:281-298 through the device path
    """A constant potential continued periodically below z_bottom is a
    semi-infinite medium: the seeded solve gives the Fresnel interface r."""
    gamma, theta0, u0 = 2.0, 30.0, complex(-0.6, -0.3)
    g = gamma * math.sin(math.radians(theta0))
    exp = F.fresnel_interface_r(g, u0)
    field = mb.PotentialField.tabulated(-2.0, [-2.0, 0.0], [((0, 0), [u0, u0])], bulk_period=1.0)
    c = mb.rocking_curve(field, dev_rods1(), gamma, mb.AngleGrid.validated([theta0], [0.0]),
                         mb.SweepOptions(method="sp6", dz=0.01))
    assert abs(c.rho[0, 0] - exp) <= 1e-8 * abs(exp)


@pytest.mark.parametrize("method", ["rk4", "sp4", "sp6"])
def test_bulk_layered_parity(ref, method):
    t0 = [2.0, 7.0, 15.0]
    of = ref.PotentialField.gaussian_layers(-10.0, F.LAYERED_LAYERS, 5.0)
    rc = oracle_curve(ref, of, F.rods11(ref), F.K_GAMMA11, t0, method, 0.05)
    field = mb.PotentialField.gaussian_layers(-10.0, F.LAYERED_LAYERS, bulk_period=5.0)
    c = mb.rocking_curve(field, dev_rods11(), F.K_GAMMA11, mb.AngleGrid.validated(t0, [0.0]),
                         mb.SweepOptions(method=method, dz=0.05))
    assert np.array_equal(c.status["rhst"], rc.rhst)
    assert H.curve_err(c.eta, rc.eta) <= TOL
    # R_bulk is defined only to the stopping rule ||dR||_F <= 1e-12 max(1, ||R||_F)
    # (proposed.cpp:334-339): entries 1e-5 below max eta carry that as ~1e-8
    assert H.entry_rel_err(c.eta, rc.eta, floor=1e-6) <= 1e-8
    assert H.entry_rel_err(c.eta, rc.eta, floor=1e-10) <= 1e-7
    assert H.entry_abs_err(c.eta, rc.eta) <= 1e-11


@pytest.mark.parametrize("method", ["rk4", "sp6"])
def test_bulk_atoms_parity(ref, oracle, method):
    w = configs.config0().subset(theta0=[0.7, 2.1, 4.5, 6.1])
    w.bulk_period = 3.13  # one 0.78 + 2.35 A layer pair, continued below z_bottom
    want, _, rh = H.run_oracle(ref, w, threads=4, method=method)
    eta, _, st = H.run_device(w, method=method)
    assert (st["code"] == 0).all()
    assert np.array_equal(st["rhst"], rh)
    # R_bulk is defined to its stopping rule only (proposed.cpp:334-339); the
    # restatement's rows give the spread two correct builds show here
    H.assert_parity(eta, want, H.run_oracle(oracle, w, threads=4, method=method)[0])


# Bulk seeding on the batched path (state in HBM, the bulk periods stepped
# from the host with one sync per period): rk4 at N > 128 does not fit the
# cluster kernel, so auto takes this path; path 2 forces it elsewhere.
@pytest.mark.parametrize("method", ["rk4", "sp4", "sp6"])
def test_bulk_batched_layered_parity(ref, method):
    t0 = [2.0, 7.0, 15.0]
    of = ref.PotentialField.gaussian_layers(-10.0, F.LAYERED_LAYERS, 5.0)
    rc = oracle_curve(ref, of, F.rods11(ref), F.K_GAMMA11, t0, method, 0.05)
    field = mb.PotentialField.gaussian_layers(-10.0, F.LAYERED_LAYERS, bulk_period=5.0)
    c = mb.rocking_curve(field, dev_rods11(), F.K_GAMMA11, mb.AngleGrid.validated(t0, [0.0]),
                         mb.SweepOptions(method=method, dz=0.05, path=2))
    assert np.array_equal(c.status["rhst"], rc.rhst)
    assert H.curve_err(c.eta, rc.eta) <= TOL
    # R_bulk is defined only to its stopping rule (proposed.cpp:334-339), as in
    # test_bulk_layered_parity
    assert H.entry_rel_err(c.eta, rc.eta, floor=1e-6) <= 1e-8
    assert H.entry_rel_err(c.eta, rc.eta, floor=1e-10) <= 1e-7
    assert H.entry_abs_err(c.eta, rc.eta) <= 1e-11


# FSAL shares one product W between the last kick of a step and the first
# kick of the next but keeps both subtractions (and the end-of-step check
# between them) with the reference's rounding, and after an RHST applies the
# first kick against Q = I. So fsal = 1 must be BITWISE the unmerged
# schedule on every design: resident (N <= 64), thread-block clusters,
# cooperative groups and the batched path (which does not merge).
@pytest.mark.parametrize("case,path", [("cfg1", 1), ("n81", 3), ("n81", 4), ("n81", 2), ("cfg3", 4)])
def test_fsal_bitwise_equals_unmerged(case, path):
    if case == "cfg1":
        w = configs.config1().subset(theta0=[0.3, 1.1, 2.0, 5.5], slices=300)
    elif case == "n81":
        w = configs.config4(81, "sp6", n_structures=2).subset(theta0=[0.5, 2.5, 6.0], slices=200, z_bottom=-3.2)
    else:
        w = configs.config3().subset(theta0=[0.5, 3.5], slices=300, z_bottom=-3.0)
    a, ra, sa = H.run_device(w, fsal=False, path=path)
    b, rb, sb = H.run_device(w, fsal=True, path=path)
    assert (sa["code"] == 0).all() and (sb["code"] == 0).all()
    assert sa["rhst"].sum() > 0, "the case must exercise RHSTs between merged kicks"
    assert np.array_equal(sa["rhst"], sb["rhst"])
    assert np.array_equal(a, b) and np.array_equal(ra, rb)


def test_config3_full_depth_worst_angles(ref, oracle):
    """cfg3 at its full depth (10 A, 1000 slices of 0.01 A) on the two angles
    with the largest full-run deviation (1.1 and 1.7 deg), through the benched
    path (auto = cooperative CTA groups) with FSAL on, against the reference
    build. The slab amplifies rounding strongly: the restatement itself
    (oracle/, same algorithm, other summation order) lands ~1e-9 from the
    reference here, so the bound is 3x that measured floor (and >= 1e-9)."""
    w = configs.config3().subset(theta0=[1.1, 1.7])
    want, _, rh = H.run_oracle(ref, w, threads=2)
    alt, _, _ = H.run_oracle(oracle, w, threads=2)
    eta, _, st = H.run_device(w, fsal=True)
    assert (st["code"] == 0).all()
    assert np.array_equal(st["rhst"], rh)
    floor = H.curve_err(alt, want)
    H.assert_parity(eta, want, alt, tol=max(TOL, 3.0 * floor), abs_tol=1e-8)
