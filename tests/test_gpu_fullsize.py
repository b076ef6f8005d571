"""Full-size properties (BASELINE.json configs at their bench sizes, where the
oracle would take minutes to hours): flux bound of an absorbing crystal,
bitwise determinism, sharding invariance (a structure block solved alone gives
the same rows as inside the full batch: what makes multi-GPU output
independent of the GPU count), stepper-variant agreement (FSAL on/off,
resident vs batched path) and RHST-threshold invariance."""
import numpy as np
import pytest

import harness as H
import paper_2306_00271_b200 as mb
from paper_2306_00271_b200 import configs
from paper_2306_00271_b200.dist import shard_structures

pytestmark = pytest.mark.gpu


def flux(eta):
    """Sum of flux-normalised reflected intensities per point
    (intensity(): |rho_i|^2 sin0 g0 / g_i, sweep.cpp analogue); <= 1 when the
    optical potential absorbs (SPEC.md:40 imaginary part)."""
    return eta.sum(axis=1)


@pytest.fixture(scope="module")
def cfg1_run():
    w = configs.config1()
    e1, r1, s1 = H.run_device(w)
    return w, e1, r1, s1


def test_cfg1_full_flux_and_determinism(cfg1_run):
    w, e1, r1, s1 = cfg1_run
    assert (s1["code"] == 0).all()
    f = flux(e1)
    assert np.isfinite(f).all() and f.max() <= 1.0 + 1e-8 and f.min() > 0.0
    e2, r2, s2 = H.run_device(w)
    assert np.array_equal(e1, e2) and np.array_equal(r1, r2)


def test_cfg1_full_fsal_and_batched_path(cfg1_run):
    w, e1, _, s1 = cfg1_run
    ef, _, sf = H.run_device(w, fsal=True)
    assert np.array_equal(sf["rhst"], s1["rhst"])
    assert H.curve_err(ef, e1) <= 1e-9
    eb, _, sb = H.run_device(w, path=2)
    assert (sb["code"] == 0).all()
    assert H.curve_err(eb, e1) <= 1e-9
    assert H.entry_rel_err(eb, e1) <= 1e-9


def test_cfg2_full_flux_and_sharding_invariance():
    w = configs.config2()
    eta, _, st = H.run_device(w)
    assert (st["code"] == 0).all()
    f = flux(eta)
    assert np.isfinite(f).all() and f.max() <= 1.0 + 1e-8
    per = len(w.theta0) * len(w.theta1)
    for rank, world in ((0, 8), (5, 8), (3, 7)):
        lo, hi = shard_structures(len(w.structures), rank, world)
        part, _, _ = H.run_device(w.subset(structures=list(range(lo, hi))))
        assert np.array_equal(part, eta[lo * per:hi * per])


def test_cfg3_full_flux_and_threshold_invariance():
    w = configs.config3()
    eta, _, st = H.run_device(w)
    assert (st["code"] == 0).all()
    assert (st["rhst"] > 0).any()
    f = flux(eta)
    assert np.isfinite(f).all() and f.max() <= 1.0 + 1e-8
    # RHST is a reformulation, not an approximation: a different
    # trigger threshold changes where transforms happen, not the answer, to
    # the conditioning noise of the chain. Measured at full depth (B200,
    # round 1): 9.4e-9 curve error between thresholds 1000 and 1500 (a thin
    # subset gives 1.9e-11 on the oracle), so the bound is 3e-8: it is a
    # property of the mathematics, not of this device path.
    e2, _, s2 = H.run_device(w, threshold=1500.0)
    assert H.curve_err(e2, eta) <= 3e-8


@pytest.mark.parametrize("method", ["rk4", "sp6"])
def test_cfg4_n255_column(method):
    w = configs.config4(n_rods=255, method=method, n_structures=1, n_angles=64)
    eta, _, st = H.run_device(w)
    assert (st["code"] == 0).all()
    f = flux(eta)
    assert np.isfinite(f).all() and f.max() <= 1.0 + 1e-8
    head, _, _ = H.run_device(w.subset(theta0=list(w.theta0[:8])))
    assert np.array_equal(head, eta[:8])


def test_edge_cases():
    w = configs.config0()
    rods = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), w.n_rods)
    opts = mb.SweepOptions(method="sp6", slices=w.slices)
    with pytest.raises(ValueError):  # empty batch: MB_ERR_ARG
        mb.solve_batch(configs.product_fields(w), rods, w.gamma, [], opts)
    with pytest.raises(mb.ConfigError):  # AngleGrid::validated, sweep.cpp:18-33
        mb.AngleGrid.validated([], [0.0])
    big = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), 257)
    with pytest.raises(mb.ConfigError):
        mb.solve_batch(configs.product_fields(w), big, w.gamma, [(0, 1.0, 0.0)], opts)
    with pytest.raises(ValueError):  # structure index out of range
        mb.solve_batch(configs.product_fields(w), rods, w.gamma, [(1, 1.0, 0.0)], opts)
    # a single pair at the largest supported rod count runs (batched path)
    top = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), 256)
    eta, _, st = mb.solve_batch(configs.product_fields(w), top, w.gamma, [(0, 1.0, 0.0)],
                                mb.SweepOptions(method="sp6", slices=20))
    assert eta.shape == (1, 256) and (st["code"] == 0).all() and np.isfinite(eta).all()


# ---------------------------------------------------------------- multi-device context
@pytest.mark.parametrize("cfg", ["cfg0", "cfg2", "cfg4n127"])
def test_multi_device_context_bitwise(cfg):
    """One context over several device shards (here two or three shards on
    the one GPU of the box, each with its own stream) gives bitwise the rows
    of the single-device context, in pair order (test_sweep.cpp:55-68: any
    thread count gives identical intensities)."""
    if cfg == "cfg0":
        w, path = configs.config0(), 0
    elif cfg == "cfg2":
        w, path = configs.config2(n_structures=24).subset(theta0=[0.5, 1.7, 3.9, 6.5], slices=200, z_bottom=-4.0), 0
    else:
        w, path = configs.config4(127, "sp6", n_structures=3).subset(theta0=[0.5, 2.5, 6.0], slices=60,
                                                                    z_bottom=-0.96), 3
    rods = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), w.n_rods)
    opts = mb.SweepOptions(method=w.method, slices=w.slices, fsal=True, path=path)
    pairs = [(s, t0, t1) for s in range(len(w.structures)) for t1 in w.theta1 for t0 in w.theta0]
    fields = configs.product_fields(w)
    one = mb.solve_batch(fields, rods, w.gamma, pairs, opts, mb.Context(0))
    for devs in ([0, 0], [0, 0, 0]):
        ctx = mb.Context(devices=devs)
        many = mb.solve_batch(fields, rods, w.gamma, pairs, opts, ctx)
        assert np.array_equal(one[0], many[0]) and np.array_equal(one[1], many[1])
        assert np.array_equal(one[2]["rhst"], many[2]["rhst"])
        ctx.close()
    if len(w.structures) == 1:  # rocking_curve over a multi-device context: angles round-robin
        grid = mb.AngleGrid.validated(w.theta0, w.theta1)
        a = mb.rocking_curve(fields[0], rods, w.gamma, grid, opts, mb.Context(0))
        b = mb.rocking_curve(fields[0], rods, w.gamma, grid, opts, mb.Context(devices=[0, 0]))
        assert np.array_equal(a.eta, b.eta)
