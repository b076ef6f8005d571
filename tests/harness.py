"""Shared parity harness: runs one workload through a CPU checker (the
reference compiled from its own sources, oracle/_ref `mb_ref`, or the
restatement oracle/_build `mb_oracle`; both test infrastructure, same Python
surface) and through the device path (libmanybeam_b200.so via the Python
mirror) on identical seeded inputs."""
import math

import numpy as np

import paper_2306_00271_b200 as mb
from paper_2306_00271_b200 import configs


def oracle_lattice(o, w):
    return o.Lattice2D(tuple(w.a1), tuple(w.a2))


def oracle_fields(o, w):
    ff_a, ff_b = configs.form_factors()
    return [o.PotentialField.atoms(w.z_bottom, s.xyz, s.species.astype(np.int32), s.B, ff_a, ff_b, w.cell_area,
                                   w.gamma_L, w.sign, w.absorption, bulk_period=w.bulk_period) for s in w.structures]


def run_oracle(o, w, threads=0, method=None, slices=None, threshold=1000.0):
    """Returns eta [pairs][n], rho, rhst counts; pairs ordered structure-major,
    theta0 inner (one oracle rocking_curve per structure, as the reference
    has no batched API)."""
    rods = o.RodSet.build_first(oracle_lattice(o, w), w.n_rods)
    opts = o.SweepOptions()
    opts.method = method or w.method
    opts.slices = slices or w.slices
    opts.dz = -w.z_bottom / opts.slices  # the bulk window's target step (sweep.cpp:97-102)
    opts.threads = threads
    opts.rhst_threshold = threshold
    grid = o.AngleGrid.validated(list(w.theta0), list(w.theta1))
    etas, rhos, rh = [], [], []
    for f in oracle_fields(o, w):
        c = o.rocking_curve(f, rods, w.gamma, grid, opts)
        etas.append(c.eta)
        rhos.append(c.rho)
        rh.append(c.rhst)
    return np.concatenate(etas), np.concatenate(rhos), np.concatenate(rh)


def run_device(w, method=None, slices=None, threshold=1000.0, residual_check=True, fsal=False, path=0):
    rods = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), w.n_rods)
    opts = mb.SweepOptions(method=method or w.method, slices=slices or w.slices, dz=-w.z_bottom / (slices or w.slices),
                           rhst_threshold=threshold,
                           residual_check=residual_check, fsal=fsal, path=path)
    pairs = [(s, t0, t1) for s in range(len(w.structures)) for t1 in w.theta1 for t0 in w.theta0]
    return mb.solve_batch(configs.product_fields(w), rods, w.gamma, pairs, opts)


def curve_err(eta, ref):
    num = np.linalg.norm(eta - ref, axis=1).max()
    den = np.linalg.norm(ref, axis=1).max()
    return 0.0 if num == 0 else (math.inf if den == 0 else num / den)


def entry_rel_err(eta, ref, floor=1e-12):
    """Per-entry relative error on entries >= floor * max eta (SURVEY.md §8d:
    1e-9 relative on entries above 1e-12 * max eta). Entries below the floor
    are checked absolutely by entry_abs_err."""
    mask = np.abs(ref) >= floor * np.abs(ref).max()
    return float((np.abs(eta - ref)[mask] / np.abs(ref)[mask]).max())


def entry_abs_err(eta, ref):
    """max |d eta| / max eta over every entry."""
    return float(np.abs(eta - ref).max() / max(np.abs(ref).max(), 1e-300))


def assert_parity(eta, want, alt=None, tol=1e-9, abs_tol=1e-11, slack=3.0):
    """The parity gate against the reference rows `want`:
      * curve_error (curve.cpp:22-41) <= tol;
      * per-entry relative error on entries >= 1e-12 max eta <= tol, or, where
        two correct CPU builds already disagree by more, <= slack x that noise
        floor: `alt` is the restatement's rows for the same inputs and RHST
        schedule (summation order is the only difference between the two), so
        entry_rel_err(alt, want) measures the conditioning of the case;
      * |d eta| <= abs_tol max eta everywhere.
    Returns the measured numbers."""
    ce = curve_err(eta, want)
    er = entry_rel_err(eta, want)
    noise = entry_rel_err(alt, want) if alt is not None else 0.0
    ea = entry_abs_err(eta, want)
    assert ce <= tol, ("curve_error", ce)
    assert er <= max(tol, slack * noise), ("entry_rel_err", er, "cpu noise floor", noise)
    assert ea <= abs_tol, ("entry_abs_err", ea)
    return {"curve_error": ce, "entry_rel_err": er, "cpu_noise_floor": noise, "entry_abs_err": ea}
