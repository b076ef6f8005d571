"""What plan creation and K1 produce, read back through the parity hooks
(mb_plan_node_heights / mb_plan_gamma / mb_plan_coefficients) and compared
with the reference build (oracle/_ref) and the restatement:
  * node heights (stages.cpp:25-47 slot order): bitwise vs the reference;
  * Gamma, 1/Gamma, Gamma^2, sin(theta0) per pair (geometry.cpp:19-57):
    bitwise vs the reference;
  * the K1 slice-potential table (atoms -> u(dg, z) per node slot, SURVEY
    §8a row P0): vs the restatement's BoundPotential::eval_coeffs at 1e-13 of
    the table's largest entry (the product sums the Gaussian terms in its own
    order on the device)."""
import numpy as np
import pytest

import paper_2306_00271_b200 as mb
from paper_2306_00271_b200 import configs

pytestmark = pytest.mark.gpu


def _plan(w, method=None, n_angles=4):
    rods = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), w.n_rods)
    opts = mb.SweepOptions(method=method or w.method, slices=w.slices, dz=-w.z_bottom / w.slices)
    pairs = [(s, t0, 0.0) for s in range(len(w.structures)) for t0 in list(w.theta0)[:n_angles]]
    return mb.Plan(rods, configs.product_fields(w), w.gamma, pairs, opts), pairs


@pytest.mark.parametrize("cfg,method", [(0, "rk4"), (1, "sp6"), (3, "sp6"), (0, "sp4")])
def test_node_heights_bitwise(ref, cfg, method):
    w = configs.CONFIGS[cfg]()
    plan, _ = _plan(w, method, 1)
    try:
        z = plan.node_heights()
    finally:
        plan.close()
    want = np.array(ref.node_heights(w.z_bottom, -w.z_bottom / w.slices, method))
    assert np.array_equal(z, want)


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_gamma_bitwise(ref, cfg):
    w = configs.CONFIGS[cfg]()
    plan, pairs = _plan(w, n_angles=len(w.theta0))
    rr = ref.RodSet.build_first(ref.Lattice2D(w.a1, w.a2), w.n_rods)
    try:
        for i, (_, t0, t1) in enumerate(pairs):
            gd, gi, g2, s0 = plan.gamma(i)
            d, inv, g2r, prop, s0r = ref.gamma_matrix(rr, w.gamma, t0, t1)
            assert np.array_equal(gd, np.array(d)) and np.array_equal(gi, np.array(inv))
            assert np.array_equal(g2, np.array(g2r)) and s0 == s0r
    finally:
        plan.close()


@pytest.mark.parametrize("cfg", [0, 1, 2, 3])
def test_k1_table_matches_restatement(oracle, cfg):
    w = configs.CONFIGS[cfg]() if cfg != 2 else configs.config2(n_structures=3)
    plan, _ = _plan(w, n_angles=1)
    try:
        plan.execute()
        z = plan.node_heights()
        rods = oracle.RodSet.build_first(oracle.Lattice2D(w.a1, w.a2), w.n_rods)
        ff_a, ff_b = configs.form_factors()
        for s, st in enumerate(w.structures):
            coef = plan.coefficients(s)
            f = oracle.PotentialField.atoms(w.z_bottom, st.xyz, st.species.astype(np.int32), st.B, ff_a, ff_b,
                                            w.cell_area, w.gamma_L, w.sign, w.absorption)
            u = oracle.BoundPotential(f, rods)
            idx = np.unique(np.linspace(0, len(z) - 1, 200).astype(int))
            want = np.array([u.eval_coeffs(z[i]) for i in idx])
            scale = np.abs(want).max()
            assert np.abs(coef[idx] - want).max() <= 1e-13 * scale
    finally:
        plan.close()
