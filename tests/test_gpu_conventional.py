"""The conventional multi-slice method on the device (SURVEY §8f row 4,
conventional.cpp:9-78 with the Pade-13 exponential of kernels.cpp:25-58)
against the reference build's own solve_conventional (oracle/_ref), and the
reference acceptance criterion c04 (acceptance.cpp:164-178) run across the two
device methods: conventional vs sp6 agree to 1e-8 at h = 0.002 on the smooth
field."""
import math

import numpy as np
import pytest

import fields as F
import harness as H
import paper_2306_00271_b200 as mb
from paper_2306_00271_b200 import configs

pytestmark = pytest.mark.gpu


def dev_rods11():
    return mb.RodSet.build(mb.Lattice2D(*F.RECT), 5.0)


def ref_curve(ref, field, rods, gamma, t0, method, dz):
    o = ref.SweepOptions()
    o.method, o.dz, o.threads = method, dz, 0
    return ref.rocking_curve(field, rods, gamma, ref.AngleGrid.validated(t0, [0.0]), o)


@pytest.mark.parametrize("dz", [0.05, 0.02])
def test_conventional_layered_vs_reference(ref, dz):
    t0 = [2.0, 5.0, 9.0, 12.0, 17.0, 25.0]
    want = ref_curve(ref, F.layered_field(ref), F.rods11(ref), F.K_GAMMA11, t0, "conventional", dz)
    c = mb.rocking_curve(mb.PotentialField.gaussian_layers(-10.0, F.LAYERED_LAYERS), dev_rods11(), F.K_GAMMA11,
                         mb.AngleGrid.validated(t0, [0.0]), mb.SweepOptions(method="conventional", dz=dz))
    assert (c.status["code"] == 0).all()
    H.assert_parity(c.eta, want.eta)
    assert np.abs(c.rho - want.rho).max() <= 1e-10 * np.abs(want.rho).max()


def test_conventional_atoms_vs_reference(ref):
    """config-0 structure (N=13, atoms -> K1 table at the slice midpoints)."""
    w = configs.config0().subset(theta0=[0.5, 1.7, 3.3, 6.1], slices=200)
    want, _, _ = H.run_oracle(ref, w, threads=0, method="conventional")
    eta, _, st = H.run_device(w, method="conventional")
    assert (st["code"] == 0).all()
    H.assert_parity(eta, want)


def test_cross_method_c04():
    """acceptance.cpp:164-178 on the device: conventional and sp6 at h = 0.002."""
    field = mb.PotentialField.gaussian_layers(-10.0, F.SMOOTH_LAYERS)
    t0 = [5.0, 15.0, 30.0, 45.0, 60.0]
    grid = mb.AngleGrid.validated(t0, [0.0])
    a = mb.rocking_curve(field, dev_rods11(), F.K_GAMMA11, grid, mb.SweepOptions(method="conventional", dz=0.002))
    b = mb.rocking_curve(field, dev_rods11(), F.K_GAMMA11, grid, mb.SweepOptions(method="sp6", dz=0.002))
    worst = max(np.linalg.norm(a.rho[i] - b.rho[i]) / np.linalg.norm(b.rho[i]) for i in range(len(t0)))
    assert worst <= 1e-8, worst


def test_conventional_breakdown_and_limits():
    # vacuum: nothing reflects (acceptance.cpp:69-94)
    c = mb.rocking_curve(mb.PotentialField.zero(-1.0), mb.RodSet.build(mb.Lattice2D(*F.RECT), 0.5), 1.0,
                         mb.AngleGrid.validated([10.0, 40.0], [0.0]), mb.SweepOptions(method="conventional", dz=0.01))
    assert np.abs(c.rho).max() <= 1e-12
    # N > 32 and bulk seeding are outside the device conventional path
    w = configs.config4(63, "rk4", n_structures=1).subset(theta0=[1.0], slices=10, z_bottom=-0.16)
    with pytest.raises(mb.ConfigError):
        H.run_device(w, method="conventional")
