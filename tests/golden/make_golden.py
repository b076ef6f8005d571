"""Generates the committed golden fixtures from the REFERENCE ITSELF: the
reference's hot-path sources compiled verbatim against the Eigen-subset shim
(oracle/_ref/mb_ref*.so, `make -C oracle ref`; SURVEY.md §8c option A). The
reference ships no golden vectors of its own, and its atom
potential enters as a Tabulated field on the exact node heights (see
oracle/ref/mb_ref_py.cpp).

    python tests/golden/make_golden.py [case ...]

Each fixture stores the workload parameters (so it is self-describing), the
intensities eta[pairs][n], the reflection amplitudes rho, and the RHST counts.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import mb_ref  # noqa: E402

import harness as H  # noqa: E402
from paper_2306_00271_b200 import configs  # noqa: E402

def _bulk(n, method):
    """Bulk-seeded slab on the cluster kernel (64 < N <= 256):
    a thin slab over a 0.32 A bulk period continued below z_bottom. The
    absorption ratio is raised to 2.0 so R settles to 1e-12 within a few
    thousand bulk steps (at 0.1 the oracle needs ~10^4 periods per angle)."""
    w = configs.config4(n, method, n_structures=1).subset(theta0=[1.0, 4.0], slices=100, z_bottom=-1.6)
    w.bulk_period = 0.32
    w.absorption = 2.0
    return w


CASES = {
    "cfg0_full": lambda: configs.config0(),
    "cfg1_sub4": lambda: configs.config1().subset(theta0=[0.1, 1.0, 2.5, 6.1]),
    "cfg2_sub3x4": lambda: configs.config2(n_structures=3).subset(theta0=[0.5, 2.0, 4.4, 6.5]),
    "cfg4_n15_rk4": lambda: configs.config4(15, "rk4", n_structures=2).subset(theta0=[0.5, 3.3, 6.8], slices=100),
    "cfg4_n63_sp6": lambda: configs.config4(63, "sp6", n_structures=2).subset(theta0=[0.5, 3.3], slices=100),
    "cfg4_n127_sp6_thin": lambda: configs.config4(127, "sp6", n_structures=1).subset(theta0=[0.5, 4.1], slices=150,
                                                                                     z_bottom=-2.4),
    "bulk_n81_rk4": lambda: _bulk(81, "rk4"),
    "bulk_n67_sp6": lambda: _bulk(67, "sp6"),
    "bulk_n143_sp6": lambda: _bulk(143, "sp6"),
    # rk4 above 128 rods: the batched path's bulk seed (the cluster kernel's third slab plane does not fit)
    "bulk_n143_rk4": lambda: _bulk(143, "rk4"),
}


def make(name):
    w = CASES[name]()
    eta, rho, rh = H.run_oracle(mb_ref, w, threads=0)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), eta=eta, rho=rho, rhst=rh, n_rods=w.n_rods,
                        slices=w.slices, method=w.method, theta0=np.array(w.theta0), z_bottom=w.z_bottom,
                        structures=len(w.structures), generator="oracle/_ref (reference sources, verbatim)")
    print(name, eta.shape, "rhst", rh.tolist()[:6])


if __name__ == "__main__":
    for name in (sys.argv[1:] or CASES):
        make(name)
