"""Generates the committed golden fixtures from the oracle (CPU restatement of
the reference hot path; the reference ships no golden vectors
and cannot be built here, so the oracle, pinned by the reference's own
known-answer tests in tests/test_oracle_*.py, is the reference of record).

    python tests/golden/make_golden.py

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
sys.path.insert(0, os.path.join(ROOT, "oracle", "_build"))

import mb_oracle  # noqa: E402

import harness as H  # noqa: E402
from paper_2306_00271_b200 import configs  # noqa: E402

CASES = {
    "cfg0_full": lambda: configs.config0(),
    "cfg1_sub4": lambda: configs.config1().subset(theta0=[0.1, 1.0, 2.5, 6.1]),
    "cfg2_sub3x4": lambda: configs.config2(n_structures=3).subset(theta0=[0.5, 2.0, 4.4, 6.5]),
    "cfg4_n15_rk4": lambda: configs.config4(15, "rk4", n_structures=2).subset(theta0=[0.5, 3.3, 6.8], slices=100),
    "cfg4_n63_sp6": lambda: configs.config4(63, "sp6", n_structures=2).subset(theta0=[0.5, 3.3], slices=100),
    "cfg4_n127_sp6_thin": lambda: configs.config4(127, "sp6", n_structures=1).subset(theta0=[0.5, 4.1], slices=150,
                                                                                     z_bottom=-2.4),
}


def make(name):
    w = CASES[name]()
    eta, rho, rh = H.run_oracle(mb_oracle, w, threads=0)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), eta=eta, rho=rho, rhst=rh, n_rods=w.n_rods,
                        slices=w.slices, method=w.method, theta0=np.array(w.theta0), z_bottom=w.z_bottom,
                        structures=len(w.structures))
    print(name, eta.shape, "rhst", rh.tolist()[:6])


if __name__ == "__main__":
    for name in (sys.argv[1:] or CASES):
        make(name)
