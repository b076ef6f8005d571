"""Cluster (path 3) vs cooperative groups (path 4) on a small batch: max
relative difference and run-to-run determinism (tools only)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import harness as H
from paper_2306_00271_b200 import configs
for n, method in [(127, "sp6"), (127, "rk4"), (199, "sp6"), (255, "sp6")]:
    w = configs.config4(n, method, n_structures=2).subset(theta0=[0.5 + 0.45 * i for i in range(13)], slices=60,
                                                         z_bottom=-0.96)
    a, ra, sa = H.run_device(w, path=3)
    b, rb, sb = H.run_device(w, path=4)
    c, rc, sc = H.run_device(w, path=4)
    d, rd, sd = H.run_device(w, path=3)
    print(n, method, "cl-vs-coop curve_err", H.curve_err(b, a), "max|drho|", np.abs(ra - rb).max(),
          "coop det", np.array_equal(b, c), "cluster det", np.array_equal(a, d), "rhst eq", np.array_equal(sa["rhst"], sb["rhst"]),
          "rows differing", int((np.abs(a - b).max(axis=1) > 0).sum()), flush=True)
