"""One plan execute of a workload (for ncu launch lists / full captures).
Usage: python tools/profile_case.py --config 1 [--reps 1]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2306_00271_b200 as mb  # noqa: E402
from paper_2306_00271_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--n-rods", type=int, default=63)
ap.add_argument("--method", default=None)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--structures", type=int, default=0)
ap.add_argument("--no-residual", action="store_true")
ap.add_argument("--angles", type=int, default=0)
ap.add_argument("--slices", type=int, default=0)
ap.add_argument("--path", type=int, default=0)
ap.add_argument("--z-bottom", type=float, default=0.0)
ap.add_argument("--threshold", type=float, default=1000.0)
a = ap.parse_args()
w = {0: configs.config0, 1: configs.config1, 3: configs.config3}.get(a.config, None)
if w is not None:
    w = w()
elif a.config == 2:
    w = configs.config2(a.structures or 1024)
else:
    w = configs.config4(a.n_rods, a.method or "rk4", n_structures=a.structures or 64)
if a.angles or a.slices or a.z_bottom:
    w = w.subset(theta0=list(w.theta0[:a.angles]) if a.angles else None, slices=a.slices or None,
                 z_bottom=a.z_bottom or None)
method = a.method or w.method
rods = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), w.n_rods)
opts = mb.SweepOptions(method=method, slices=w.slices, fsal=True, residual_check=not a.no_residual, path=a.path,
                       rhst_threshold=a.threshold)
pairs = [(s, t0, t1) for s in range(len(w.structures)) for t1 in w.theta1 for t0 in w.theta0]
plan = mb.Plan(rods, configs.product_fields(w), w.gamma, pairs, opts)
for _ in range(a.reps):
    plan.execute()
eta, rho, st = plan.results(raise_on_error=False)
print(w.name, plan.timing(), plan.info(), "rhst/pt", float(st["rhst"].mean()), "pivoting/pt", float(st["rhst_pivoting"].mean()))
prof = plan.profile()
if sum(prof.values()) > 0:
    tot = sum(list(prof.values())[:8])
    print("phase cycles per CTA:", {k: f"{v:.3e} ({100 * v / tot:.1f}%)" for k, v in prof.items()})
