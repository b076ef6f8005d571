"""Full-size sweep of the five BASELINE configs: one plan execute per case,
device time from CUDA events (mb_plan_timing), algorithmic TFLOP/s
(L * s_eff * 8 N^3 per point), fraction of the measured
DMMA peak, and the nvidia-smi clock record of the timed executes (bench.py's
Clocks: median SM clock, max clock, throttle reasons). JSON line per case."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2306_00271_b200 as mb  # noqa: E402
from paper_2306_00271_b200 import configs  # noqa: E402
from bench import Clocks, fp64_peaks  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="0,1,2,3,4")
ap.add_argument("--n4", default="15,31,63,127,255")
ap.add_argument("--methods4", default="rk4,sp6")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--fsal", type=int, default=1)
a = ap.parse_args()
S_EFF = {"rk4": 4, "sp4": 6, "sp6": 11}
cases = []
for c in a.cases.split(","):
    c = int(c)
    if c == 4:
        for n in a.n4.split(","):
            for m in a.methods4.split(","):
                cases.append(configs.config4(int(n), m))
    else:
        cases.append(configs.CONFIGS[c]())
ctx = mb.Context(0)
for w in cases:
    rods = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), w.n_rods)
    opts = mb.SweepOptions(method=w.method, slices=w.slices, fsal=bool(a.fsal))
    pairs = [(s, t0, t1) for s in range(len(w.structures)) for t1 in w.theta1 for t0 in w.theta0]
    t0 = time.perf_counter()
    plan = mb.Plan(rods, configs.product_fields(w), w.gamma, pairs, opts, ctx)
    t_plan = time.perf_counter() - t0
    best = None
    plan.execute()  # warm-up (first-touch of the table, clocks up)
    ck = Clocks(0)
    ck.start()
    for _ in range(a.reps):
        plan.execute()
        t = plan.timing()
        best = t if best is None or t["ms_total"] < best["ms_total"] else best
    clocks = ck.stop()
    eta, rho, st = plan.results(raise_on_error=False)
    info = plan.info()
    plan.close()
    flops = len(pairs) * w.slices * S_EFF[w.method] * 8.0 * w.n_rods ** 3
    print(json.dumps({"case": w.name, "points": len(pairs), "n": w.n_rods, "method": w.method,
                      "ms_total": best["ms_total"], "ms_potential": best["ms_potential"],
                      "ms_propagate": best["ms_propagate"], "launches": best["launches"],
                      "points_per_s": len(pairs) / (best["ms_total"] * 1e-3),
                      "tflops_propagate": flops / (best["ms_propagate"] * 1e-3) / 1e12,
                      "frac_dmma_peak": flops / (best["ms_propagate"] * 1e-3) / 1e12 / fp64_peaks()[0],
                      "path": ("resident" if info["npad"] <= 64 else "on-chip (cluster / cooperative groups)"
                               if w.method != "rk4" or len(pairs) < 512 else "batched"),
                      "clocks": clocks,
                      "rhst_per_point": float(st["rhst"].mean()), "rhst_pivoting_per_point": float(st["rhst_pivoting"].mean()), "failed": int((st["code"] != 0).sum()),
                      "npad": info["npad"], "plan_s": t_plan}), flush=True)
