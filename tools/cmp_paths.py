"""A/B of the large-N paths on cfg4 batches (tools only)."""
import sys
sys.path.insert(0, ".")
import paper_2306_00271_b200 as mb
from paper_2306_00271_b200 import configs
for n in [int(x) for x in sys.argv[1].split(",")]:
    for meth in sys.argv[2].split(","):
        w = configs.config4(n, meth)
        rods = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), w.n_rods)
        pairs = [(s, t0, t1) for s in range(len(w.structures)) for t1 in w.theta1 for t0 in w.theta0]
        for path in [int(x) for x in sys.argv[3].split(",")]:
            try:
                plan = mb.Plan(rods, configs.product_fields(w), w.gamma, pairs,
                               mb.SweepOptions(method=meth, slices=w.slices, fsal=True, path=path))
            except mb.Error as e:
                print(n, meth, "path", path, "n/a", e)
                continue
            plan.execute()
            t = plan.timing()
            fl = len(pairs) * w.slices * {"rk4": 4, "sp6": 11}[meth] * 8 * n ** 3
            print(n, meth, "path", path, round(t["ms_propagate"], 1), "ms", round(fl / t["ms_propagate"] / 1e9, 2), "TF", flush=True)
            plan.close()
