"""cfg3 (N=199, 10 A, 1000 slices, 61 angles) accuracy study: how far apart
two correct implementations of the reference algorithm land at full depth,
and where the device sits among them (the noise floor at
the SAME RHST schedule, and a 3M-vs-4M A/B of the complex GEMM).

  python tools/cfg3_accuracy.py run --role dev3m    --out gpurun_out/a_dev3m.npz
  MB_LIB=.../libmanybeam_b200_4m.so python tools/cfg3_accuracy.py run --role dev4m --out ...
  python tools/cfg3_accuracy.py run --role ref      --out ...   (oracle/_ref, threshold 1000)
  python tools/cfg3_accuracy.py run --role ref1500  --out ...   (oracle/_ref, threshold 1500)
  python tools/cfg3_accuracy.py run --role port     --out ...   (restatement, oracle/_build)
  python tools/cfg3_accuracy.py report a_*.npz  > profiles/cfg3_accuracy_r02.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle", "_ref"),
                os.path.join(ROOT, "oracle", "_build")]


def run(role, out, slices=None):
    import harness as H
    from paper_2306_00271_b200 import configs
    w = configs.config3()
    t0 = time.time()
    if role == "refdevU":
        # the reference propagating the DEVICE's K1 table (tabulated on the
        # exact node heights): separates U-input sensitivity from propagation
        import mb_ref
        import paper_2306_00271_b200 as mb
        rods = mb.RodSet.build_first(mb.Lattice2D(w.a1, w.a2), w.n_rods)
        plan = mb.Plan(rods, configs.product_fields(w), w.gamma, [(0, w.theta0[0], 0.0)],
                       mb.SweepOptions(method=w.method, slices=w.slices, dz=-w.z_bottom / w.slices))
        plan.execute()
        z, coef = plan.node_heights(), plan.coefficients(0)
        plan.close()
        order = np.argsort(z, kind="stable")
        zs, keep = np.unique(z[order], return_index=True)
        tab = coef[order][keep]
        dm = mb_ref.RodSet.build_first(mb_ref.Lattice2D(w.a1, w.a2), w.n_rods).diff_m
        f = mb_ref.PotentialField.tabulated(w.z_bottom, list(zs), [((int(a), int(b)), list(tab[:, d]))
                                                                  for d, (a, b) in enumerate(dm)])
        rr = mb_ref.RodSet.build_first(mb_ref.Lattice2D(w.a1, w.a2), w.n_rods)
        o = mb_ref.SweepOptions()
        o.method, o.slices, o.dz, o.threads = w.method, w.slices, -w.z_bottom / w.slices, 0
        c = mb_ref.rocking_curve(f, rr, w.gamma, mb_ref.AngleGrid.validated(list(w.theta0), [0.0]), o)
        eta, rho, rh = c.eta, c.rho, c.rhst
    elif role.startswith("dev"):
        # dev3m: auto path (cooperative groups at cfg3); devpath2 / devpath3:
        # the batched and the thread-block-cluster designs on the same inputs
        path = int(role[len("devpath"):]) if role.startswith("devpath") else 0
        eta, rho, st = H.run_device(w, fsal=role != "dev3m_nofsal", path=path)
        rh = st["rhst"]
    elif role.startswith("ref"):
        import mb_ref
        thr = 1500.0 if role == "ref1500" else 1000.0
        eta, rho, rh = H.run_oracle(mb_ref, w, threads=0, threshold=thr)
    else:
        # port: the restatement; portgj: the same with the study-only
        # Gauss-Jordan solve (MB_ORACLE_SOLVE=gj), the device's elimination form
        if role == "portgj":
            os.environ["MB_ORACLE_SOLVE"] = "gj"
        import mb_oracle
        eta, rho, rh = H.run_oracle(mb_oracle, w, threads=0)
    np.savez_compressed(out, eta=eta, rho=rho, rhst=np.asarray(rh), role=role, seconds=time.time() - t0)
    print(role, "done", time.time() - t0, flush=True)


def report(paths):
    import harness as H
    d = {str(np.load(p)["role"]): np.load(p) for p in paths}
    want = d["ref"]["eta"]
    out = {"workload": "cfg3-manybeam-N199-sp6 (full: 61 angles, 1000 slices)", "against": "ref (oracle/_ref, threshold 1000)",
           "rows": {}}
    if "refdevU" in d and "dev3m" in d:
        out["dev3m_vs_refdevU"] = {"curve_error": H.curve_err(d["dev3m"]["eta"], d["refdevU"]["eta"]),
                                   "entry_rel_err_floor_1e-10": H.entry_rel_err(d["dev3m"]["eta"], d["refdevU"]["eta"], 1e-10),
                                   "rhst_differs_at_angles": np.nonzero(d["dev3m"]["rhst"] != d["refdevU"]["rhst"])[0].tolist()}
    for k, v in d.items():
        if k == "ref":
            continue
        e = v["eta"]
        rows = np.linalg.norm(e - want, axis=1) / np.linalg.norm(want, axis=1).max()
        out["rows"][k] = {"curve_error": H.curve_err(e, want),
                          "entry_rel_err_floor_1e-12": H.entry_rel_err(e, want, 1e-12),
                          "entry_rel_err_floor_1e-10": H.entry_rel_err(e, want, 1e-10),
                          "entry_rel_err_floor_1e-6": H.entry_rel_err(e, want, 1e-6),
                          "rhst_differs_at_angles": np.nonzero(v["rhst"] != d["ref"]["rhst"])[0].tolist(),
                          "worst_angles": np.argsort(rows)[::-1][:5].tolist(),
                          "worst_angle_errors": np.sort(rows)[::-1][:5].tolist()}
    if "dev3m" in d and "dev4m" in d:
        out["dev3m_vs_dev4m_curve_error"] = H.curve_err(d["dev3m"]["eta"], d["dev4m"]["eta"])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        args = dict(zip(sys.argv[2::2], sys.argv[3::2]))
        run(args["--role"], args["--out"])
    else:
        report(sys.argv[2:])
