"""Full-size parity of the device path against the reference build
(oracle/_ref: the reference's hot-path sources compiled verbatim) on the
BASELINE configs at their bench sizes. Runs on the GPU
box (device + the host's cores for the reference). One JSON record per case
into the output file (default profiles/parity_r02.json):

  curve_error                    curve.cpp:22-41 (max-row normalised)
  entry_rel_err_floor_1e-12/-10  per-entry relative error above that fraction of max eta
  entry_abs_err                  max |d eta| / max eta
  rhst_equal                     fraction of points with the reference's RHST count
  noise_floor_*                  the same metrics between the restatement and the
                                 reference (two correct CPU builds, same RHST
                                 schedule), where --noise covers the case

Usage: python tools/parity_full.py [--cases cfg0,cfg1,cfg2,cfg3,cfg4] [--out F]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle", "_ref"),
                os.path.join(ROOT, "oracle", "_build")]

import harness as H  # noqa: E402
import mb_ref  # noqa: E402  (checker)
from paper_2306_00271_b200 import configs  # noqa: E402


def cases(which):
    out = []
    if "cfg0" in which:
        out.append(("cfg0 full", configs.config0(), True))
    if "cfg1" in which:
        out.append(("cfg1 full (121 angles, FSAL on as benched)", configs.config1(), False))
    if "cfg2" in which:
        out.append(("cfg2 128 structures x 61 angles", configs.config2().subset(structures=list(range(128))), False))
    if "cfg3" in which:
        out.append(("cfg3 full (10 A, 1000 slices, 61 angles)", configs.config3(), False))
    if "cfg4" in which:
        for n in (15, 31, 63, 127, 255):
            for m in ("rk4", "sp6"):
                w = configs.config4(n, m)
                # 64 pairs per N: 8 structures x 8 angles spread over the grid
                t0 = [w.theta0[i] for i in np.linspace(0, len(w.theta0) - 1, 8).round().astype(int)]
                out.append((f"cfg4 N={n} {m}, 64 pairs, 500 slices", w.subset(structures=list(range(0, 64, 8)),
                                                                          theta0=t0), n <= 63))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg0,cfg1,cfg2,cfg3,cfg4")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "parity_r02.json"))
    ap.add_argument("--noise", action="store_true", help="also run the restatement where marked cheap")
    a = ap.parse_args()
    recs = []
    for name, w, cheap in cases(a.cases.split(",")):
        t0 = time.time()
        eta, _, st = H.run_device(w, fsal=True)
        t_dev = time.time() - t0
        t0 = time.time()
        want, _, rh = H.run_oracle(mb_ref, w, threads=0)
        t_ref = time.time() - t0
        rec = {"case": name, "workload": w.name, "points": int(w.points()), "n_rods": w.n_rods, "method": w.method,
               "slices": w.slices, "device_ok": bool((st["code"] == 0).all()),
               "curve_error": H.curve_err(eta, want),
               "entry_rel_err_floor_1e-12": H.entry_rel_err(eta, want, 1e-12),
               "entry_rel_err_floor_1e-10": H.entry_rel_err(eta, want, 1e-10),
               "entry_abs_err": H.entry_abs_err(eta, want),
               "rhst_equal": float((st["rhst"] == rh).mean()), "rhst_per_point": float(np.mean(rh)),
               "seconds_device_call": t_dev, "seconds_reference": t_ref, "reference_threads": os.cpu_count(),
               "checker": "oracle/_ref (reference sources compiled verbatim)", "device_fsal": True}
        if a.noise and cheap:
            import mb_oracle
            alt, _, _ = H.run_oracle(mb_oracle, w, threads=0)
            rec["noise_floor_curve_error"] = H.curve_err(alt, want)
            rec["noise_floor_entry_rel_err_floor_1e-12"] = H.entry_rel_err(alt, want, 1e-12)
            rec["noise_floor_entry_rel_err_floor_1e-10"] = H.entry_rel_err(alt, want, 1e-10)
        recs.append(rec)
        print(json.dumps(rec), flush=True)
        json.dump(recs, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
