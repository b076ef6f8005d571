"""E-6 dz time-error study on B200 (driver.cpp:10-11,41-90,
PAPER.md Table 3): the B200 CLI's `bench` subcommand over the reference's
step-width presets for each method, error against a fine sp6 reference curve
(and, where the device runs it, against the conventional baseline at
dz = 0.01, the paper's "orig" setting). Per method it then reports the
fastest cell whose error is below a target, the paper's speed-at-equal-
accuracy comparison.

  python tools/dz_study.py [--cases cfg0,cfg1,cfg3] [--outdir gpurun_out/dz]
"""
import argparse
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from paper_2306_00271_b200 import configs  # noqa: E402
from test_gpu_cli import workload_json  # noqa: E402

CLI = os.path.join(ROOT, "paper_2306_00271_b200", "manybeam_b200")


def case(name):
    if name == "cfg0":  # TRHEPD N=13: every method incl. the conventional one (N <= 32 on device)
        w = configs.config0()
        methods, ref_dz, base = ["conventional", "rk4", "sp4", "sp6"], 0.001, {"method": "conventional", "dz": 0.01}
    elif name == "cfg1":
        w = configs.config1()
        methods, ref_dz, base = ["rk4", "sp4", "sp6"], 0.001, None
    else:
        w = configs.config3().subset(theta0=list(configs.config3().theta0[::4]))
        methods, ref_dz, base = ["rk4", "sp4", "sp6"], 0.002, None
    cfg = workload_json(w, "sp6", extra={"fsal": True})
    del cfg["slices"]
    cfg["bench"] = {"reference": {"method": "sp6", "dz": ref_dz}, "methods": methods, "repeats": 3}
    if base:
        cfg["bench"]["baseline"] = base
    return w, cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="cfg0,cfg1,cfg3")
    ap.add_argument("--outdir", default=os.path.join(ROOT, "gpurun_out", "dz"))
    ap.add_argument("--target", type=float, default=1e-4)
    a = ap.parse_args()
    os.makedirs(a.outdir, exist_ok=True)
    summary = {}
    for name in a.cases.split(","):
        w, cfg = case(name)
        pj = os.path.join(a.outdir, f"{name}.json")
        pc = os.path.join(a.outdir, f"{name}_bench.csv")
        json.dump(cfg, open(pj, "w"))
        r = subprocess.run([CLI, "bench", "--config", pj, "--out", pc], capture_output=True, text=True)
        if r.returncode != 0:
            summary[name] = {"error": r.stderr.strip(), "rc": r.returncode}
            continue
        rows = [row for row in csv.reader(l for l in open(pc) if not l.startswith("#"))]
        hdr, rows = rows[0], rows[1:]
        recs = [dict(zip(hdr, r)) for r in rows]
        best = {}
        for rec in recs:
            if rec["status"] != "ok":
                continue
            err, t = float(rec["err_reference"]), float(rec["median_seconds"])
            if err <= a.target and (rec["method"] not in best or t < best[rec["method"]]["seconds"]):
                best[rec["method"]] = {"dz": float(rec["dz"]), "seconds": t, "err_reference": err,
                                       "points_per_s": w.points() / t}
        summary[name] = {"workload": w.name, "points": w.points(), "n_rods": w.n_rods,
                         "reference": cfg["bench"]["reference"], "target_err": a.target,
                         "fastest_below_target": best, "cells": recs,
                         "timing": "CLI bench: median of 3 wall-clock runs of mb_rocking_curve (host buffers)"}
        print(name, json.dumps(best), flush=True)
    json.dump(summary, open(os.path.join(a.outdir, "dz_study.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
