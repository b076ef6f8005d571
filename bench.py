#!/usr/bin/env python
"""Benchmark of the B200-native forward model (driver contract).

Headline workload: BASELINE.json configs[3], the largest single-GPU config
(hex 19.2 A cell, 40 atoms, N=199 beams, 10 keV positrons, 1000 slices of
0.01 A, sp6 = the reference's highest-order stepper, 61 glancing angles), on
seeded synthetic atoms (no dataset exists; configs.py). BASELINE.json's
metric names no config, so the N=1 line is the largest single-GPU one. A
"step" is one full pass over the workload: K1 (slice-potential coefficients)
+ K2 (propagation + RHST + surface solve + intensities) for all points.

  value     points/s, inputs resident in HBM (plan created once; CUDA events
            on the launching stream around K1+K2; L2 flushed between steps by
            a 512 MiB write); under torchrun the max step time over ranks
  e2e       the same metric through the reference-facing C-ABI call with HOST
            buffers (mb_rocking_curve; solve_batch for batches): plan build,
            H2D, kernels, D2H inside the timed region
  roofline  dominant kernel (propagation, FP64 DMMA-bound): algorithmic flops
            L * s_eff * 8 N^3 per point / its CUDA-event time,
            against the measured DMMA peak (profiles/fp64_peak_r01.json;
            MEASURED_PEAKS.json has no FP64 entry)
  legs      configs[1] (N=61 sp6) and configs[2] (1024 structures, N=31 rk4,
            62,464 points) timed the same way, each with its own roofline and
            clock record
  cpu_baseline / parity
            the REFERENCE itself (oracle/_ref: its hot-path sources compiled
            verbatim, OpenBLAS GEMM, its own std::thread row pool) on a
            bounded sample of the headline workload on this host's cores, and
            the device rows of the same sample compared with it

Multi-GPU: one process per GPU (torchrun, or `--gpus N` which launches it);
batches are sharded in contiguous structure blocks, single-structure configs
round-robin by angle; no collective on the data path.
`--impl reference` times the reference's own rocking_curve (oracle/_ref) on
rank 0 only, on the bounded sample it can finish.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rocking-curve points/sec (structure x angle, fp64)"
UNIT = "points/s"
HEADLINE = 3
LEGS = (1, 2)
# committed ncu --set full summaries of the propagation kernel per workload
NCU = {3: "ncu_summary_r02ag_cfg3.json", 1: "ncu_summary_r01ab.json", 2: "ncu_summary_r01i_cfg2.json"}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def workload(cfg, args=None):
    from paper_2306_00271_b200 import configs
    if cfg == 4:
        return configs.config4(args.n_rods, args.method or "rk4")
    return configs.CONFIGS[cfg]()


def s_eff(method):
    return {"rk4": 4, "sp4": 6, "sp6": 11}[method]


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc = device, None
        self.path = f"/tmp/mb_clocks_{os.getpid()}_{str(device).replace(',', '_')}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7:
                try:
                    rows.append((float(f[0]), float(f[1]), f[3:7]))
                except ValueError:
                    pass
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def fp64_peaks():
    p = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
    try:
        d = json.load(open(p))
        return float(d["fp64_dmma_tflops"]), float(d["fp64_dfma_tflops"]), \
            "profiles/fp64_peak_r01.json (own DMMA/DFMA microbenchmark; MEASURED_PEAKS.json has no FP64 entry)"
    except Exception:
        return 37.1, 34.1, "fallback 37.1 / 34.1 TF/s (own DMMA/DFMA measurement, round 1)"


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), \
            "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6551.0, "fallback: MEASURED_PEAKS.json value of round 2 (6551 GB/s)"


def ncu_traffic(cfg):
    """dram__bytes_read + dram__bytes_write of the propagation kernel per
    launch, from the committed ncu --set full summary of this workload."""
    name = NCU.get(cfg)
    if not name:
        return None, None
    try:
        s = json.load(open(os.path.join(ROOT, "profiles", name)))
    except Exception:
        return None, None
    for k in s.get("kernels", []):
        if any(x in k.get("kernel", "") for x in ("propagate_kernel", "cluster_kernel", "big_stage")):
            return k.get("dram_bytes"), f"profiles/{name}"
    p = s.get("propagate") or {}
    return p.get("dram_bytes_per_launch"), f"profiles/{name}"


def shard(w, rank, world):
    """The rank's part of workload w and the global rows it owns:
    contiguous structure blocks for batches, angles round-robin for a single
    structure. Rows are structure-major, theta1, then theta0 (sweep.cpp:90-91)."""
    per = len(w.theta0) * len(w.theta1)
    if world == 1:
        return w, np.arange(w.points())
    if len(w.structures) > 1:
        from paper_2306_00271_b200.dist import shard_structures
        lo, hi = shard_structures(len(w.structures), rank, world)
        return w.subset(structures=list(range(lo, hi))), np.arange(lo * per, hi * per)
    if len(w.theta1) != 1:
        raise SystemExit("angle sharding expects one theta1")
    idx = np.arange(rank, len(w.theta0), world)
    return w.subset(theta0=[w.theta0[i] for i in idx]), idx


def run_leg(mb, configs, torch, cfg, w, args, ctx, rank, world, dist, local_rank, flush):
    """Times one workload (whole job over all ranks). Returns the leg record
    and this rank's (rows, eta)."""
    total_points = w.points()
    wl, rows = shard(w, rank, world)
    method = wl.method
    rods = mb.RodSet.build_first(mb.Lattice2D(wl.a1, wl.a2), wl.n_rods)
    opts = mb.SweepOptions(method=method, slices=wl.slices, fsal=not args.no_fsal)
    fields = configs.product_fields(wl)
    pairs = [(s, t0, t1) for s in range(len(wl.structures)) for t1 in wl.theta1 for t0 in wl.theta0]
    plan = mb.Plan(rods, fields, wl.gamma, pairs, opts, ctx) if pairs else None
    info = plan.info() if plan else {"coef_bytes": 0, "npad": 0, "h2d_bytes": 0, "slots": 0, "ndiff": 0}

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        flush.zero_()
        torch.cuda.synchronize()
        if plan:
            plan.execute()
    barrier()
    clocks = Clocks(",".join(str(d) for d in ctx.devices))
    clocks.start()
    tot = pot = prop = 0.0
    launches = 0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if plan:
            plan.execute()
            t = plan.timing()
            tot += t["ms_total"]
            pot += t["ms_potential"]
            prop += t["ms_propagate"]
            launches += t["launches"]
    barrier()
    ck = clocks.stop()
    if plan:
        eta, _, status = plan.results()
        plan.close()
    else:
        eta, status = np.zeros((0, w.n_rods)), None
    ms_step = tot / args.steps
    ms_prop = prop / args.steps
    if dist:
        tt = torch.tensor([ms_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_step = float(tt.tolist()[0])
    flops_launch = len(pairs) * wl.slices * s_eff(method) * 8.0 * wl.n_rods ** 3
    peak, dfma_peak, peak_src = fp64_peaks()
    achieved = flops_launch / (ms_prop * 1e-3) / 1e12 if ms_prop > 0 else 0.0
    traffic, traffic_src = ncu_traffic(cfg)
    path = ("resident propagate_kernel" if wl.n_rods <= 64 else
            "cluster_kernel (cooperative CTA groups)" if len(pairs) < 512 else "batched big_* kernels")
    leg = {
        "workload": w.name, "value": total_points / (ms_step * 1e-3), "unit": UNIT, "ms_per_step": ms_step,
        "points": total_points, "points_this_rank": len(pairs), "n_rods": w.n_rods, "method": method,
        "slices": w.slices, "fsal": opts.fsal,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": f"{path} (NP={info['npad']})", "peak_source": peak_src,
                     "flops_per_launch": flops_launch,
                     "flops_rule": f"points * L * {s_eff(method)} * 8 N^3 (N={wl.n_rods}; RHST/extraction excluded)",
                     "ms_per_launch": ms_prop, "rank": rank},
        "clocks": ck, "gpu_launches": launches,
        "kernel_ms": {"potential": pot / args.steps, "propagate": ms_prop},
        "rhst_per_point": float(status["rhst"].mean()) if status is not None and len(status) else None,
        "rhst_pivoting_per_point": float(status["rhst_pivoting"].mean()) if status is not None and len(status) else None,
        "coef_table_mib": info["coef_bytes"] / 2 ** 20,
    }
    # K1 (slice potential): HBM write of the coefficient table; each 16-B
    # output sums T = 4 x atoms complex x real terms = 2T DFMA = 4T flops
    if pot > 0:
        T = 4 * max(len(s.species) for s in wl.structures)
        gbs = info["coef_bytes"] / (pot / args.steps * 1e-3) / 1e9
        ceil = dfma_peak * 1e12 / (4.0 * T) * 16 / 1e9
        leg["potential_roofline"] = {
            "bound": "hbm", "kernel": "potential_coef_kernel (K1)", "achieved": gbs, "unit": "GB/s",
            "peak": hbm_peak()[0], "peak_source": hbm_peak()[1], "frac": gbs / hbm_peak()[0],
            "bytes_per_launch": info["coef_bytes"],
            "bytes_rule": "16 B x structures x node slots x ndiff (coefficient table write)",
            "compute_ceiling_gbs": ceil, "frac_of_compute_ceiling": gbs / ceil,
            "ceiling_rule": f"DFMA peak {dfma_peak} TF/s / (4 T flops per 16-B output), T = {T}"}
    return leg, (rows, eta, info, rods, fields, opts, wl, pairs)


def e2e_leg(mb, torch, w, state, args, ctx, dist):
    """The same metric through the public host-buffer API, per rank."""
    rows, eta, info, rods, fields, opts, wl, pairs = state
    if not pairs:
        te = [0.0] * args.steps
    elif len(wl.structures) == 1:
        grid = mb.AngleGrid.validated(wl.theta0, wl.theta1)
        for _ in range(max(1, args.warmup)):
            mb.rocking_curve(fields[0], rods, wl.gamma, grid, opts, ctx)
        te = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            c = mb.rocking_curve(fields[0], rods, wl.gamma, grid, opts, ctx)
            te.append(time.perf_counter() - t0)
        assert np.array_equal(c.eta, eta), "e2e path must reproduce the plan path bitwise"
    else:
        for _ in range(max(1, args.warmup)):
            mb.solve_batch(fields, rods, wl.gamma, pairs, opts, ctx)
        te = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            eb, _, _ = mb.solve_batch(fields, rods, wl.gamma, pairs, opts, ctx)
            te.append(time.perf_counter() - t0)
        assert np.array_equal(eb, eta), "e2e path must reproduce the plan path bitwise"
    tmean = statistics.mean(te)
    world = 1
    if dist:
        tt = torch.tensor([tmean], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tmean = float(tt.item())
        world = dist.get_world_size()
    call = "mb_rocking_curve (C-ABI, host buffers)" if len(w.structures) == 1 else \
        "solve_batch (Plan over the C-ABI, host buffers)"
    return {"value": w.points() / tmean, "unit": UNIT, "h2d_bytes_per_step": info["h2d_bytes"] * world,
            "d2h_bytes_per_step": w.points() * (w.n_rods * (8 + 16) + 16), "ms_per_step": 1000.0 * tmean,
            "call": call}


# ------------------------------------------------------------ CPU reference
def _ref_module():
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import mb_ref  # the reference build: baseline / checker only, never the measured GPU path
    return mb_ref


def ref_sample(w, cores):
    """Bounded sample of workload w: one point per host core (at most 16),
    angles spread evenly over the grid, structure 0."""
    nang = max(1, min(len(w.theta0), cores, 16))
    idx = np.unique(np.linspace(0, len(w.theta0) - 1, nang).round().astype(int))
    return w.subset(structures=[0], theta0=[w.theta0[i] for i in idx]), idx


def cpu_baseline(w, eta_dev=None):
    """The reference (oracle/_ref) on the bounded sample, timed by its own
    sweep timer (sweep.cpp:56,140-141) with threads = host cores; plus the
    device rows of the same points compared with it."""
    mb_ref = _ref_module()
    import harness as H
    cores = os.cpu_count() or 1
    sub, idx = ref_sample(w, cores)
    rods = mb_ref.RodSet.build_first(mb_ref.Lattice2D(sub.a1, sub.a2), sub.n_rods)
    opts = mb_ref.SweepOptions()
    opts.method, opts.slices, opts.dz, opts.threads = sub.method, sub.slices, -sub.z_bottom / sub.slices, 0
    f = H.oracle_fields(mb_ref, sub)[0]
    rows = mb_ref.rocking_curve(f, rods, sub.gamma, mb_ref.AngleGrid.validated(list(sub.theta0), list(sub.theta1)),
                                opts)
    secs = rows.solve_seconds
    cb = {"value": sub.points() / secs, "unit": UNIT, "cores": cores, "kind": "reference",
          "sample": f"{sub.points()} points of {w.name} (structure 0, angles {idx.tolist()}), full depth, "
                    f"{secs:.1f} s, reference sources compiled verbatim against the Eigen-subset shim "
                    f"(oracle/_ref, -O3 no -march, OpenBLAS GEMM single-threaded per row), "
                    f"its row pool with threads = {cores}"}
    parity = None
    if eta_dev is not None:
        dev = eta_dev[idx]
        want = rows.eta
        parity = {"points": int(len(idx)), "curve_error": H.curve_err(dev, want),
                  "entry_rel_err_floor_1e-12": H.entry_rel_err(dev, want, 1e-12),
                  "entry_rel_err_floor_1e-10": H.entry_rel_err(dev, want, 1e-10),
                  "entry_abs_err": H.entry_abs_err(dev, want),
                  "checker": "oracle/_ref (the reference build)"}
    return cb, parity, rows


def run_reference(args):
    """Reference arm: the reference's own rocking_curve (sweep.cpp:54-143,
    compiled verbatim, oracle/_ref) on the host cores, rank 0 only. Each step
    is one call over the bounded sample (one full-depth point per core);
    every number printed was measured, nothing is extrapolated."""
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    mb_ref = _ref_module()
    import harness as H
    w = workload(args.config, args)
    cores = os.cpu_count() or 1
    sub, idx = ref_sample(w, cores)
    rods = mb_ref.RodSet.build_first(mb_ref.Lattice2D(sub.a1, sub.a2), sub.n_rods)
    grid = mb_ref.AngleGrid.validated(list(sub.theta0), list(sub.theta1))

    def opts_for(ws):
        o = mb_ref.SweepOptions()
        o.method, o.slices, o.dz, o.threads = ws.method, ws.slices, -ws.z_bottom / ws.slices, 0
        return o

    # warm-up steps: the same grid through a 0.5 A slab at the workload's step
    # (1/20 of cfg3's depth): page-in, thread start-up, OpenBLAS init
    h = -w.z_bottom / w.slices
    warm = sub.subset(slices=max(1, int(round(0.5 / h))), z_bottom=-max(1, int(round(0.5 / h))) * h)
    fw = H.oracle_fields(mb_ref, warm)[0]
    for _ in range(args.warmup):
        mb_ref.reference_sweep(fw, rods, warm.gamma, grid, opts_for(warm))
    f = H.oracle_fields(mb_ref, sub)[0]
    secs = []
    for _ in range(args.steps):
        _, s = mb_ref.reference_sweep(f, rods, sub.gamma, grid, opts_for(sub))
        secs.append(s)
    ms = 1000.0 * statistics.mean(secs)
    v = sub.points() / (ms * 1e-3)
    sample = (f"{sub.points()} full-depth points of {w.name} (structure 0, angles {idx.tolist()}) per step; "
              f"warm-up steps on a {warm.slices}-slice slab")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "points_per_step": sub.points(), "n_rods": w.n_rods, "method": w.method,
                       "slices": w.slices, "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "timer": "the reference's own solve_seconds (sweep.cpp:56,140-141)"}
    print(json.dumps(line), flush=True)
    return 0


def relaunch(args):
    """--gpus N without a launcher: one process per GPU via torchrun."""
    import torch
    if torch.cuda.device_count() < args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but only {torch.cuda.device_count()} CUDA device(s) are visible")
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=HEADLINE)
    ap.add_argument("--legs", default=",".join(str(c) for c in LEGS), help="extra configs timed as legs ('' = none)")
    ap.add_argument("--n-rods", type=int, default=63)
    ap.add_argument("--method", default=None)
    ap.add_argument("--no-fsal", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--launcher", default="context", choices=["context", "torchrun"],
                    help="--gpus N without torchrun: one process over a multi-device context, or relaunch")
    args = ap.parse_args()
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        return run_reference(args)
    if world == 1 and args.gpus > 1 and args.launcher == "torchrun":
        return relaunch(args)
    if world != args.gpus and "WORLD_SIZE" in os.environ and args.gpus != 1:
        raise SystemExit(f"--gpus {args.gpus} disagrees with WORLD_SIZE={world}")
    # --gpus N in one process: the library's multi-device context
    # (mb_context_create_multi: one host thread per GPU, fixed pair map, rows
    # gathered in order); under torchrun each rank drives its own GPU
    ndev = args.gpus if world == 1 else 1

    import torch
    if torch.cuda.device_count() < max(ndev, local_rank + 1):
        raise SystemExit(f"rank {rank}: needs {max(ndev, local_rank + 1)} CUDA device(s), "
                         f"{torch.cuda.device_count()} visible (no CPU fallback)")
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_2306_00271_b200 as mb
    from paper_2306_00271_b200 import configs

    ctx = mb.Context(devices=list(range(ndev))) if ndev > 1 else mb.Context(local_rank)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2
    w = workload(args.config, args)
    if args.method:
        w.method = args.method
    t_wall = time.perf_counter()
    head, state = run_leg(mb, configs, torch, args.config, w, args, ctx, rank, world, dist, local_rank, flush)
    t_wall = time.perf_counter() - t_wall
    e2e = None if args.no_e2e else e2e_leg(mb, torch, w, state, args, ctx, dist)
    legs = {}
    for c in [int(x) for x in args.legs.split(",") if x.strip()]:
        if c == args.config:
            continue
        wc = workload(c, args)
        leg, _ = run_leg(mb, configs, torch, c, wc, args, ctx, rank, world, dist, local_rank, flush)
        legs[wc.name] = leg

    if rank == 0:
        cb, parity = None, None
        if not args.no_cpu_baseline and world == 1 and ndev == 1:
            rows, eta, *_ = state
            cb, parity, _ = cpu_baseline(w, eta)
        sharded = world > 1
        if ndev > 1:
            par = (f"one process, mb_context_create_multi over {ndev} GPUs (" +
                   ("angles round-robin" if len(w.structures) == 1 else "contiguous structure blocks") +
                   "), no collective")
        elif sharded:
            par = (("angles round-robin" if len(w.structures) == 1 else "contiguous structure blocks") +
                   f" over {world} rank(s), no collective")
        else:
            par = "1 GPU"
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world * ndev, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "points": w.points(), "n_rods": w.n_rods, "method": head["method"],
                       "slices": w.slices, "energy_ev": w.energy_ev, "particle": w.particle, "fsal": head["fsal"],
                       "rhst_threshold": 1000.0, "residual_check": True,
                       "l2": "flushed between steps (512 MiB write); coefficient table "
                             f"{head['coef_table_mib']:.1f} MiB",
                       "parallelism": par},
            "roofline": head["roofline"], "potential_roofline": head.get("potential_roofline"),
            "cpu_baseline": cb, "parity": parity, "e2e": e2e, "gpu_launches": head["gpu_launches"],
            "kernel_ms": head["kernel_ms"], "rhst_per_point": head["rhst_per_point"],
            "rhst_pivoting_per_point": head["rhst_pivoting_per_point"], "clocks": head["clocks"],
            "wall_s_headline_leg": t_wall, "legs": legs,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
