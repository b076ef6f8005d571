"""Summarise ncu reports into profiles/ncu_summary_<tag>.json: per kernel
duration, DRAM bytes, FP64 tensor (DMMA) pipe use, shared-memory traffic, and
(from a --metrics gpu__time_duration launch list) each kernel's share of the
step time."""
import csv
import io
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append((d, dict(zip(hdr, units))))
    return res


KEYS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dmma_pipe_active_pct_of_active_sm": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "sm_active_cycles": ("sm__cycles_active.avg", 1),
    "sm_elapsed_cycles": ("sm__cycles_elapsed.avg", 1),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    "smem_pct_peak": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1),
    "fp64_pipe_pct": ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1,
        "nsecond": 1e-6, "s": 1e3, "second": 1e3}


def summarize(rep):
    out = []
    for d, u in raw(rep):
        e = {"kernel": d.get("Kernel Name", "")[:90], "grid": d.get("Grid Size"), "block": d.get("Block Size")}
        for k, (m, scale) in KEYS.items():
            if m not in d or d[m] in ("", "n/a"):
                continue
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:
                continue
            unit = u.get(m, "")
            if k.endswith("bytes"):
                v *= UNIT.get(unit, 1)
            elif k == "duration_ms":
                v *= UNIT.get(unit, 1e-6)
            e[k] = v
        if "dram_read_bytes" in e:
            e["dram_bytes"] = e["dram_read_bytes"] + e.get("dram_write_bytes", 0.0)
        out.append(e)
    return out


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    tot, per = 0.0, {}
    for r in rows[1:]:
        name = r[ix["Kernel Name"]].split("(")[0]
        t = float(r[ix["Metric Value"]].replace(",", "")) * 1e-6  # ns -> ms
        per[name] = per.get(name, 0.0) + t
        tot += t
    return {"total_ms": tot, "kernels": {k: {"ms": v, "share": v / tot} for k, v in sorted(per.items(), key=lambda x: -x[1])}}


if __name__ == "__main__":
    tag, rep, launches = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None
    s = {"report": rep, "kernels": summarize(rep)}
    if launches:
        s["launch_list"] = launch_shares(launches)
    for k in s["kernels"]:
        if "propagate" in k["kernel"]:
            s["propagate"] = {"dram_bytes_per_launch": k.get("dram_bytes"), "duration_ms": k.get("duration_ms"),
                              "dmma_pipe_active_pct_of_active_sm": k.get("dmma_pipe_active_pct_of_active_sm")}
        if "potential_coef" in k["kernel"]:
            s["potential"] = {"dram_bytes_per_launch": k.get("dram_bytes"), "duration_ms": k.get("duration_ms")}
    json.dump(s, open(f"profiles/ncu_summary_{tag}.json", "w"), indent=1)
    print(json.dumps(s, indent=1)[:3000])
