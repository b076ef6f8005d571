"""Per-CUDA-source-line warp-stall samples and shared-memory excess
wavefronts from an `ncu --page source --csv --print-source cuda,sass` dump
(first kernel block). Usage: python tools/ncu_lines.py dump.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lines = []
fname, ix, kernels, first = "", None, 0, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        first = first or r[1]
        kernels = 1 if r[1] == first else 2
        continue
    if r[0] == "Line No":
        ix = {}
        for i, h in enumerate(r):
            ix.setdefault(h, i)
        S = ix["Warp Stall Sampling (All Samples)"]
        X = ix.get("L1 Wavefronts Shared Excessive")
        W = ix.get("L1 Wavefronts Shared")
        continue
    if ix is None or r[0] == "" or kernels > 1:
        continue
    try:
        lines.append((int(r[0]), (fname[:10] + ":" + r[1])[:90], float(r[S] or 0), float(r[X] or 0) if X else 0,
                      float(r[W] or 0) if W else 0))
    except (ValueError, IndexError):
        pass
tot = sum(l[2] for l in lines) or 1
totx = sum(l[3] for l in lines) or 1
print(f"{first[:100]}\ntotal samples {tot:.0f}; smem excess wavefronts {totx:.3e}")
for ln, src, s, x, w in sorted(lines, key=lambda l: -l[2])[:top]:
    print(f"{ln:5d} {100 * s / tot:6.2f}% smemX {100 * x / totx:5.1f}%  {src}")
print("-- top smem excess")
for ln, src, s, x, w in sorted(lines, key=lambda l: -l[3])[:10]:
    print(f"{ln:5d} {100 * s / tot:6.2f}% smemX {100 * x / totx:5.1f}% wf {w:.2e} {src}")
