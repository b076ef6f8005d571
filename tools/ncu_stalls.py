"""Summarise an ncu --page source --csv --print-source sass dump: stall
reasons overall and per code region (by SASS opcode class)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
data = []
for r in rows[2:]:  # first kernel block only
    if r and r[0] == "Kernel Name":
        break
    if len(r) >= len(hdr) - 1:
        data.append(r)
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def f(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError):
        return 0.0


tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
agg = collections.Counter()
for r in data:
    for k in reasons:
        agg[k] += f(r, k)
print("stall reasons (% of samples):")
for k, v in agg.most_common(12):
    print(f"  {k:28s} {100 * v / tot:6.2f}")
byop = collections.Counter()
for r in data:
    toks = r[ix["Source"]].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    byop[op.split(".")[0]] += f(r, "Warp Stall Sampling (All Samples)")
print("samples by opcode:")
for k, v in byop.most_common(15):
    print(f"  {k:12s} {100 * v / tot:6.2f}")
