"""Per-source-line stall reasons from an `ncu --page source --csv
--print-source cuda,sass` dump (first kernel): the top lines by samples with
their dominant stall reasons. Usage: python tools/ncu_reasons.py dump.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ix, fname, first, kern = None, "", None, 0
acc, src, tot = {}, {}, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        first = first or r[1]
        kern = 1 if r[1] == first else 2
        continue
    if r[0] == "Line No":
        ix = {h: i for i, h in reversed(list(enumerate(r)))}
        reasons = [h for h in r if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if ix is None or kern > 1 or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    try:
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    tot[key] = tot.get(key, 0) + s
    src[key] = r[ix["Source"]] if "Source" in ix else ""
    d = acc.setdefault(key, {})
    for h in reasons:
        try:
            d[h] = d.get(h, 0) + float(r[ix[h]] or 0)
        except ValueError:
            pass
T = sum(tot.values())
print(f"total samples {T:.0f}")
for key in sorted(tot, key=lambda k: -tot[k])[:top]:
    rs = sorted(acc[key].items(), key=lambda x: -x[1])[:3]
    rtxt = ", ".join(f"{h[6:]} {v / max(tot[key], 1):.0%}" for h, v in rs)
    print(f"{tot[key] / T:6.2%} {key[0][:10]}:{key[1]:<5} [{rtxt}] {src[key].strip()[:70]}")
