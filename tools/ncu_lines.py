"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass) per CUDA source
line: warp-stall samples, executed warp instructions and the top stall reasons.

    ncu -i REP --page source --csv --print-source cuda,sass -k regex:NAME > x.csv
    python tools/ncu_lines.py x.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fname = "?"
hdr = None
agg = collections.defaultdict(lambda: collections.Counter())
text = {}
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0].strip().isdigit():
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()
    if cur is None or not r[2].strip():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    c = agg[cur]
    for k in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
        v = d.get(k, "")
        if v.replace(".", "").isdigit():
            c[k] += float(v)
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k and v.replace(".", "").isdigit():
            c[k] += float(v)
tot = sum(c["Warp Stall Sampling (All Samples)"] for c in agg.values())
toti = sum(c["Instructions Executed"] for c in agg.values())
print(f"samples {tot:.0f}  warp instructions {toti:.0f}")
top = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:N]
for (f, ln), c in sorted(top, key=lambda kv: kv[0]):
    s = c["Warp Stall Sampling (All Samples)"]
    st = sorted(((v, k[6:]) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:3]
    print(f"{f}:{ln:<5d} {100 * s / tot:5.1f}% inst {c['Instructions Executed']:10.0f}  "
          f"{' '.join(f'{k}={v:.0f}' for v, k in st):40s} {text.get((f, ln), '')[:70]}")
