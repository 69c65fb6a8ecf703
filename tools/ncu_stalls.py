"""Per-CUDA-line stall samples (top N) and role totals for a kernel in an .ncu-rep.

    python tools/ncu_stalls.py REP KERNEL_REGEX [N] [lo:hi=name ...]
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
ranges = [a for a in sys.argv[4:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, cur = None, None
agg = defaultdict(lambda: [0, 0])
for x in rows:
    if x and x[0] == "Line No":
        hdr = x
        continue
    if hdr is None or len(x) < 8:
        continue
    if x[0]:
        cur = (int(x[0]) if x[0].isdigit() else -1, x[1])
        continue
    try:
        ws, ie = int(x[4] or 0), int(x[7] or 0)
    except ValueError:
        continue
    agg[cur][0] += ie
    agg[cur][1] += ws
print("samples", sum(v[1] for v in agg.values()), "warp-instr", sum(v[0] for v in agg.values()))
for r in ranges:
    span, name = r.split("=")
    lo, hi = map(int, span.split(":"))
    s = sum(v[1] for k, v in agg.items() if lo <= k[0] <= hi)
    i = sum(v[0] for k, v in agg.items() if lo <= k[0] <= hi)
    print(f"  {name}: samples {s} warp-instr {i}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:n]:
    print(f"{v[1]:6d} {v[0]:10d} L{k[0]} {k[1].strip()[:100]}")
