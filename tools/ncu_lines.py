"""Per-CUDA-source-line instruction and stall totals from an .ncu-rep (needs -lineinfo)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg = defaultdict(lambda: [0, 0, ""])
cur = None
for x in rows:
    if x and x[0] == "Line No":
        hdr = x
        continue
    if hdr is None or len(x) < 8:
        continue
    if x[0]:
        cur = (x[0], x[1])
        continue
    try:
        ws = int(x[4] or 0)
        ie = int(x[7] or 0)
    except ValueError:
        continue
    a = agg[cur]
    a[0] += ie
    a[1] += ws
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"total warp-instr {tot_i}  samples {tot_s}")
for (ln, src), (ie, ws, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{ie:11d} {100*ie/max(tot_i,1):5.1f}%  st {ws:6d}  L{ln:>4} {src.strip()[:90]}")
