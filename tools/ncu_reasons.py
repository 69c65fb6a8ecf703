"""Stall-reason totals per CUDA-line range for a kernel in an .ncu-rep (needs -lineinfo).

    python tools/ncu_reasons.py REP KERNEL_REGEX lo:hi=name [lo:hi=name ...]
"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
ranges = [(tuple(map(int, r.split("=")[0].split(":"))), r.split("=")[1]) for r in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, line = None, -1
tot = {name: defaultdict(int) for _, name in ranges}
for x in rows:
    if x and x[0] == "Line No":
        hdr = x
        cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(x) < len(hdr):
        continue
    if x[0]:
        line = int(x[0]) if x[0].isdigit() else -1
        continue
    for (lo, hi), name in ranges:
        if lo <= line <= hi:
            for i in cols:
                try:
                    tot[name][hdr[i]] += int(x[i] or 0)
                except ValueError:
                    pass
for name, d in tot.items():
    s = sum(d.values())
    top = sorted(d.items(), key=lambda kv: -kv[1])[:8]
    print(name, s, "  ".join(f"{k[6:]}={v}" for k, v in top))
