"""Top SASS lines by warp-stall samples for the first kernel matching a regex in an .ncu-rep."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for x in r:
    if x and x[0] == "Kernel Name":
        cur = []
        blocks.append(cur)
    elif cur is not None:
        cur.append(x)
rows = blocks[0]
h = rows[0]
si, ws, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
rows = rows[1:]
tot_s = sum(int(x[ws] or 0) for x in rows)
tot_i = sum(int(x[ie] or 0) for x in rows)
print("samples", tot_s, "warp-instr", tot_i, "sass lines", len(rows))
for x in sorted(rows, key=lambda x: -int(x[ws] or 0))[:n]:
    print("%6s %10s  %s" % (x[ws], x[ie], x[si][:100]))
