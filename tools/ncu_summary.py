"""Summarise an ncu --set full report: per kernel launch, duration, DRAM bytes, throughput."""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
units = rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size"]
idx = {w: h.index(w) for w in want if w in h}
recs = []
for r in rows[2:]:
    rec = {w: r[i] for w, i in idx.items()}
    rec["units"] = {w: units[i] for w, i in idx.items()}
    recs.append(rec)
print("| kernel | time | DRAM read | DRAM write | DRAM % peak | SM % | warps active % | regs | grid x block |")
print("|---|---|---|---|---|---|---|---|---|")
for rec in recs:
    u = rec["units"]
    name = rec["Kernel Name"].split("(")[0].replace("void ", "")
    print(f"| {name} | {rec.get('gpu__time_duration.sum')} {u.get('gpu__time_duration.sum')} | "
          f"{rec.get('dram__bytes_read.sum')} {u.get('dram__bytes_read.sum')} | {rec.get('dram__bytes_write.sum')} {u.get('dram__bytes_write.sum')} | "
          f"{rec.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | {rec.get('sm__throughput.avg.pct_of_peak_sustained_elapsed')} | "
          f"{rec.get('sm__warps_active.avg.pct_of_peak_sustained_active')} | {rec.get('launch__registers_per_thread')} | "
          f"{rec.get('launch__grid_size')} x {rec.get('launch__block_size')} |")
if len(sys.argv) > 2:
    json.dump(recs, open(sys.argv[2], "w"), indent=1)
