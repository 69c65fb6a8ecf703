"""Summarise an ncu --csv launch list: per-kernel count, total and mean device time."""
import csv
import sys
from collections import OrderedDict

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    for r in rows[h + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")[:48]
        t = float(r[vi].replace(",", ""))
        c, s = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, s + t)
    print(f)
    for name, (c, s) in agg.items():
        print(f"  {name:50s} n={c:3d} total={s/1e3:10.1f}us mean={s/c/1e3:9.1f}us")
