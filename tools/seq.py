"""Per-kernel summary of an ncu --csv launch list (any name filter): last N launches."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
by = collections.OrderedDict()
for r in rows:
    d = by.setdefault(r[0], {"name": r[4].split("(")[0].replace("void ", "")})
    try:
        d[r[12]] = float(r[14].replace(",", ""))
    except ValueError:
        pass
for d in list(by.values())[-n:]:
    t = d.get("gpu__time_duration.sum", 0) / 1e3
    b = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{d['name'][:34]:34s} {t:8.1f} us {b:9.1f} MB")
