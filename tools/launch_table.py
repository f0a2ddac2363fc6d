"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: one line per launch
of the last complete step (kernel name, duration us), plus per-kernel totals."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
launches = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi and r[vi]]
per = int(sys.argv[2]) if len(sys.argv) > 2 else len(launches)
last = launches[-per:]
tot = sum(v for _, v in last)
for n, v in last:
    print(f"{v / 1000:9.1f} us  {100 * v / tot:5.1f}%  {n[:110]}")
print(f"total {tot / 1000:.1f} us over {len(last)} launches")
