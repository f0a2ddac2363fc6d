"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list.
    python tools/launch_table.py launches.csv [N]                 last N launches
    python tools/launch_table.py launches.csv --step MARKER [k]   the k-th training step (default 5): the
                                                                  launches from the k-th kernel whose name
                                                                  contains MARKER up to the next one"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
launches = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi and r[vi]]
if len(sys.argv) > 2 and sys.argv[2] == "--step":
    marker = sys.argv[3]
    k = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    idx = [i for i, (n, _) in enumerate(launches) if marker in n]
    last = [x for x in launches[idx[k]:idx[k + 1]] if "FillFunctor<unsigned char>" not in x[0]]   # L2 flush
    print(f"# step {k} of the timed loop (launches between two '{marker}' kernels, L2 flush memset excluded)")
else:
    per = int(sys.argv[2]) if len(sys.argv) > 2 else len(launches)
    last = launches[-per:]
tot = sum(v for _, v in last)
for n, v in last:
    print(f"{v / 1000:9.1f} us  {100 * v / tot:5.1f}%  {n[:110]}")
print(f"total {tot / 1000:.1f} us over {len(last)} launches (serialised under ncu, cold caches)")
