"""Warp-stall reason totals of an ncu report (pc sampling):  python tools/ncu_stalls.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
tot = {}
for k, x in d.items():
    if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
        try:
            tot[k.split("stalled_")[1]] = float(x.replace(",", ""))
        except ValueError:
            pass
s = sum(tot.values())
for k, x in sorted(tot.items(), key=lambda kv: -kv[1]):
    if x > 0:
        print(f"{k:28s} {x:8.0f} {100 * x / s:5.1f}%")
