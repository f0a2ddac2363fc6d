"""Summarise an ncu report: key metrics, instruction mix and the hottest SASS lines (with the
CUDA source line they map to).   python tools/ncu_hot.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
want = ("Duration", "Registers Per Thread", "Executed Ipc Active", "Issue Slots Busy", "DRAM Throughput",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "No Eligible", "Achieved Occupancy",
        "L2 Cache Throughput", "Compute (SM) Throughput")
for row in det[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
hi = next(i for i, r in enumerate(src) if "Source" in r and "Instructions Executed" in r)
h = src[hi]
iS, iW, iN = h.index("Source"), h.index("Warp Stall Sampling (Not-issued Samples)"), h.index("Instructions Executed")
op, stall, data = collections.Counter(), collections.Counter(), []
for row in src[hi + 1:]:
    try:
        w, n = int(row[iW] or 0), int(row[iN] or 0)
    except (ValueError, IndexError):
        continue
    m = row[iS].split()
    mn = (m[1] if m and m[0].startswith("@") and len(m) > 1 else (m[0] if m else "")).split(".")[0]
    op[mn] += n
    stall[mn] += w
    data.append((w, n, row[iS][:90]))
print("instructions", sum(op.values()))
for k, v in op.most_common(20):
    print(f"  {k:10s} {v:10d}  stall {stall[k]}")
print("--- top not-issued stall SASS")
for d in sorted(data, reverse=True)[:top]:
    print(d)
