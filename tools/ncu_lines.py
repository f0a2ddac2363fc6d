"""Per-CUDA-source-line totals of an ncu report (instructions executed, stall samples, branch
instructions):   python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
iW = h.index("Warp Stall Sampling (All Samples)")
iN = h.index("Instructions Executed")
agg = collections.defaultdict(lambda: [0, 0, 0, ""])
cur = None
for r in rows[hi + 1:]:
    if len(r) <= iN:
        continue
    if r[0]:
        cur = (int(r[0]), r[1][:80]) if r[0].isdigit() else None
        continue
    if cur is None:
        continue
    try:
        w, n = int(r[iW] or 0), int(r[iN] or 0)
    except ValueError:
        continue
    a = agg[cur]
    a[0] += n
    a[1] += w
    if any(x in r[3] for x in ("BRA", "BSSY", "BSYNC")):
        a[2] += n
tot = sum(v[0] for v in agg.values())
print("total instructions", tot)
for (ln, src), (n, w, br, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"L{ln:4d} instr {n:9d} ({100 * n / tot:4.1f}%) stall {w:5d} branch {br:8d}  {src}")
