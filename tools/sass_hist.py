"""Opcode / stall histogram of an `ncu --page source --csv` SASS dump (tools/, profiling aid)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
c, s, lines = collections.Counter(), collections.Counter(), collections.Counter()
tot = stt = 0
for x in rows:
    if x and x[0] == "Address":
        hdr = x
        ie, src, st = x.index("Instructions Executed"), x.index("Source"), x.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(x) < len(hdr):
        continue
    toks = x[src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    n, m = int(x[ie] or 0), int(x[st] or 0)
    c[op] += n; s[op] += m; tot += n; stt += m
    lines[(x[0], x[src][:70])] += m
print("instructions", tot, "stall samples", stt)
for k, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{k:32s} {v:11d} {v / tot * 100:5.1f}%  stall {s[k] / max(stt, 1) * 100:5.1f}%")
print("--- hottest stall sites")
for (a, t), v in lines.most_common(20):
    print(f"{a} {v / max(stt, 1) * 100:5.1f}%  {t}")
