"""Compact per-kernel summary of an ncu raw CSV (ncu -i rep --page raw --csv):
duration, DRAM bytes, DRAM % of peak, tensor-pipe %, issue-slot %, warps active, registers.
    python tools/ncu_summary.py raw.csv out.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, u = rows[0], rows[1]
want = [("kernel", "Kernel Name"), ("us", "gpu__time_duration.sum"), ("dram_rd_MB", "dram__bytes_read.sum"),
        ("dram_wr_MB", "dram__bytes_write.sum"),
        ("dram_pct", "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("tensor_pct", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
        ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("regs", "launch__registers_per_thread")]
idx = [(n, h.index(m)) for n, m in want if m in h]
with open(sys.argv[2], "w", newline="") as f:
    w = csv.writer(f)
    w.writerow([n for n, _ in idx])
    w.writerow([u[i] for _, i in idx])
    for r in rows[2:]:
        if "at::" in r[h.index("Kernel Name")]:
            continue          # torch fills of the driver script
        w.writerow([r[i][:70] for _, i in idx])
