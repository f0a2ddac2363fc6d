"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and duration of the
kernels of one step in an ncu --set full report, keyed by the bench's launch tags ->
profiles/ncu_traffic.json.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep gpurun_out/step_tags.json [out.json]

The ncu rows of the LAST step (the report's last N launches, N = len(tags)) are matched to the
tags tools/profile_step.py recorded in call order (the side stream serialised, so ncu's launch
order is the call order).  Tags launched more than once per step (e.g. a multi-kernel call) sum."""
import csv
import io
import json
import subprocess
import sys


def main(rep, tags_path, out="profiles/ncu_traffic.json"):
    tags = json.load(open(tags_path))["tags"]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki, rd, wr, du = (h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"),
                      h.index("gpu__time_duration.sum"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}
    data = rows[2:][-len(tags):]
    if len(data) != len(tags):
        raise SystemExit(f"report has {len(data)} launches, the step has {len(tags)}")
    res, dur, names = {}, {}, {}
    for tag, r in zip(tags, data):
        b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
        res[tag] = res.get(tag, 0) + round(b)
        dur[tag] = dur.get(tag, 0.0) + float(r[du]) * tscale.get(units[du], 1)
        names.setdefault(tag, []).append(r[ki][:90])
    json.dump(res, open(out, "w"), indent=1)
    json.dump({"dram_bytes": res, "duration_us": dur, "kernels": names},
              open(out.replace(".json", "_detail.json"), "w"), indent=1)
    for t in res:
        print(f"{t:22s} {dur[t]:8.1f} us  {res[t] / 1e6:9.2f} MB  {names[t][0][:60]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
