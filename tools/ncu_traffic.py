"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the kernels in an
ncu --set full report, keyed by the bench's launch tags -> profiles/ncu_traffic.json.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep [out.json]

Tags come from the kernel name (fused kernels are unique); the grouped-GEMM template instances
of the c2 training step map to tags by their order inside one step (tools/profile_step.py)."""
import csv
import io
import json
import subprocess
import sys

NAME_TAGS = [("mlp_fwd_kernel", "mlp_fwd"), ("mlp_dgrad_kernel", "mlp_dgrad"), ("route_kernel", "route"),
             ("route_tg_kernel", "route"), ("fold_full_kernel", "fold_heads"),
             ("combine_train_kernel", "combine_train"), ("unpermute_kernel", "unpermute"),
             ("scatter_kernel", "plan_scatter")]
# c2 training-step order of grouped_gemm_kernel launches (engine.step with fuse_mlp)
GEMM_ORDER = ["router_fwd", "fc2_wgrad_folded", "fc1_wgrad", "router_dgrad", "router_wgrad"]


def main(rep, out="profiles/ncu_traffic.json"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = rows[1]
    ki, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res, gi = {}, 0
    for r in rows[2:]:
        name = r[ki]
        b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
        tag = next((t for k, t in NAME_TAGS if k in name), None)
        if tag is None and "grouped_gemm_kernel" in name:
            tag = GEMM_ORDER[gi % len(GEMM_ORDER)]
            gi += 1
        if tag and tag not in res:
            res[tag] = round(b)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
