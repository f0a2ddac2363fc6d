"""Where the drop-in API step (bench.e2e_api: forward_sparse on a host batch + backward with host
labels) spends its time: host wall time per call, and the CUDA kernels/copies under torch.profiler.
    python tools/api_profile.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_09386_b200 as smes  # noqa: E402


def main():
    c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    dev = torch.device("cuda:0")
    params = bench._make_params(c, dev)
    T, E = c["T"], c["E"]
    pools = [smes.ExpertPool([smes.Affine(l.weight[e], l.bias[e]) for e in range(E)], l.act) for l in params.layers]
    routers = smes.RouterBank([smes.Affine(params.router_w[t], params.router_b[t]) for t in range(T)])
    heads = [smes.Affine(params.head_w[t:t + 1], params.head_b[t:t + 1]) for t in range(T)]
    model = smes.MoeModel(None, None, pools, routers, heads, torch.ones(T), c["beta"],
                          smes.RoutingBudget(c["ks"], c["ka"]))
    h_host, y_host = bench._host_inputs(c, c["B"], 0)
    x_host = h_host.float().pin_memory()
    for _ in range(3):
        res = smes.forward_sparse(x_host, model)
        smes.backward(res, model, y_host)
    torch.cuda.synchronize()
    for _ in range(3):
        t0 = time.perf_counter()
        res = smes.forward_sparse(x_host, model)
        t1 = time.perf_counter()
        bw = smes.backward(res, model, y_host)
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"host: forward_sparse {1e3 * (t1 - t0):.3f} ms  backward {1e3 * (t2 - t1):.3f} ms  "
              f"drain {1e3 * (t3 - t2):.3f} ms  total {1e3 * (t3 - t0):.3f} ms")
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        res = smes.forward_sparse(x_host, model)
        bw = smes.backward(res, model, y_host)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=60))
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25, max_name_column_width=60))
    print("loss", bw.total)


if __name__ == "__main__":
    main()
