#!/usr/bin/env python
"""Benchmark: SMES fwd+bwd samples/s on B200 (BASELINE.json configs[1], c2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one SMES-layer fwd+bwd over one batch of synthetic KuaiRand-shaped
input: routers -> progressive routing -> dedup plan/permute -> expert MLP
(256->512->256, grouped tcgen05 GEMMs) -> combine -> task heads -> BCE +
beta*L_lb, and the full backward (all parameter grads + d_hidden).
c2: T=8 tasks, E=32 experts, K_s=4 shared + K_a=2 private, d_model=256,
batch 16384 per GPU, bf16 storage / fp32 accumulate (Stage-I routing fp64).
Weights: reference init (model.py:117-156), seed 0.  Inputs: h ~ N(0,1).

N>1 (torchrun, one rank per GPU): weak scaling, 16384 samples per rank,
data-parallel with the LB-statistics all-reduce and the gradient all-reduce
(NCCL).  Timing: CUDA events per step, L2 flushed between steps, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(T=8, E=32, ks=4, ka=2, d=256, d_ff=512, d_out=256, B=16384, beta=0.01)
WORKLOAD = ("c2: SMES fwd+bwd, 8 tasks, 32 experts, shared top-4 + private top-2, d_model=256, "
            "expert MLP 256->512->256, batch 16384 per GPU, bf16")
METRIC = "SMES fwd+bwd samples/sec"
UNIT = "samples/s"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return FALLBACK_PEAKS, "fallback"


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------- CPU legs

def _cpu_sample(b_sample: int, steps: int, warm: int = 1):
    """Time the oracle port (the reference's algorithm restated in NumPy f64) on a
    bounded sub-batch of the c2 workload: forward_sparse + backward."""
    from oracle import smes_oracle as O
    rng = np.random.default_rng(0)
    c = CFG
    p = O.init_layer_params(rng, c["d"], c["d_out"], c["E"], c["T"], d_ff=c["d_ff"])
    h = rng.normal(size=(b_sample, c["d"]))
    y = (rng.uniform(size=(c["T"], b_sample)) < np.resize([0.3, 0.1, 0.05, 0.2], c["T"])[:, None]).astype(float)
    times = []
    for i in range(warm + steps):
        t0 = time.perf_counter()
        f = O.forward_sparse(h, p, c["ks"], c["ka"])
        O.backward(f, p, y, None, c["beta"])
        dt = time.perf_counter() - t0
        if i >= warm:
            times.append(dt)
    med = statistics.median(times)
    cores = len(os.sched_getaffinity(0))
    return {"value": b_sample / med, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"c2 shape at B={b_sample} (sub-batch of 16384), oracle/smes_oracle.py forward_sparse+backward, "
                      f"median of {steps} steps after {warm} warm-up, numpy f64 with {cores} host threads"}


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(len(os.sched_getaffinity(0))))
    b_sample = 2048
    steps = max(1, min(args.steps, 5))
    cb = _cpu_sample(b_sample, steps, warm=min(1, args.warmup))
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": min(1, args.warmup), "ms_per_step": 1e3 * b_sample / cb["value"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": CFG["B"] * args.gpus,
                       "parallelism": f"dp{args.gpus}", "reference_sample_batch": b_sample},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU leg

class ClockSampler:
    """Samples SM clock + throttle reasons via NVML while the timed region runs."""

    def __init__(self, index=0, period=0.01):
        self.samples, self.reasons, self.period = [], set(), period
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2602_09386_b200 import ExpertLayer, SMESEngine, SMESParams, _lib
    from paper_2602_09386_b200.dp import DataParallelStep

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    c = CFG
    # reference init (model.py:117-156): experts/heads U(+-1/sqrt(fan_in)), routers U(+-1e-3/sqrt(d)), bias 0
    g = torch.Generator(device="cpu").manual_seed(0)
    u = lambda shape, s: ((torch.rand(*shape, generator=g, dtype=torch.float64) * 2 - 1) * s).float().to(dev)
    T, E, d, dff, do = c["T"], c["E"], c["d"], c["d_ff"], c["d_out"]
    params = SMESParams(
        router_w=u((T, E, d), 1e-3 / d ** 0.5), router_b=torch.zeros(T, E, device=dev),
        layers=[ExpertLayer(u((E, dff, d), d ** -0.5), torch.zeros(E, dff, device=dev), "relu"),
                ExpertLayer(u((E, do, dff), dff ** -0.5), torch.zeros(E, do, device=dev), "identity")],
        head_w=u((T, do), do ** -0.5), head_b=torch.zeros(T, device=dev), lb_strength=c["beta"])
    B = c["B"]
    eng = SMESEngine(params, B, c["ks"], c["ka"], device=dev)
    gh = torch.Generator(device="cpu").manual_seed(1000 + rank)
    h_host = torch.randn(B, d, generator=gh).to(torch.bfloat16).pin_memory()
    rates = torch.tensor(np.resize([0.3, 0.1, 0.05, 0.2], T), dtype=torch.float32)[:, None]
    y_host = (torch.rand(T, B, generator=gh) < rates).float().pin_memory()
    loss_host = torch.zeros(3, dtype=torch.float64).pin_memory()
    eng.set_inputs(h_host.to(dev), y_host.to(dev))

    dp = DataParallelStep(eng)
    dp.capture(warmup=1)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        dp.step()
    barrier()

    # ---------------- device-resident timed region (value)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = _lib.launch_count
    per_step_launches = count_step_launches(eng)
    with ClockSampler(local) as clk:
        barrier()
        for i in range(args.steps):
            flush.zero_()
            starts[i].record()
            dp.step()
            ends[i].record()
        barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = tot.item() / args.steps
    value = world * B / (ms / 1e3)

    # ---------------- end-to-end through the public API with host buffers (e2e): every step's
    # inputs are copied H2D from pinned memory (double-buffered, step i+1's copy overlapping
    # step i) and every step's loss is read back D2H.
    from paper_2602_09386_b200.pipeline import HostStepPipeline
    pipe = HostStepPipeline(eng, step_fn=dp.step)
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):                                   # warm the pipeline path
        pipe.prefetch(h_host, y_host)
        pipe.step()
    barrier()
    flush.zero_()
    e_start.record()
    pipe.prefetch(h_host, y_host)
    for i in range(args.steps):
        last = i == args.steps - 1
        pipe.step(None if last else h_host, None if last else y_host)
    e_end.record()
    barrier()
    e_tot = torch.tensor([e_start.elapsed_time(e_end)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_tot, op=dist.ReduceOp.MAX)
    e_ms = e_tot.item() / args.steps
    e2e = {"value": world * B / (e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": h_host.numel() * h_host.element_size() + y_host.numel() * y_host.element_size(),
           "d2h_bytes_per_step": pipe.loss_host.numel() * pipe.loss_host.element_size(),
           "ms_per_step": e_ms,
           "api": "pipeline.HostStepPipeline.step (pinned H2D of each step's inputs, double-buffered on a copy "
                  "stream and overlapped with the previous step; D2H of each step's loss)"}

    # ---------------- per-kernel breakdown (eager, queued behind a sleep so events time pure GPU work)
    n_act = eng.n_act()
    kern = per_kernel_times(eng, reps=5)
    peaks, peak_src = _peaks()
    work = eng.work_model(n_act, balance=peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9))
    breakdown = {}
    for tag, t_ms in kern.items():
        fl, by, bound = work.get(tag, (0.0, 0.0, "hbm"))
        ach = (fl / (t_ms * 1e-3) / 1e12) if bound == "tensor" else (by / (t_ms * 1e-3) / 1e9)
        pk = peaks["bf16_tflops"] if bound == "tensor" else peaks["hbm_gbs"]
        breakdown[tag] = {"ms": round(t_ms, 4), "bound": bound, "achieved": round(ach, 2),
                          "unit": "TFLOP/s" if bound == "tensor" else "GB/s", "frac": round(ach / pk, 4)}
    dom = max(kern, key=kern.get)
    dominant = breakdown[dom]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom)
        except Exception:
            traffic = None
    roofline = {"kernel": dom, "bound": dominant["bound"], "achieved": dominant["achieved"],
                "peak": peaks["bf16_tflops"] if dominant["bound"] == "tensor" else peaks["hbm_gbs"],
                "unit": dominant["unit"], "frac": dominant["frac"], "traffic": traffic,
                "peak_source": f"{peak_src} (burst; kernel timed alone with CUDA events)",
                "step_share": round(kern[dom] / sum(kern.values()), 4)}
    expert_flops = sum(work[t][0] for t in kern if t in work and (t.startswith("fc") or t.startswith("mlp_"))
                       and not t.endswith("bias"))
    step_tflops = (expert_flops + sum(work[t][0] for t in ("router_fwd", "router_dgrad", "router_wgrad"))) / (ms * 1e-3) / 1e12

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = _cpu_sample(2048, 2)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": WORKLOAD, "global_batch": world * B, "per_gpu_batch": B,
                           "parallelism": f"dp{world}", "n_act_rows": n_act, "mean_union": n_act / B,
                           "l2": "flushed between steps (256 MiB memset outside the per-step event brackets)",
                           "graph": "fwd+bwd captured as 2 CUDA graphs around the LB-stats all-reduce"},
                "e2e": e2e, "gpu_launches": per_step_launches * args.steps,
                "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary(),
                "step_tflops": round(step_tflops, 1), "kernels": breakdown}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def count_step_launches(eng):
    from paper_2602_09386_b200 import _lib
    import torch
    c0 = _lib.launch_count
    eng.step()
    torch.cuda.synchronize()
    return _lib.launch_count - c0


def per_kernel_times(eng, reps=5):
    import contextlib
    import torch
    from paper_2602_09386_b200 import _lib

    rec = []

    @contextlib.contextmanager
    def timer(tag):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        yield
        b.record()
        rec.append((tag, a, b))

    acc = {}
    for _ in range(reps):
        rec.clear()
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)   # keep the GPU busy while the launches queue up
        _lib._timer = timer
        try:
            eng.step()
        finally:
            _lib._timer = None
        torch.cuda.synchronize()
        for tag, a, b in rec:
            acc[tag] = acc.get(tag, 0.0) + a.elapsed_time(b)
    return {k: v / reps for k, v in acc.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline sample")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
