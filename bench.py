#!/usr/bin/env python
"""Benchmark: SMES fwd+bwd samples/s on B200 (BASELINE.json configs[1], c2, by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c4|c5] [--transport nccl|peer]

One step = one SMES-layer fwd+bwd over one batch of synthetic KuaiRand-shaped
input: routers -> progressive routing -> dedup plan/permute -> expert MLP
(grouped tcgen05 GEMMs; the identity fc2 folded into the task heads) -> combine ->
task heads -> BCE + beta*L_lb, and the full backward (all parameter grads + d_hidden).
c2 (default, the headline): T=8 tasks, E=32 experts, K_s=4 shared + K_a=2 private,
d_model=256, expert MLP 256->512->256, batch 16384 per GPU, bf16 storage / fp32
accumulate (Stage-I routing fp64).  Weights: reference init (model.py:117-156), seed 0.
Inputs: h ~ N(0,1), Bernoulli labels at (0.3, 0.1, 0.05, 0.2) cycled.

N>1 (torchrun, one rank per GPU): c2 weak scaling (16384 per rank), c3 strong scaling
(65536 global), both data-parallel with the LB-statistics all-reduce and the gradient
all-reduce (NCCL); c5 expert-parallel (experts sharded E/N, dispatch / return all-to-all,
NCCL or the peer-memory transport).  c4 is the single-GPU inference latency sweep.
Timing: CUDA events per step, L2 flushed between steps, max over ranks.
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

CONFIGS = {
    # BASELINE.json configs (Appendix A assumptions for the fields it leaves open)
    "c1": dict(T=4, E=16, ks=2, ka=1, d=128, d_ff=256, d_out=128, B=1024, beta=0.01, mode="fwd32", scaling="weak",
               workload="c1: SMES layer fwd+loss, KuaiRand-shaped batch 1024, 4 tasks, 16 experts, shared top-2 + "
                        "private top-1, d_model=128, expert MLP 128->256->128, fp32 (bf16x3 tensor-core GEMMs)"),
    "c2": dict(T=8, E=32, ks=4, ka=2, d=256, d_ff=512, d_out=256, B=16384, beta=0.01, mode="dp", scaling="weak",
               workload="c2: SMES fwd+bwd, 8 tasks, 32 experts, shared top-4 + private top-2, d_model=256, "
                        "expert MLP 256->512->256, batch 16384 per GPU, bf16"),
    "c3": dict(T=16, E=64, ks=4, ka=2, d=512, d_ff=1024, d_out=512, B=65536, beta=0.01, mode="dp", scaling="strong",
               workload="c3: SMES fwd+bwd with multi-gate LB regularizer, 16 tasks, 64 experts, shared top-4 + "
                        "private top-2, d_model=512, expert MLP 512->1024->512, global batch 65536, data-parallel, bf16"),
    "c4": dict(T=16, E=64, ks=4, ka=2, d=512, d_ff=1024, d_out=512, beta=0.0, mode="infer",
               batches=[256, 512, 1024, 2048, 4096, 8192],
               workload="c4: SMES inference scoring (fwd only, no regularizer), 16 tasks, 64 experts, d_model=512, "
                        "expert MLP 512->1024->512, batch 256..8192 sweep, bf16"),
    "c5": dict(T=32, E=256, ks=4, ka=2, d=1024, d_ff=2048, d_out=1024, B=32768, beta=0.01, mode="ep",
               scaling="weak",
               workload="c5: SMES expert-parallel fwd+bwd, 32 tasks, 256 experts, shared top-4 + private top-2, "
                        "d_model=1024, expert MLP 1024->2048->1024, 32768 samples per GPU (the 8-GPU share of the "
                        "256K global batch), experts sharded E/N, bf16"),
}
CFG = CONFIGS["c2"]
WORKLOAD = CFG["workload"]
METRIC = "SMES fwd+bwd samples/sec"
METRIC_C1 = "SMES fwd+loss samples/sec (fp32)"
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

# bounded CPU samples of each configuration: c2 runs the FULL 16384 batch;
# c3 / c5 full batches need minutes and tens of GB of f64 (T,B,E) arrays per step
CPU_SAMPLE = {"c1": 1024, "c2": 16384, "c3": 4096, "c4": 1024, "c5": 256}


def _host_cpu():
    """CPU model and the BLAS numpy runs on (threadpoolctl), for the cpu_baseline record."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        libs = [i for i in threadpool_info() if i.get("user_api") == "blas"]
        if libs:
            b = libs[0]
            blas = f"{b.get('internal_api')} {b.get('version')} ({b.get('num_threads')} threads)"
    except Exception:
        pass
    return model, blas


def _cpu_sample(cfg_name: str, steps: int, warm: int = 1):
    """Time the oracle port (the reference's algorithm restated in NumPy f64) on a bounded
    (sub-)batch of the configuration: forward_sparse + backward (forward only for c4).
    Median of ``steps`` after ``warm`` warm-up steps (the cli.py:333-345 convention)."""
    from oracle import smes_oracle as O
    c = CONFIGS[cfg_name]
    b_sample = CPU_SAMPLE[cfg_name]
    rng = np.random.default_rng(0)
    p = O.init_layer_params(rng, c["d"], c["d_out"], c["E"], c["T"], d_ff=c["d_ff"])
    h = rng.normal(size=(b_sample, c["d"]))
    y = (rng.uniform(size=(c["T"], b_sample)) < np.resize([0.3, 0.1, 0.05, 0.2], c["T"])[:, None]).astype(float)
    fwd_only = c["mode"] in ("infer", "fwd32")
    times = []
    for i in range(warm + steps):
        t0 = time.perf_counter()
        f = O.forward_sparse(h, p, c["ks"], c["ka"])
        if not fwd_only:
            O.backward(f, p, y, None, c["beta"])
        dt = time.perf_counter() - t0
        if i >= warm:
            times.append(dt)
    med = statistics.median(times)
    cores = len(os.sched_getaffinity(0))
    what = "forward_sparse" if fwd_only else "forward_sparse+backward"
    full = c.get("B") == b_sample
    model, blas = _host_cpu()
    return {"value": b_sample / med, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{cfg_name} shape at B={b_sample} ({'the full batch' if full else 'sub-batch'}), "
                      f"oracle/smes_oracle.py {what}, median of {steps} steps after {warm} warm-up, "
                      f"numpy f64 with {cores} host threads",
            "full_batch": full, "cpu_model": model, "blas": blas}


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(len(os.sched_getaffinity(0))))
    c = CONFIGS[args.config]
    steps = max(1, min(args.steps, 5))
    cb = _cpu_sample(args.config, steps, warm=min(1, args.warmup))
    b_sample = CPU_SAMPLE[args.config]
    metric = {"infer": "SMES inference samples/sec", "fwd32": METRIC_C1}.get(c["mode"], METRIC)
    line = {"impl": "reference", "metric": metric, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": min(1, args.warmup), "ms_per_step": 1e3 * b_sample / cb["value"],
            "higher_is_better": True, "scaling": c.get("scaling", "weak"), "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": c["workload"], "global_batch": c.get("B", b_sample) * (args.gpus if c.get(
                "scaling") == "weak" else 1), "parallelism": f"{c['mode']}{args.gpus}",
                       "reference_sample_batch": b_sample},
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


def _make_params(c, dev, expert_range=None):
    """Reference init (model.py:117-156): experts/heads U(+-1/sqrt(fan_in)), routers
    U(+-1e-3/sqrt(d)), biases 0; seed 0.  ``expert_range`` keeps only [lo, hi) of the experts
    (expert parallelism); the full bank is drawn so every rank sees the same weights."""
    import torch
    from paper_2602_09386_b200 import ExpertLayer, SMESParams
    g = torch.Generator(device="cpu").manual_seed(0)
    u = lambda shape, s: ((torch.rand(*shape, generator=g, dtype=torch.float32) * 2 - 1) * s)
    T, E, d, dff, do = c["T"], c["E"], c["d"], c["d_ff"], c["d_out"]
    rw = u((T, E, d), 1e-3 / d ** 0.5)
    w1 = u((E, dff, d), d ** -0.5)
    w2 = u((E, do, dff), dff ** -0.5)
    hw = u((T, do), do ** -0.5)
    lo, hi = expert_range or (0, E)
    dv = lambda t: t.to(dev)
    return SMESParams(router_w=dv(rw), router_b=torch.zeros(T, E, device=dev),
                      layers=[ExpertLayer(dv(w1[lo:hi]), torch.zeros(hi - lo, dff, device=dev), "relu"),
                              ExpertLayer(dv(w2[lo:hi]), torch.zeros(hi - lo, do, device=dev), "identity")],
                      head_w=dv(hw), head_b=torch.zeros(T, device=dev), lb_strength=c["beta"])


def _host_inputs(c, B, rank):
    import torch
    gh = torch.Generator(device="cpu").manual_seed(1000 + rank)
    h_host = torch.randn(B, c["d"], generator=gh).to(torch.bfloat16).pin_memory()
    rates = torch.tensor(np.resize([0.3, 0.1, 0.05, 0.2], c["T"]), dtype=torch.float32)[:, None]
    y_host = (torch.rand(c["T"], B, generator=gh) < rates).float().pin_memory()
    return h_host, y_host


def _oracle_params(params):
    """The bench's SMESParams as the oracle sees them: the kernel operands (bf16 router and
    expert weights, fp32 biases and heads) upcast to f64 -- identical operands."""
    from oracle import smes_oracle as O
    f64 = lambda t, bf=False: (t.detach().to(torch_bf16()) if bf else t.detach()).double().cpu().numpy()
    return O.LayerParams(router_w=f64(params.router_w, True), router_b=f64(params.router_b),
                         layers=[(f64(l.weight, True), f64(l.bias), l.act) for l in params.layers],
                         head_w=f64(params.head_w), head_b=f64(params.head_b))


def torch_bf16():
    import torch
    return torch.bfloat16


def parity_sample(src, params, labels, n_rows=256, full_loss=True):
    """Checker run next to the CPU baseline (oracle = test infrastructure, never measured): on an
    evenly spaced row subset of the batch the timed steps just processed, the router logits against
    RouterBank.logits (routing.py:101-103), the expert selections index-exact against route_batch
    (routing.py:235-281), and predictions + BCE of those rows against forward_sparse with the GPU's
    selections (model.py:284-300, training.py:54-57).  Also the full-batch loss against the BCE of
    the GPU's own predictions (the loss reduction)."""
    import torch
    from oracle import smes_oracle as O
    T, E, B, ks, ka = src.T, src.E, src.B, src.ks, src.ka
    rows = np.linspace(0, B - 1, min(n_rows, B)).astype(np.int64)
    p = _oracle_params(params)
    h = src.h.double().cpu().numpy()[rows]
    z = src.z.double().cpu().numpy().reshape(B, T, E)[rows].transpose(1, 0, 2)
    zr = O.router_logits(h, p)
    z_rel = float(np.abs(z - zr).max() / np.abs(zr).max())
    r = O.route_batch(z, ks, ka, p.task_weights)
    act = src.active.cpu().numpy()[:, rows]
    sel_ok = bool(np.array_equal(act, r.active) and np.array_equal(src.shared.cpu().numpy()[rows], r.shared))
    plan = O.build_execution_plan(r.unions, E)
    f = O.forward_sparse(h, p, ks, ka, logits=z, frozen=r, frozen_plan=plan)
    preds = src.preds.double().cpu().numpy()
    y = labels.double().cpu().numpy()
    pr_rel = float(np.abs(preds[:, rows] - f.predictions).max() / np.abs(f.predictions).max())
    lam = np.ones(T)
    bce_gpu_rows = O.weighted_bce(preds[:, rows], y[:, rows], lam)
    bce_ora_rows = O.weighted_bce(f.predictions, y[:, rows], lam)
    loss = src.loss_out.double().cpu().numpy()
    bce_full = O.weighted_bce(preds, y, lam)
    ok = sel_ok and z_rel < 1e-5 and pr_rel < 2e-2 and abs(bce_gpu_rows - bce_ora_rows) < 2e-2 * bce_ora_rows \
        and (not full_loss or abs(loss[0] - bce_full) < 1e-5 * bce_full)
    return {"ok": bool(ok), "rows": int(len(rows)), "selections_index_exact": sel_ok,
            "router_logits_rel": z_rel, "predictions_rel": pr_rel,
            "bce_rows_gpu": bce_gpu_rows, "bce_rows_oracle": bce_ora_rows,
            "loss_gpu": float(loss[0]), "loss_from_gpu_preds": bce_full,
            "stage1_min_margin": float(O.stage1_margin(z, ks)) if ks > 0 else None,
            "tolerances": "logits 1e-5 (identical bf16 operands, fp32 accumulate), selections exact, "
                          "predictions / BCE 2e-2 (bf16), loss reduction 1e-5"}


def _roofline(kern, work, peaks, peak_src, config="c2"):
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
    if config == "c2" and os.path.exists(tpath):      # the committed ncu capture is of the c2 step
        try:
            traffic = json.load(open(tpath)).get(dom)
        except Exception:
            traffic = None
    roofline = {"kernel": dom, "bound": dominant["bound"], "achieved": dominant["achieved"],
                "peak": peaks["bf16_tflops"] if dominant["bound"] == "tensor" else peaks["hbm_gbs"],
                "unit": dominant["unit"], "frac": dominant["frac"], "traffic": traffic,
                "peak_source": f"{peak_src} (burst; kernel timed alone with CUDA events)",
                "step_share": round(kern[dom] / sum(kern.values()), 4)}
    return roofline, breakdown


def _timed_steps(step_fn, steps, world, dev, flush, local):
    import torch
    import torch.distributed as dist

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    with ClockSampler(local) as clk:
        barrier()
        for i in range(steps):
            flush.zero_()
            starts[i].record()
            step_fn()
            ends[i].record()
        barrier()
    step_ms = [s_.elapsed_time(e) for s_, e in zip(starts, ends)]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    return tot.item() / steps, clk.summary()


def _timed_e2e(pipe, h_host, y_host, steps, world, dev, flush):
    """End to end through the host-fed step API: each step's inputs copied H2D from pinned
    memory (double-buffered, overlapped with the previous step) and its loss read back D2H."""
    import torch
    import torch.distributed as dist
    for _ in range(2):
        pipe.prefetch(h_host, y_host)
        pipe.step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    flush.zero_()
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_start.record()
    pipe.prefetch(h_host, y_host)
    for i in range(steps):
        last = i == steps - 1
        pipe.step(None if last else h_host, None if last else y_host)
    e_end.record()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e_tot = torch.tensor([e_start.elapsed_time(e_end)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_tot, op=dist.ReduceOp.MAX)
    return e_tot.item() / steps


def run_ours(args):
    import torch
    import torch.distributed as dist
    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    c = CONFIGS[args.config]
    mode = c["mode"]
    if mode == "dp":
        line = run_dp(args, c, world, rank, local, dev)
    elif mode == "ep":
        line = run_ep(args, c, world, rank, local, dev)
    elif mode == "fwd32":
        line = run_fwd32(args, c, world, rank, local, dev)
    else:
        line = run_infer(args, c, world, rank, local, dev)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_dp(args, c, world, rank, local, dev):
    import torch
    from paper_2602_09386_b200 import SMESEngine, _lib
    from paper_2602_09386_b200.dp import DataParallelStep
    from paper_2602_09386_b200.pipeline import HostStepPipeline

    B = c["B"] if c["scaling"] == "weak" else c["B"] // world
    eng = SMESEngine(_make_params(c, dev), B, c["ks"], c["ka"], device=dev)
    h_host, y_host = _host_inputs(c, B, rank)
    eng.set_inputs(h_host.to(dev), y_host.to(dev))
    eng.keep_logits = False        # the training step does not write the router logits (fused front)
    # N > 1: LoadStats over CUDA-IPC peer memory + gradient buckets overlapped with the backward;
    # the whole step (collectives included) is one CUDA graph.  SMES_DP_SAFE=1: NCCL statistics,
    # one gradient all-reduce after the backward, two graphs (round-1 path).
    safe = os.environ.get("SMES_DP_SAFE") == "1"
    dp = DataParallelStep(eng, stats="group" if safe else "peer", overlap=not safe)
    try:
        dp.capture(warmup=1)
    except Exception as err:     # a graph capture the NCCL build refuses: keep the eager step
        print(f"dp capture failed ({err}); eager step", file=sys.stderr, flush=True)
        dp._ga = dp._gb = None
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)   # > 126 MB L2
    for _ in range(args.warmup):
        dp.step()
    per_step_launches = count_step_launches(eng.step)
    ms, clocks = _timed_steps(dp.step, args.steps, world, dev, flush, local)
    value = world * B / (ms / 1e3)
    pipe = HostStepPipeline(eng, step_fn=dp.step)
    e_ms = _timed_e2e(pipe, h_host, y_host, args.steps, world, dev, flush)
    e2e = {"value": world * B / (e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": h_host.numel() * h_host.element_size() + y_host.numel() * y_host.element_size(),
           "d2h_bytes_per_step": pipe.loss_host.numel() * pipe.loss_host.element_size(), "ms_per_step": e_ms,
           "api": "pipeline.HostStepPipeline.step (pinned H2D of each step's inputs, double-buffered on a copy "
                  "stream and overlapped with the previous step; D2H of each step's loss)"}
    n_act = eng.n_act()
    parity = None
    if rank == 0 and not args.no_cpu:
        # one more step of the same batch with the logits written out, for the checker
        eng.keep_logits = True
        dp.step_eager()
        torch.cuda.synchronize()
        eng.keep_logits = False
        parity = parity_sample(eng, eng.p, eng.labels, full_loss=world == 1)
    kern = per_kernel_times(eng.step, reps=5, serial=eng)
    peaks, peak_src = _peaks()
    work = eng.work_model(n_act, balance=peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9))
    roofline, breakdown = _roofline(kern, work, peaks, peak_src, args.config)
    expert_flops = sum(work[t][0] for t in kern if t in work and (t.startswith("fc") or t.startswith("mlp_"))
                       and not t.endswith("bias"))
    # the expert MLP as the reference computes it (no head folding): fc1 + fc2 forward, dgrad of
    # both, wgrad of both = 3 x 2 x N_act x (d d_ff + d_ff d_out) FLOP per step
    nominal = 3 * 2.0 * n_act * (c["d"] * c["d_ff"] + c["d_ff"] * c["d_out"])
    expert_gemm = {"nominal_flop_per_step": nominal,
                   "nominal_tflops": round(nominal / (ms * 1e-3) / 1e12, 1),
                   "nominal_frac_of_bf16_peak": round(nominal / (ms * 1e-3) / 1e12 / peaks["bf16_tflops"], 4),
                   "note": "nominal = the unfolded expert MLP (what the reference computes) over the whole step "
                           "time; the kernels run the folded algebra (DESIGN.md section 2), fewer FLOPs"}
    comparator = gemm_comparator(eng, peaks) if rank == 0 else None
    api = e2e_api(c, dev, args.steps) if (rank == 0 and world == 1 and args.config == "c2") else None
    step_tflops = (expert_flops + sum(work[t][0] for t in ("router_fwd", "router_dgrad", "router_wgrad"))) / (
        ms * 1e-3) / 1e12
    cpu = _cpu_sample(args.config, 2) if (rank == 0 and not args.no_cpu) else None
    if rank != 0:
        return None
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": c["scaling"],
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": c["workload"], "global_batch": world * B, "per_gpu_batch": B,
                       "parallelism": f"dp{world}", "n_act_rows": n_act, "mean_union": n_act / B,
                       "l2": "flushed between steps (256 MiB memset outside the per-step event brackets)",
                       "graph": ("fwd+bwd in one CUDA graph" if world == 1 else "fwd+bwd captured as 2 CUDA graphs around the LB-stats all-reduce")},
            "e2e": e2e, "gpu_launches": per_step_launches * args.steps,
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks, "parity": parity,
            "step_tflops": round(step_tflops, 1), "expert_gemm": expert_gemm, "gemm_comparator": comparator,
            "e2e_api": api, "kernels": breakdown,
            "kernels_note": "per-kernel CUDA-event times from an eager step with the backward side stream "
                            "serialised onto the timing stream (so each kernel is timed alone, like ncu)"}


def gemm_comparator(eng, peaks, reps=10):
    """Library anchor for the grouped GEMM: the fc1 forward of this batch (padded expert segments,
    X (rows, d) x W1_e^T) through our tcgen05 kernel (smes_gemm_ragged_m, no epilogue) and through
    torch._grouped_mm (PyTorch's CUTLASS grouped GEMM) on the same operands, CUDA events, L2 warm."""
    import torch
    from paper_2602_09386_b200._lib import call, ptr
    E, d, dff = eng.E, eng.d, eng.dims[1]
    rows = int(eng.seg_pad[E].item())
    a = eng.X[:rows, :d].contiguous()
    w = eng.w_bf[0]                                   # (E, d_ff, d)
    out = torch.empty(rows, dff, dtype=torch.bfloat16, device=a.device)
    st = torch.cuda.current_stream().cuda_stream

    def ours():
        call("smes_gemm_ragged_m", ptr(a), d, rows, ptr(w), E, dff, d, 0, ptr(eng.seg_pad), None, 0, None, None, 0,
             ptr(out), dff, 0, rows, st)

    def timeit(fn):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    flop = 2.0 * rows * d * dff
    res = {"shape": f"fc1 forward, {rows} padded rows in {E} expert groups, K={d}, N={dff}, bf16 -> bf16",
           "ours_ms": None, "torch_grouped_mm_ms": None}
    t = timeit(ours)
    res["ours_ms"] = round(t, 4)
    res["ours_tflops"] = round(flop / (t * 1e-3) / 1e12, 1)
    try:
        offs = eng.seg_pad[1:E + 1].contiguous()
        wt = w.transpose(1, 2)                       # (E, d, d_ff) view: the layout grouped_mm wants
        ref = torch._grouped_mm(a, wt, offs=offs)
        t2 = timeit(lambda: torch._grouped_mm(a, wt, offs=offs))
        ours()
        torch.cuda.synchronize()
        res["torch_grouped_mm_ms"] = round(t2, 4)
        res["torch_grouped_mm_tflops"] = round(flop / (t2 * 1e-3) / 1e12, 1)
        res["max_rel_diff"] = float((out.float() - ref.float()).abs().max() / ref.float().abs().max())
    except Exception as err:           # library path unavailable on this build: say so
        res["torch_grouped_mm_error"] = str(err)[:200]
    res["bf16_peak_tflops"] = peaks["bf16_tflops"]
    return res


def e2e_api(c, dev, steps):
    """The drop-in API end to end (the calls a user of the reference makes): forward_sparse on a
    host batch (H2D inside), backward with host labels (H2D), the loss read back (D2H) and the
    gradient blocks returned as fresh device tensors -- per step, CUDA events, L2 flushed between
    steps outside the brackets."""
    import torch
    import paper_2602_09386_b200 as smes
    params = _make_params(c, dev)
    T, E = c["T"], c["E"]
    pools = [smes.ExpertPool([smes.Affine(l.weight[e], l.bias[e]) for e in range(E)], l.act) for l in params.layers]
    routers = smes.RouterBank([smes.Affine(params.router_w[t], params.router_b[t]) for t in range(T)])
    heads = [smes.Affine(params.head_w[t:t + 1], params.head_b[t:t + 1]) for t in range(T)]
    model = smes.MoeModel(None, None, pools, routers, heads, torch.ones(T), c["beta"],
                          smes.RoutingBudget(c["ks"], c["ka"]))
    h_host, y_host = _host_inputs(c, c["B"], 0)
    x_host = h_host.float().pin_memory()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for _ in range(3):
        res = smes.forward_sparse(x_host, model)
        smes.backward(res, model, y_host)
    n = max(5, min(steps, 20))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for e0, e1 in ev:
        flush.zero_()
        e0.record()
        res = smes.forward_sparse(x_host, model)
        bw = smes.backward(res, model, y_host)
        e1.record()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / n
    return {"value": c["B"] / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "loss": bw.total,
            "h2d_bytes_per_step": x_host.numel() * 4 + y_host.numel() * 4, "d2h_bytes_per_step": 24,
            "api": "paper_2602_09386_b200.forward_sparse(host batch) + backward(result, model, host labels): "
                   "reference-shaped results (routing, plan, task reps, named gradient blocks), host syncs "
                   "for the reference's validation and float losses"}


def run_ep(args, c, world, rank, local, dev):
    import torch
    from paper_2602_09386_b200.ep import EPRank, ExpertParallelStep, LoopbackComm, NcclComm, PeerComm
    from paper_2602_09386_b200.pipeline import HostStepPipeline

    B = c["B"]
    E = c["E"]
    El = E // world
    rk = EPRank(_make_params(c, dev, (rank * El, (rank + 1) * El)), E, rank, world, B, c["ks"], c["ka"],
                device=dev, capacity_factor=1.25)
    h_host, y_host = _host_inputs(c, B, rank)
    rk.set_inputs(h_host.to(dev), y_host.to(dev))
    if world == 1:
        comm = LoopbackComm([rk], fused=args.transport == "peer")
    elif args.transport == "peer":
        comm = PeerComm(rk)
    else:
        comm = NcclComm(rk)
    ep = ExpertParallelStep([rk], comm)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        ep.step()
    torch.cuda.synchronize()
    rk.check()
    per_step_launches = count_step_launches(ep.step)
    ms, clocks = _timed_steps(ep.step, args.steps, world, dev, flush, local)
    value = world * B / (ms / 1e3)
    pipe = HostStepPipeline(rk, step_fn=ep.step)
    e_ms = _timed_e2e(pipe, h_host, y_host, args.steps, world, dev, flush)
    e2e = {"value": world * B / (e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": h_host.numel() * h_host.element_size() + y_host.numel() * y_host.element_size(),
           "d2h_bytes_per_step": pipe.loss_host.numel() * pipe.loss_host.element_size(), "ms_per_step": e_ms,
           "api": "pipeline.HostStepPipeline.step over ep.ExpertParallelStep.step"}
    rk.check()
    n_own = int(rk.totals_o[2].item())
    n_src = int(rk.totals[2].item())
    parity = None
    if rank == 0 and not args.no_cpu:
        parity = parity_sample(rk, rk.p, rk.labels, full_loss=world == 1)
    kern = per_kernel_times(ep.step, reps=2)
    peaks, peak_src = _peaks()
    sh = rk.shard
    d, dff, T, E, El, K = c["d"], c["d_ff"], c["T"], c["E"], rk.El, rk.K
    bal = peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    fl = 2.0 * n_own * d * dff
    sent = int(rk.cnt.sum().item())
    Br = rk.Br
    # algorithmic (flops, bytes) per launch tag of one EP step on this rank (SURVEY 8d formulas;
    # n_src = packed rows of the local batch over all E experts, n_own = rows this rank's experts run)
    work = {"router_fwd": (2.0 * B * d * T * E, B * (d * 2 + T * E * 4)),
            "router_dgrad": (2.0 * B * d * T * E, B * (T * E * 2 + d * 4)),
            "router_wgrad": (2.0 * B * d * T * E, B * (T * E * 2 + d * 2)),
            "route": (0.0, B * (T * E * 4 + T * K * 8 + c["ks"] * 4 + rk.EW * 4 + 4)),
            "plan_reduce": (0.0, rk.C * E * 24),
            "plan_scatter": (0.0, B * (rk.EW * 4 + rk.umax * 4) + n_src * (8 + rk.ldc * 2)),
            "ep_pack": (0.0, B * (d * 2 + rk.EW * 4) + sent * (d * 2 + rk.wpr * 4)),
            "owner_plan": (0.0, Br * rk.wpr * 4 * 2 + rk.C_o * El * 8),
            "owner_scatter": (0.0, Br * d * 2 + n_own * (d * 2 + 8 + sh.ldc * 2)),
            "fold_heads": (2.0 * El * T * d * dff, El * d * dff * 2 + El * sh.ldg * dff * 2),
            "fc1_fwd": (fl, n_own * (d + dff) * 2 + n_own * dff / 8),
            "fc1_dgrad": (fl, n_own * (d + dff) * 2),
            "fc1_wgrad": (fl, n_own * (d + dff) * 2),
            "mlp_fwd": (fl + 2.0 * n_own * dff * T, n_own * (d * 2 + dff * 2 + dff / 8 + sh.ldp * 4)),
            "mlp_dgrad": (fl + 2.0 * n_own * dff * T, n_own * (sh.ldc * 2 + dff / 8 + d * 2 + dff * 2)),
            "fc2_fwd_folded": (2.0 * n_own * dff * T, n_own * (dff * 2 + sh.ldp * 4)),
            "fc2_dgrad_folded": (2.0 * n_own * dff * T, n_own * (sh.ldc * 2 + dff * 2 + dff / 8)),
            "fc2_wgrad_folded": (2.0 * n_own * dff * T, n_own * (dff * 2 + sh.ldc * 2)),
            "unfold": (4.0 * El * T * d * dff, El * dff * sh.ldg * 4 + El * d * dff * 6),
            "ep_segments": (0.0, El * rk.n * 12),
            "ep_copy_rows": (0.0, 2 * (n_own + n_src) * (rk.ldp * 4 + rk.ldc * 2)),
            "combine_train": (0.0, B * (rk.umax * T * 4 + T * K * 8 + T * 16 + T * E * 2) + n_src * rk.ldc * 2),
            "unpermute": (0.0, n_own * d * 2 + Br * d * 4),
            "ep_combine_dh": (0.0, rk.n * B * d * 4 + B * d * 8)}
    work = {k: (f, b, "tensor" if b > 0 and f / b > bal else "hbm") for k, (f, b) in work.items()}
    roofline, breakdown = _roofline(kern, work, peaks, peak_src, args.config)
    expert_flops = 3 * fl + 3 * 2.0 * n_own * dff * T
    cpu = _cpu_sample(args.config, 1) if (rank == 0 and not args.no_cpu) else None
    if rank != 0:
        return None
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": c["scaling"],
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": c["workload"], "global_batch": world * B, "per_gpu_batch": B,
                       "parallelism": f"ep{world}", "experts_per_gpu": El,
                       "transport": (f"loopback (1 rank, {args.transport} code path)" if world == 1
                                     else args.transport),
                       "expert_rows_on_rank0": n_own,
                       "l2": "flushed between steps (256 MiB memset outside the per-step event brackets)"},
            "e2e": e2e, "gpu_launches": per_step_launches * args.steps,
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks, "parity": parity,
            "step_tflops": round(expert_flops / (ms * 1e-3) / 1e12, 1), "kernels": breakdown}


def run_infer(args, c, world, rank, local, dev):
    """c4: fwd-only scoring (routers, routing, plan, expert MLP with the folded heads, combine ->
    predictions; `SMESEngine.score`), one CUDA graph per batch size, p50/p99 over >= 1000 replays
    each.  Ranks > 0 idle (single-GPU configuration)."""
    import torch
    from paper_2602_09386_b200 import SMESEngine, _lib
    if rank != 0:
        return None
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    c = dict(c, beta=0.0)
    params = _make_params(c, dev)
    sweep, launches = {}, 0
    clocks_all = []
    reps = max(1000, args.steps)
    for Bb in c["batches"]:
        eng = SMESEngine(params, Bb, c["ks"], c["ka"], device=dev)
        eng.keep_logits = False        # scoring does not return the router logits / dense statistics
        h_host, y_host = _host_inputs(c, Bb, rank)
        eng.set_inputs(h_host.to(dev), y_host.to(dev))
        st = torch.cuda.Stream(dev)
        st.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(st):
            eng.score()
        torch.cuda.current_stream(dev).wait_stream(st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            eng.score()
        for _ in range(max(3, args.warmup)):
            g.replay()
        torch.cuda.synchronize()
        c0 = _lib.launch_count
        eng.score()
        per = _lib.launch_count - c0
        ts = []
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        with ClockSampler(local) as clk:
            for a, b in ev:
                flush.zero_()
                a.record()
                g.replay()
                b.record()
            torch.cuda.synchronize()
        clocks_all.append(clk.summary())
        ts = sorted(a.elapsed_time(b) for a, b in ev)
        launches += per * reps
        # end to end: pinned H2D of h, graph, D2H of the predictions
        preds_host = torch.empty(c["T"], Bb, dtype=torch.float32).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_e2e = 200
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n_e2e):
            eng.h.copy_(h_host, non_blocking=True)
            g.replay()
            preds_host.copy_(eng.preds, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        sweep[str(Bb)] = {"p50_ms": ts[len(ts) // 2], "p99_ms": ts[min(len(ts) - 1, int(0.99 * len(ts)))],
                          "samples_per_s": Bb / (ts[len(ts) // 2] / 1e3),
                          "e2e_ms": e0.elapsed_time(e1) / n_e2e, "launches_per_batch": per}
        last = (Bb, eng, h_host, preds_host)
        del g
    Bb, eng, h_host, preds_host = last
    top = sweep[str(Bb)]
    # roofline of the largest batch's scoring pass: per-kernel CUDA events (eager, one stream)
    n_act = eng.n_act()
    kern = per_kernel_times(eng.score, reps=5, serial=eng)
    peaks, peak_src = _peaks()
    work = eng.work_model(n_act, balance=peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9))
    roofline, breakdown = _roofline(kern, work, peaks, peak_src, args.config)
    cpu = _cpu_sample(args.config, 2) if not args.no_cpu else None
    return {"metric": f"SMES inference p50 latency per batch (B={Bb})", "value": top["p50_ms"], "unit": "ms",
            "n_gpus": 1, "steps": reps, "warmup": max(3, args.warmup), "ms_per_step": top["p50_ms"],
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": c["workload"], "global_batch": Bb, "parallelism": "single-GPU",
                       "l2": "flushed before every timed replay (256 MiB memset outside the event brackets)",
                       "graph": "one CUDA graph per batch size"},
            "e2e": {"value": top["e2e_ms"], "unit": "ms", "h2d_bytes_per_step": h_host.numel() * 2,
                    "d2h_bytes_per_step": preds_host.numel() * 4,
                    "api": "pinned H2D of h, graph replay of SMESEngine.score, D2H of predictions"},
            "gpu_launches": launches, "sweep": sweep, "cpu_baseline": cpu, "clocks": _merge_clocks(clocks_all),
            "roofline": roofline, "kernels": breakdown}


def run_fwd32(args, c, world, rank, local, dev):
    """c1: the SMES layer forward + loss in fp32 (fp32.SMESForwardF32: bf16x3 tensor-core GEMMs, fp64
    Stage-I routing, fp32 combine/heads/BCE), one CUDA graph per step.  N > 1: independent replicas
    (batch-sharded, weak scaling; the forward has no cross-rank exchange but the LB statistics,
    which the fwd+loss value reads only for the regularizer term -- replicas report their own)."""
    import torch
    import torch.distributed as dist
    from paper_2602_09386_b200 import _lib
    from paper_2602_09386_b200.fp32 import SMESForwardF32
    B = c["B"]
    params = _make_params(c, dev)
    eng = SMESForwardF32(params, B, c["ks"], c["ka"], device=dev)
    gh = torch.Generator(device="cpu").manual_seed(1000 + rank)
    h_host = torch.randn(B, c["d"], generator=gh).pin_memory()
    rates = torch.tensor(np.resize([0.3, 0.1, 0.05, 0.2], c["T"]), dtype=torch.float32)[:, None]
    y_host = (torch.rand(c["T"], B, generator=gh) < rates).float().pin_memory()
    eng.set_inputs(h_host.to(dev), y_host.to(dev))
    st = torch.cuda.Stream(dev)
    st.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(st):
        eng.forward(with_loss=True)
    torch.cuda.current_stream(dev).wait_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        eng.forward(with_loss=True)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        g.replay()
    per_step = count_step_launches(lambda: eng.forward(with_loss=True))
    ms, clocks = _timed_steps(g.replay, args.steps, world, dev, flush, local)
    # end to end: pinned H2D of h and labels, the graph, D2H of the loss
    loss_host = torch.empty(3, dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for e0, e1 in ev:
        flush.zero_()                     # outside the bracket, as in the device-timed loop
        e0.record()
        eng.h.copy_(h_host, non_blocking=True)
        eng.labels.copy_(y_host, non_blocking=True)
        g.replay()
        loss_host.copy_(eng.loss_out, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    e_ms = e_ms.item()
    parity = None
    if rank == 0 and not args.no_cpu:
        parity = parity_fp32(eng, params)
    n_act = eng.n_act()
    kern = per_kernel_times(lambda: eng.forward(with_loss=True), reps=5)
    peaks, peak_src = _peaks()
    work = eng.work_model(n_act, balance=peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9))
    roofline, breakdown = _roofline(kern, work, peaks, peak_src, args.config)
    cpu = _cpu_sample(args.config, 3) if (rank == 0 and not args.no_cpu) else None
    if rank != 0:
        return None
    return {"metric": METRIC_C1, "value": world * B / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": c["workload"], "global_batch": world * B, "per_gpu_batch": B,
                       "parallelism": f"replicas{world}", "n_act_rows": n_act,
                       "l2": "flushed between steps (256 MiB memset outside the per-step event brackets)",
                       "graph": "fwd+loss in one CUDA graph"},
            "e2e": {"value": world * B / (e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": h_host.numel() * 4 + y_host.numel() * 4, "d2h_bytes_per_step": 24,
                    "ms_per_step": e_ms,
                    "api": "per step: pinned H2D of h and labels, graph replay of SMESForwardF32.forward, D2H of "
                           "the loss (CUDA events around the three; L2 flushed between steps)"},
            "gpu_launches": per_step * args.steps, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
            "parity": parity, "kernels": breakdown,
            "kernels_note": "per-kernel CUDA-event times from an eager forward on one stream"}


def parity_fp32(eng, params):
    """Checker (oracle = test infrastructure): the whole c1 batch against the f64 oracle on the same
    fp32 operands -- logits, selections (index-exact on the GPU's logits), predictions, loss."""
    from oracle import smes_oracle as O
    T, E, B, ks, ka = eng.T, eng.E, eng.B, eng.ks, eng.ka
    f64 = lambda t: t.detach().double().cpu().numpy()
    p = O.LayerParams(router_w=f64(params.router_w), router_b=f64(params.router_b),
                      layers=[(f64(l.weight), f64(l.bias), l.act) for l in params.layers],
                      head_w=f64(params.head_w), head_b=f64(params.head_b))
    h = f64(eng.h)
    z = eng.z.double().cpu().numpy().reshape(B, T, E).transpose(1, 0, 2)
    zr = O.router_logits(h, p)
    z_rel = float(np.abs(z - zr).max() / np.abs(zr).max())
    r = O.route_batch(z, ks, ka)
    sel_ok = bool(np.array_equal(eng.active.cpu().numpy(), r.active))
    f = O.forward_sparse(h, p, ks, ka, logits=z, frozen=r)
    pr_rel = float(np.abs(f64(eng.preds) - f.predictions).max() / np.abs(f.predictions).max())
    bw = O.backward(f, p, f64(eng.labels), None, params.lb_strength)
    lo = eng.loss_out.double().cpu().numpy()
    loss_rel = abs(lo[2] - bw.total) / abs(bw.total)
    ok = sel_ok and z_rel < 1e-5 and pr_rel < 1e-5 and loss_rel < 1e-5
    return {"ok": bool(ok), "rows": int(B), "selections_index_exact": sel_ok, "router_logits_rel": z_rel,
            "predictions_rel": pr_rel, "loss_gpu": float(lo[2]), "loss_oracle": float(bw.total),
            "loss_rel": float(loss_rel), "tolerances": "fp32 1e-5 relative (north star), selections exact"}


def _merge_clocks(cl):
    """One clocks record over the per-batch-size samplers (median of medians, union of reasons)."""
    med = [c["sm_mhz"] for c in cl if c.get("sm_mhz")]
    return {"sm_mhz": float(statistics.median(med)) if med else None,
            "sm_max_mhz": next((c["sm_max_mhz"] for c in cl if c.get("sm_max_mhz")), None),
            "reasons": sorted({r for c in cl for r in c.get("reasons", [])}),
            "samples": sum(c.get("samples", 0) for c in cl), "per_batch": cl}


def count_step_launches(step_fn):
    from paper_2602_09386_b200 import _lib
    import torch
    c0 = _lib.launch_count
    step_fn()
    torch.cuda.synchronize()
    return _lib.launch_count - c0


def per_kernel_times(step_fn, reps=5, serial=None):
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
    if serial is not None:
        serial.serial = True        # one stream: the events bracket exactly the tagged launch
    for _ in range(reps):
        rec.clear()
        torch.cuda.synchronize()
        torch.cuda._sleep(20_000_000)   # keep the GPU busy while the launches queue up
        _lib._timer = timer
        try:
            step_fn()
        finally:
            _lib._timer = None
        torch.cuda.synchronize()
        for tag, a, b in rec:
            acc[tag] = acc.get(tag, 0.0) + a.elapsed_time(b)
    if serial is not None:
        serial.serial = False
    return {k: v / reps for k, v in acc.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline sample")
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS),
                    help="BASELINE.json configuration (default c2, the headline)")
    ap.add_argument("--transport", default="peer", choices=["nccl", "peer"],
                    help="c5 all-to-all: the fused CUDA-IPC peer-memory put (default) or NCCL all_to_all_single")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
