#!/usr/bin/env python
"""Benchmark: split-FC softmax-CE fwd+bwd samples/s on 1..8 B200 (BASELINE.json metric).

One step = one pass of the whole hot path (bridge all-gather,
logits GEMM with fused row statistics, cross-GPU stats combine + loss, softmax-minus-
onehot gradient, dW GEMM, dX GEMM + reduce-scatter) over one synthetic batch, through the
C-ABI.  Default workload: configs[1] c2 (D=2048, C=100K, B=32 per GPU, bf16, even shards).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
  N > 1: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Prints ONE JSON line on rank 0.  `--impl reference` times the fp64 CPU oracle (the only
reference this paper-only tier has) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic as syn  # noqa: E402

METRIC = "split-FC softmax-CE fwd+bwd samples/s"
UNIT = "samples/s"
L2_BYTES = 126 * 2 ** 20
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        d["source"] = "measured"
        return d
    except Exception:
        return dict(FALLBACK_PEAKS)


def capacity_for(cfg, world):
    """The config's capacity weights for `world` ranks (c3's 2:1:...:1 pattern keeps its first
    `world` entries, so the uneven plan also runs on fewer than 8 GPUs)."""
    if cfg.capacity is None:
        return None
    cap = list(cfg.capacity[:world]) + [1] * max(0, world - len(cfg.capacity))
    return cap if world > 1 else None


def workload_desc(name, cfg, world):
    cap = capacity_for(cfg, world)
    shards = "even" if cap is None else ":".join(str(c) for c in cap)
    return (f"{name}: D={cfg.D}, C={cfg.C}, B={cfg.B}/GPU x {world} GPU(s), {cfg.dtype}, {shards} class shards "
            f"(split-FC softmax-CE, Whale hybrid DP+MP)")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons in a background thread."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev_index: int, period_s: float = 0.001):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period_s
        self.dev = dev_index
        self._stop = threading.Event()
        self.t = None
        self.sm_max = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.sm_max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.t:
            self._stop.set()
            self.t.join()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.sm_max, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.sm_max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- oracle timing
def time_oracle(cfg, seed, min_seconds: float, rows: int):
    """fp64 oracle fwd+bwd on a bounded row sample of the workload (samples/s is
    batch-invariant: all three GEMMs are linear in the row count)."""
    import oracle  # test infrastructure: allowed in the cpu_baseline / reference legs only
    X = syn.gen_features((0, rows), cfg.D, seed, cfg.dtype)
    y = syn.gen_labels((0, rows), cfg.C, seed).numpy()
    W = syn.gen_weight((0, cfg.C), cfg.D, seed, "init", cfg.dtype)
    Xd = X.double().numpy()
    Wd = W.double().numpy()
    n, t0 = 0, time.perf_counter()
    while True:
        oracle.forward_backward(Xd, Wd, y)
        n += 1
        el = time.perf_counter() - t0
        if el >= min_seconds:
            break
    return n * rows / el, n, el


def host_cores():
    return len(os.sched_getaffinity(0))


_BLAS_LIMIT = None


def oracle_threads() -> int:
    """Let the oracle's BLAS use every host core (torchrun exports OMP_NUM_THREADS=1 to its
    workers) and return the thread count it actually runs with."""
    global _BLAS_LIMIT
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        _BLAS_LIMIT = threadpool_limits(limits=host_cores(), user_api="blas")
        n = [p.get("num_threads", 1) for p in threadpool_info() if p.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return int(os.environ.get("OMP_NUM_THREADS", host_cores()))


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=list(syn.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of one CUDA graph per step")
    ap.add_argument("--no-autograd", action="store_true", help="skip the autograd-path timing leg")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torch.distributed.run (one rank per GPU)")
    cfg = syn.CONFIGS[args.config]
    seed = syn.config_seed(args.config, world)

    if args.impl == "reference":
        return run_reference(args, cfg, seed, world, rank)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    group = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    import paper_2011_09208_b200 as whale
    from paper_2011_09208_b200 import _lib
    _lib.lib()

    dtype = syn.torch_dtype(cfg.dtype)
    op = whale.SplitFCSoftmaxCE(cfg.C, cfg.D, cfg.B, capacity=capacity_for(cfg, world), dtype=dtype, group=group,
                                device=dev)
    C_r, o_r = op.C_r, op.o_r
    X = syn.gen_features((rank * cfg.B, (rank + 1) * cfg.B), cfg.D, seed, cfg.dtype, device=dev)
    y = syn.gen_labels((rank * cfg.B, (rank + 1) * cfg.B), cfg.C, seed, device=dev).to(torch.int32)
    W = syn.gen_weight((o_r, o_r + C_r), cfg.D, seed, "init", cfg.dtype, device=dev)
    dx = torch.empty(cfg.B, cfg.D, dtype=dtype, device=dev)
    dw = torch.empty(C_r, cfg.D, dtype=torch.float32, device=dev)
    es = 2 if cfg.dtype == "bf16" else 4
    w_bytes = C_r * cfg.D * es
    flush_l2 = w_bytes < 2 * L2_BYTES
    flush_bufs = None
    if flush_l2:
        flush_bufs = (torch.empty(64 * 2 ** 20, dtype=torch.float32, device=dev),
                      torch.ones(64 * 2 ** 20, dtype=torch.float32, device=dev))

    def flush():
        # write 256 MiB (> L2), then read another 256 MiB: the read evicts the written dirty
        # lines too, so their write-back happens here and not inside the next timed step
        flush_bufs[0].zero_()
        flush_bufs[1].sum()

    def step():
        op.forward(X, y, W)
        op.backward(W, dx, dw)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier(device_ids=[local_rank])

    for _ in range(args.warmup):
        step()
    op.check()
    torch.cuda.synchronize()
    # one CUDA graph per step (the library keeps its step epoch on the device, so replays
    # are valid collective steps); falls back to eager launches with --no-graph
    run = step
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
        op.check()
        run = graph.replay

    # ---------------- timed region (device time, CUDA events on the launching stream)
    clocks = ClockSampler(local_rank)
    s = torch.cuda.current_stream()
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    if flush_l2:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for a, b in evs:
            flush()  # > L2: evicts the previous step's working set (outside the events)
            # N > 1: the step's exchanges couple the ranks, so a rank whose flush ends first
            # would count its peers' flush as step time: align the ranks on the device first
            op.device_barrier()
            a.record(s)
            run()
            b.record(s)
        torch.cuda.synchronize()
        total_ms = sum(a.elapsed_time(b) for a, b in evs)
    else:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(args.steps):
            run()
        b.record(s)
        torch.cuda.synchronize()
        total_ms = a.elapsed_time(b)
    barrier()
    clk = clocks.stop()
    op.check()
    t_max = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    total_ms = float(t_max.item())
    ms_per_step = total_ms / args.steps
    Bt = cfg.B * world
    value = Bt * args.steps / (total_ms / 1e3)

    # ---------------- per-kernel timing pass (events around each library launch)
    op.profile(True)
    for _ in range(args.steps):
        if flush_l2:
            flush()
        step()
    torch.cuda.synchronize()
    kern = op.profile_read()
    op.profile(False)

    # ---------------- end-to-end through the public API with host buffers
    # Every step copies its inputs from pinned host memory and reads its loss back.  The copies
    # run on a side stream, double-buffered: step i+1's inputs travel while step i computes,
    # and step i's loss is read back while its backward runs (one H2D + one D2H per step, all
    # inside the timed region; a graph replay = 2 steps, joined at the end).
    Xh = X.cpu().pin_memory()
    yh = y.cpu().pin_memory()
    loss_h = torch.empty(2, dtype=torch.float32).pin_memory()
    Xd_e = [torch.empty_like(X) for _ in range(2)]
    yd_e = [torch.empty_like(y) for _ in range(2)]
    cs = torch.cuda.Stream(device=dev)

    def e2e_two_steps():
        main = torch.cuda.current_stream(dev)
        ev_start = torch.cuda.Event()
        ev_start.record(main)
        cs.wait_event(ev_start)
        with torch.cuda.stream(cs):  # inputs of step 1 while step 0 runs
            Xd_e[1].copy_(Xh, non_blocking=True)
            yd_e[1].copy_(yh, non_blocking=True)
        ev_c1 = torch.cuda.Event()
        ev_c1.record(cs)
        loss = op.forward(Xd_e[0], yd_e[0], W)
        ev_f0 = torch.cuda.Event()
        ev_f0.record(main)
        cs.wait_event(ev_f0)
        with torch.cuda.stream(cs):  # step 0's loss while its backward runs
            loss_h[0].copy_(loss, non_blocking=True)
        ev_d0 = torch.cuda.Event()
        ev_d0.record(cs)
        op.backward(W, dx, dw)
        ev_b0 = torch.cuda.Event()
        ev_b0.record(main)
        main.wait_event(ev_c1)
        main.wait_event(ev_d0)
        loss = op.forward(Xd_e[1], yd_e[1], W)
        ev_f1 = torch.cuda.Event()
        ev_f1.record(main)
        cs.wait_event(ev_b0)
        with torch.cuda.stream(cs):  # inputs of the next replay's step 0 (buffer 0 is free now)
            Xd_e[0].copy_(Xh, non_blocking=True)
            yd_e[0].copy_(yh, non_blocking=True)
        cs.wait_event(ev_f1)
        with torch.cuda.stream(cs):
            loss_h[1].copy_(loss, non_blocking=True)
        op.backward(W, dx, dw)
        main.wait_stream(cs)

    Xd_e[0].copy_(Xh)
    yd_e[0].copy_(yh)
    for _ in range(3):
        e2e_two_steps()
    torch.cuda.synchronize()
    run_e2e = e2e_two_steps
    if not args.no_graph:
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            e2e_two_steps()
        g2.replay()
        torch.cuda.synchronize()
        run_e2e = g2.replay
    e2e_steps = 2 * ((args.steps + 1) // 2)
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(e2e_steps // 2):
        run_e2e()
    b.record(s)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = Bt * e2e_steps / (float(e2e_ms.item()) / 1e3)

    # ---------------- the user-facing autograd step (N = 1): bf16 W leaf, grad_output applied
    # in-kernel, W.grad written in bf16 by the backward (no eager pass), eager launches, timed
    # against the same eager raw C-ABI step
    autograd = None
    if world == 1 and cfg.dtype == "bf16" and not args.no_autograd:
        op16 = whale.SplitFCSoftmaxCE(cfg.C, cfg.D, cfg.B, dtype=dtype, device=dev, dw_dtype=torch.bfloat16)
        xl = X.clone().requires_grad_(True)
        wl = W.clone().requires_grad_(True)

        def ag_step():
            xl.grad = None
            wl.grad = None
            whale.split_fc_softmax_ce(xl, wl, y, op16).backward()

        def ev_time(fn, n):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record()
            for _ in range(n):
                if flush_l2:
                    flush()
                fn()
            eb.record()
            torch.cuda.synchronize()
            return ea.elapsed_time(eb) / n

        raw_ms = ev_time(step, args.steps)
        ag_ms = ev_time(ag_step, args.steps)
        op16.check()
        op16.close()
        autograd = {"ms_per_step": ag_ms, "raw_eager_ms_per_step": raw_ms, "ratio": ag_ms / raw_ms,
                    "what": "split_fc_softmax_ce(x, W_bf16, y).backward() vs op.forward+op.backward (fp32 dW), "
                            "both eager"}

    # ---------------- roofline of the dominant kernel
    peaks = load_peaks()
    cfgj = op.config()
    roof, kernels = roofline(kern, cfgj, cfg, es, peaks)

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = oracle_threads()
        sps, n, el = time_oracle(cfg, seed, args.cpu_seconds, rows=min(cfg.B * world, 64))
        cpu = {"value": sps, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{n} x fp64 numpy fwd+bwd of {min(cfg.B * world, 64)} rows of {args.config} "
                         f"(D={cfg.D}, C={cfg.C}) in {el:.1f} s"}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic (seeded; ReLU(N(0,1)) features, N(0,1/D) weights, uniform labels)",
        "config": {
            "workload": workload_desc(args.config, cfg, world), "D": cfg.D, "C": cfg.C, "B_per_gpu": cfg.B,
            "global_batch": Bt, "C_shard_rank0": cfgj["C_r"], "parallelism": f"dp{world}-backbone/mp{world}-fc",
            "l2": ("flushed between timed steps outside the step events (256 MiB write + 256 MiB read, so no "
                   "dirty flush lines are written back inside a step)" if flush_l2
                   else f"inputs larger than L2 (W shard {w_bytes / 2 ** 20:.0f} MiB > 2x126 MiB)"),
            "tiles": {k: cfgj[k] for k in ("fwd", "dw", "dx")},
            "launch": "eager" if args.no_graph else "CUDA graph per step",
        },
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": X.numel() * X.element_size() + y.numel() * 4,
                "d2h_bytes_per_step": 4,
                "pipeline": "side-stream copies, double-buffered: step i+1's inputs H2D and step i's loss D2H "
                            "overlap compute; CUDA graph of 2 steps (value: graph of 1 step)"},
        "gpu_launches": op.launches_per_step() * args.steps,
        "roofline": roof,
        "kernels": kernels,
        "cpu_baseline": cpu,
        "autograd": autograd,
        "peaks_source": peaks["source"],
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def kernel_work(name, cfgj, cfg, es):
    """Algorithmic bytes and FLOPs per launch of each library kernel."""
    Bt, D, Cr = cfgj["Bt"], cfgj["D"], cfgj["C_r"]
    B = cfgj["B"]
    T = cfgj["fwd"]["n_blocks"]
    S = cfgj["dx"]["splits"]
    world = cfgj["world"]
    f1 = cfgj.get("f1", 0) == 1
    ncl = cfgj.get("f1_clusters", 0)
    if f1 and name == "logits_gemm":  # F1: read W_r once, X; write P~, tile stats, U partials
        return (Cr * D * es + Bt * D * es + Bt * Cr * es + 3 * Bt * T * 4 + ncl * Bt * D * 4 + ncl * Bt * 4,
                4 * Bt * Cr * D)
    if f1 and name == "bwd_gemm":     # F1: dW tiles + the dX combine units (U partials -> dX)
        bw, fw = kernel_work("dw_gemm", cfgj, cfg, es)
        return bw + ncl * Bt * D * 4 + Bt * D * es + Bt * D * (es if world == 1 else 4), fw
    if f1 and name == "dx_gemm":      # F1 combine: read U partials + label rows of W, write dX
        return ncl * Bt * D * 4 + Bt * D * es + Bt * D * (es if world == 1 else 4), 0
    if name == "logits_gemm":   # read W_r, X; write P~ and tile stats
        return Cr * D * es + Bt * D * es + Bt * Cr * es + 2 * Bt * T * 4, 2 * Bt * Cr * D
    if name == "dw_gemm":       # read G, X; write dW fp32
        return Bt * Cr * es + Bt * D * es + Cr * D * 4, 2 * Bt * Cr * D
    if name == "dx_gemm":       # read G, W_r; write split-K partials
        return Bt * Cr * es + Cr * D * es + S * Bt * D * 4, 2 * Bt * Cr * D
    if name == "bwd_gemm":      # fused dX (read G, W_r; partials) + dW (read G, X; write dW)
        bx, fx = kernel_work("dx_gemm", cfgj, cfg, es)
        bw, fw = kernel_work("dw_gemm", cfgj, cfg, es)
        return bx + bw, fx + fw
    if name == "softmax_grad":  # read + write P~/G in place, read tile maxima
        return 2 * Bt * Cr * es + Bt * T * 4, 0
    if name == "stats_combine":  # tile partials (+ true maxima for F1) + the fused in-place G rewrite
        return (3 if f1 else 2) * Bt * T * 4 + Bt * 16 * world + 2 * Bt * Cr * es, 0
    if name == "bridge_gather":
        return B * D * es * (1 + world), 0
    if name == "dx_rs_push":
        return S * Bt * D * 4 + Bt * D * (4 if world > 1 else es), 0
    if name == "dx_rs_reduce":
        return world * B * D * 4 + B * D * es, 0
    return 0, 0


def roofline(kern, cfgj, cfg, es, peaks):
    hbm = float(peaks["hbm_gbs"])
    # kernels are timed per launch (CUDA events around each launch, sub-second loop): the
    # burst bf16 figure is the matching denominator (B200_PROFILING.md, "Peaks")
    tf = float(peaks["bf16_tflops"])
    if es == 4:
        tf = tf / 2.0  # tf32 dense = half of bf16 (guide's nominal ratio 1.1 : 2.25)
    kernels = {}
    for name, v in kern.items():
        if v["launches"] == 0:
            continue
        avg_ms = v["total_ms"] / v["launches"]
        by, fl = kernel_work(name, cfgj, cfg, es)
        kernels[name] = {"avg_us": avg_ms * 1e3, "launches": v["launches"], "bytes": by, "flops": fl,
                         "GBps": by / (avg_ms / 1e3) / 1e9 if avg_ms > 0 else None,
                         "TFLOPs": fl / (avg_ms / 1e3) / 1e12 if avg_ms > 0 else None}
    if not kernels:
        return None, kernels
    top = max(kernels, key=lambda k: kernels[k]["avg_us"] * kernels[k]["launches"])
    k = kernels[top]
    t_mem = k["bytes"] / (hbm * 1e9)
    t_tc = k["flops"] / (tf * 1e12) if k["flops"] else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(cfgj and f"{cfg.name}/N{cfgj['world']}", {}).get(top)
        except Exception:
            traffic = None
    if t_tc > t_mem:
        roof = {"kernel": top, "bound": "tensor", "achieved": k["TFLOPs"], "peak": tf, "unit": "TFLOP/s",
                "frac": k["TFLOPs"] / tf, "traffic": traffic, "peak_kind": f"bf16 burst ({peaks['source']})"}
    else:
        roof = {"kernel": top, "bound": "hbm", "achieved": k["GBps"], "peak": hbm, "unit": "GB/s",
                "frac": k["GBps"] / hbm, "traffic": traffic, "peak_kind": f"HBM copy ({peaks['source']})"}
    roof["share_of_step"] = (kernels[top]["avg_us"] * kernels[top]["launches"]) / max(
        1e-9, sum(v["avg_us"] * v["launches"] for v in kernels.values()))
    return roof, kernels


def run_reference(args, cfg, seed, world, rank):
    """Reference arm: the fp64 CPU oracle as it stands, on the host cores, bounded sample per step."""
    if rank != 0:
        return
    rows = min(cfg.B * world, 32)  # same sample as the cpu_baseline leg
    threads = oracle_threads()
    import oracle
    X = syn.gen_features((0, rows), cfg.D, seed, cfg.dtype).double().numpy()
    y = syn.gen_labels((0, rows), cfg.C, seed).numpy()
    W = syn.gen_weight((0, cfg.C), cfg.D, seed, "init", cfg.dtype).double().numpy()
    for _ in range(args.warmup):
        oracle.forward_backward(X, W, y)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.forward_backward(X, W, y)
    el = time.perf_counter() - t0
    value = rows * args.steps / el
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
        "config": {"workload": workload_desc(args.config, cfg, world), "D": cfg.D, "C": cfg.C,
                   "B_per_gpu": cfg.B, "global_batch": cfg.B * world},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"each step: fp64 numpy fwd+bwd of {rows} rows of {args.config} (D={cfg.D}, C={cfg.C})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
