"""Autograd step vs the raw C-ABI step at c2, N = 1 (eager launches, CUDA events).

  python scripts/autograd_step.py [--steps 30] [--warmup 5]

raw_f32  : op.forward + op.backward into preallocated fp32 dW (the bench's step, eager)
raw_bf16 : the same with an op built with dw_dtype=bf16
autograd : loss = split_fc_softmax_ce(x, W, y, op_bf16); loss.backward()  (W bf16 leaf,
           grad_output applied in-kernel, W.grad written in bf16: no eager pass)
Prints one JSON line.  W_r (391 MiB) exceeds L2, so no flush is needed between steps.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as syn  # noqa: E402
import paper_2011_09208_b200 as whale  # noqa: E402


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    args = ap.parse_args()
    cfg = syn.CONFIGS[args.config]
    seed = syn.config_seed(args.config, 1)
    B, D, C = cfg.B, cfg.D, cfg.C
    X = syn.gen_features((0, B), D, seed, "bf16", device="cuda")
    y = syn.gen_labels((0, B), C, seed, device="cuda").to(torch.int32)
    W = syn.gen_weight((0, C), D, seed, "init", "bf16", device="cuda")
    op32 = whale.SplitFCSoftmaxCE(C, D, B)
    op16 = whale.SplitFCSoftmaxCE(C, D, B, dw_dtype=torch.bfloat16)
    dx = torch.empty(B, D, dtype=torch.bfloat16, device="cuda")
    dw32 = torch.empty(C, D, dtype=torch.float32, device="cuda")
    dw16 = torch.empty(C, D, dtype=torch.bfloat16, device="cuda")

    def raw32():
        op32.forward(X, y, W)
        op32.backward(W, dx, dw32)

    def raw16():
        op16.forward(X, y, W)
        op16.backward(W, dx, dw16)

    xl = X.clone().requires_grad_(True)
    wl = W.clone().requires_grad_(True)

    def autograd():
        xl.grad = None
        wl.grad = None
        loss = whale.split_fc_softmax_ce(xl, wl, y, op16)
        loss.backward()

    r = {"config": args.config, "B": B, "D": D, "C": C, "steps": args.steps}
    r["raw_f32_ms"] = timed(raw32, args.steps, args.warmup)
    r["raw_bf16_ms"] = timed(raw16, args.steps, args.warmup)
    r["autograd_ms"] = timed(autograd, args.steps, args.warmup)
    op16.check()
    op32.check()
    r["autograd_over_raw_bf16"] = r["autograd_ms"] / r["raw_bf16_ms"]
    r["autograd_over_raw_f32"] = r["autograd_ms"] / r["raw_f32_ms"]
    print(json.dumps(r))


if __name__ == "__main__":
    main()
