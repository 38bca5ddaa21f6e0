"""Per-kernel CUDA-event times (library profiling hooks) for one config at N=1."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
import synthetic as syn  # noqa: E402
from paper_2011_09208_b200 import SplitFCSoftmaxCE  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--B", type=int, default=0)
ap.add_argument("--C", type=int, default=0)
args = ap.parse_args()
cfg = syn.CONFIGS[args.config]
B = args.B or cfg.B
C = args.C or cfg.C
seed = syn.config_seed(args.config, 1)
dt = syn.torch_dtype(cfg.dtype)
X = syn.gen_features((0, B), cfg.D, seed, cfg.dtype, device="cuda")
y = syn.gen_labels((0, B), C, seed, device="cuda").to(torch.int32)
W = syn.gen_weight((0, C), cfg.D, seed, "init", cfg.dtype, device="cuda")
op = SplitFCSoftmaxCE(C, cfg.D, B, dtype=dt)
dx = torch.empty(B, cfg.D, dtype=dt, device="cuda")
dw = torch.empty(C, cfg.D, dtype=torch.float32, device="cuda")
for _ in range(3):
    op.forward(X, y, W)
    op.backward(W, dx, dw)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(args.steps):
    op.forward(X, y, W)
    op.backward(W, dx, dw)
b.record()
torch.cuda.synchronize()
step_us = a.elapsed_time(b) / args.steps * 1e3
op.profile(True)
for _ in range(args.steps):
    op.forward(X, y, W)
    op.backward(W, dx, dw)
k = op.profile_read()
op.check()
out = {"config": args.config, "B": B, "C": C, "cfg": {k: op.config()[k] for k in ("fwd", "dw", "dx")}, "step_us": round(step_us, 1),
       "kernels_us": {n: round(v["total_ms"] / v["launches"] * 1e3, 1) for n, v in k.items() if v["launches"]}}
print(json.dumps(out))
