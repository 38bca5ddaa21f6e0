"""Run K fwd+bwd steps of a config at N=1 (for ncu / sanitizer captures)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import synthetic as syn  # noqa: E402
from paper_2011_09208_b200 import SplitFCSoftmaxCE  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=3)
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
for _ in range(args.steps):
    op.forward(X, y, W)
    op.backward(W, dx, dw)
op.check()
torch.cuda.synchronize()
print("ok", op.config()["dw"])
