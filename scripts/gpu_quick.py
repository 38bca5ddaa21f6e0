"""Quick single-GPU parity sweep vs the fp64 oracle (development aid; tests/ hold the gates)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import synthetic as syn  # noqa: E402
from paper_2011_09208_b200 import SplitFCSoftmaxCE  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run(B, D, C, dtype="bf16", regime="init", seed=1):
    X = syn.gen_features((0, B), D, seed, dtype)
    W = syn.gen_weight((0, C), D, seed, regime, dtype)
    y = syn.gen_labels((0, B), C, seed)
    op = SplitFCSoftmaxCE(C, D, B, dtype=syn.torch_dtype(dtype))
    xd, wd, yd = X.cuda(), W.cuda(), y.cuda()
    t = time.time()
    loss = op.forward(xd, yd, wd, row_loss=True)
    dx, dw = op.backward(wd)
    op.check()
    torch.cuda.synchronize()
    f = oracle.forward_backward(X, W, y.numpy())
    r = {
        "shape": (B, D, C, dtype, regime),
        "loss": float(loss), "loss_ref": float(f["loss"]),
        "loss_rel": abs(float(loss) - f["loss"]) / abs(f["loss"]),
        "rowloss_rel": rel(op.row_loss.cpu(), f["row_loss"]),
        "dx_rel": rel(dx.float().cpu(), f["dX"]),
        "dw_rel": rel(dw.cpu(), f["dW"]),
        "cfg": {k: op.config()[k] for k in ("fwd", "dw", "dx")},
    }
    print(r, flush=True)
    op.close()
    return r


if __name__ == "__main__":
    torch.cuda.init()
    cases = [(128, 64, 256), (40, 192, 1000), (16, 64, 1000), (200, 520, 3001), (32, 2048, 100000)]
    for c in cases:
        try:
            run(*c)
        except Exception as e:  # keep sweeping
            print("FAIL", c, repr(e), flush=True)
    for c in [(16, 64, 1000)]:
        try:
            run(*c, dtype="f32")
        except Exception as e:
            print("FAIL f32", c, repr(e), flush=True)
    run(40, 192, 1000, regime="peaked")
