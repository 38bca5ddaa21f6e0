"""Debug driver for the single-GPU emulated-rank harness: one case per process.

  python scripts/emu_debug.py WORLD B D C [steps] [timeout_ms] [f1|plain]

Runs `steps` steps with new inputs each, synchronises, calls check() on every rank and
prints per-rank status, loss and relative errors against the fp64 oracle (test-only code).
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synthetic as syn  # noqa: E402
import paper_2011_09208_b200 as whale  # noqa: E402


def fro(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    world, B, D, C = (int(v) for v in sys.argv[1:5])
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    tmo = int(sys.argv[6]) if len(sys.argv) > 6 else 3000
    ops, streams = whale.emulated_ranks(C, D, world, local_batch=B, timeout_ms=tmo)
    dev = ops[0].device
    print("config rank0:", {k: ops[0].config()[k] for k in ("f1", "sms", "Bt", "C_r")}, flush=True)
    W = syn.gen_weight((0, C), D, 5, "peaked", "bf16")
    wr = [W[o.o_r:o.o_r + o.C_r].to(dev).contiguous() for o in ops]
    for step in range(steps):
        X = syn.gen_features((0, world * B), D, 10 + step, "bf16")
        y = syn.gen_labels((0, world * B), C, 10 + step)
        keep, outs = [], []
        t0 = time.perf_counter()
        for r, o in enumerate(ops):
            with torch.cuda.stream(streams[r]):
                xr, yr = X[r * B:(r + 1) * B].to(dev), y[r * B:(r + 1) * B].to(dev)
                keep.append((xr, yr))
                o.forward(xr, yr, wr[r])
        for r, o in enumerate(ops):
            with torch.cuda.stream(streams[r]):
                outs.append(o.backward(wr[r]))
        torch.cuda.synchronize(dev)
        el = time.perf_counter() - t0
        f = oracle.forward_backward(X, W, y.numpy())
        for r, o in enumerate(ops):
            try:
                with torch.cuda.stream(streams[r]):
                    o.check()
                st = "ok"
            except whale.WhaleError as e:
                st = str(e)
            print(f"step {step} rank {r} {el * 1e3:.1f} ms: {st} loss {float(o.loss):.6f} (oracle {f['loss']:.6f}) "
                  f"dX {fro(outs[r][0].float().cpu(), f['dX'][r * B:(r + 1) * B]):.2e} "
                  f"dW {fro(outs[r][1].cpu(), f['dW'][o.o_r:o.o_r + o.C_r]):.2e}", flush=True)
    for o in ops:
        o.close()


if __name__ == "__main__":
    main()
