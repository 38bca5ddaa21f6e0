"""Multi-GPU parity of the split-FC path vs the fp64 oracle (run with torchrun, one rank per GPU).

Every rank builds the same seeded global batch and full weight on the CPU, takes its DP rows
and its class shard (plan from the C-ABI), runs forward/backward through the library and
checks its own dX_r rows and dW_r shard against the unsharded oracle; the loss must be
bit-identical on all ranks.  Prints one JSON line per case on rank 0; exit code 1 on failure.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synthetic as syn  # noqa: E402
from paper_2011_09208_b200 import SplitFCSoftmaxCE  # noqa: E402
from paper_2011_09208_b200._lib import whale_splitfc_plan as plan  # noqa: E402


def fro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run_case(rank, world, dev, B, D, C, capacity=None, regime="init", dtype="bf16", seed=1, steps=3, bias=False,
             batch=None):
    """`steps` forward+backward steps with NEW seeded (X, y) every step (W stays), every step
    checked against the oracle (a stale gathered row or label would show up here)."""
    bc = batch if batch is not None else [B] * world  # per-rank DP batch (NEXT-3 when uneven)
    Bt = sum(bc)
    r0 = sum(bc[:rank])
    B = bc[rank]
    W = syn.gen_weight((0, C), D, seed, regime, dtype)
    bfull = syn.gen_bias((0, C), seed, 2.0, dtype) if bias else None
    op = SplitFCSoftmaxCE(C, D, B, capacity=capacity, dtype=syn.torch_dtype(dtype), group=dist.group.WORLD, device=dev,
                          batch_counts=batch)
    o, c = op.o_r, op.C_r
    wr = W[o:o + c].to(dev).contiguous()
    br = bfull[o:o + c].to(dev).contiguous() if bias else None
    ok = True
    res = {}
    for step in range(steps):  # repeated steps exercise the device epoch / flag protocol
        sd = seed + 7919 * (step + 1)
        X = syn.gen_features((0, Bt), D, sd, dtype)
        y = syn.gen_labels((0, Bt), C, sd)
        xr = X[r0:r0 + B].to(dev)
        yr = y[r0:r0 + B].to(dev)
        loss = op.forward(xr, yr, wr, row_loss=True, bias=br, predictions=bias).clone()
        out = op.backward(wr, bias_grad=bias)
        dx, dw = out[0], out[1]
        op.check()
        torch.cuda.synchronize(dev)
        f = oracle.forward_backward(X, W, y.numpy(), bfull)
        losses = [torch.zeros((), device=dev) for _ in range(world)]
        dist.all_gather(losses, loss)
        bit_equal = all(torch.equal(l, losses[0]) for l in losses)
        res = {
            "B": B, "batch": bc, "D": D, "C": C, "world": world, "capacity": capacity, "regime": regime, "dtype": dtype,
            "C_r": c, "step": step, "nvls": op.config().get("nvls", 0), "loss": float(loss), "loss_ref": float(f["loss"]),
            "loss_rel": abs(float(loss) - f["loss"]) / abs(f["loss"]),
            "rowloss_rel": fro(op.row_loss.cpu(), f["row_loss"][r0:r0 + B]),
            "dx_rel": fro(dx.float().cpu(), f["dX"][r0:r0 + B]) if B else 0.0,
            "dw_rel": fro(dw.cpu(), f["dW"][o:o + c]),
            "loss_bit_equal": bool(bit_equal),
        }
        ok_s = res["loss_rel"] <= 1e-3 and res["dx_rel"] <= 1e-2 and res["dw_rel"] <= 1e-2 and bit_equal
        if bias:
            rows = slice(r0, r0 + B)
            Zs = np.sort(f["Z"][rows], axis=1)
            clear = (Zs[:, -1] - Zs[:, -2]) > 1e-3
            pred = op.pred.cpu().numpy()
            res["db_rel"] = fro(out[2].cpu(), f["db"][o:o + c])
            res["pred_ok"] = bool(np.array_equal(pred[clear], f["pred"][rows][clear]))
            res["prob_rel"] = float(np.max(np.abs(op.prob.cpu().numpy() - f["prob"][rows]) / f["prob"][rows])) if B else 0.0
            ok_s = ok_s and res["db_rel"] <= 1e-2 and res["pred_ok"] and res["prob_rel"] <= 1e-3
        ok = ok and ok_s
    # run-to-run reproducibility of the reduce-scattered dX and of dW: the last step again
    dx_last, dw_last = dx.clone(), dw.clone()
    op.forward(xr, yr, wr, bias=br, predictions=bias)
    out = op.backward(wr, bias_grad=bias)
    op.check()
    res["dx_repeat_bitwise"] = bool(torch.equal(out[0], dx_last))
    res["dw_repeat_bitwise"] = bool(torch.equal(out[1], dw_last))
    res["nvls_rs"] = op.config().get("nvls_rs", 0)
    ok = ok and res["dx_repeat_bitwise"] and res["dw_repeat_bitwise"]
    res["ok"] = ok
    allres = [None] * world
    dist.all_gather_object(allres, res)
    op.close()
    return allres


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cases = [
        dict(B=8, D=64, C=1000, dtype="f32"),                       # tiny-like (fp32 operands)
        dict(B=8, D=64, C=1000),
        dict(B=40, D=192, C=3001, regime="peaked"),
        dict(B=32, D=256, C=5000, capacity=[2] + [1] * (world - 1)),  # uneven (c3-like)
        dict(B=64, D=520, C=20000),
        dict(B=32, D=2048, C=100_000),                              # c2 shape
        dict(B=24, D=256, C=7001, regime="peaked", bias=True),      # NEXT-4: bias, db, predictions
        # NEXT-3: uneven per-rank batch from the proportional plan (2:1:...:1 capacity)
        dict(B=None, D=512, C=9000, batch=plan(12 * world, world, [2] + [1] * (world - 1))[0]),
        dict(B=None, D=256, C=7001, regime="peaked", bias=True, batch=plan(10 * world + 3, world, list(range(1, world + 1)))[0]),
        dict(B=None, D=256, C=3000, batch=[40] * (world - 1) + [0]),  # a rank with no rows
        dict(B=None, D=2048, C=100_000, batch=plan(32 * world, world, [2] + [1] * (world - 1))[0]),
        # F1 path (fused forward + dX; B_tot <= 32, D % 256 == 0): total batch 32
        dict(B=32 // world, D=2048, C=100_000),
        dict(B=None, D=1024, C=30_011, regime="peaked", bias=True, batch=plan(32, world, list(range(1, world + 1)))[0]),
    ]
    ok = True
    for cs in cases:
        allres = run_case(rank, world, dev, **cs)
        if rank == 0:
            for r in allres:
                print(json.dumps(r), flush=True)
        ok = ok and all(r["ok"] for r in allres)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
