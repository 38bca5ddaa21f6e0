"""World-size-2 `gloo` tests (CPU) of the N > 1 host logic.

What runs here without a GPU:
* every rank computes the class plan through the C-ABI and the plans agree bit-for-bit;
* every rank computes the same symmetric-buffer size (the buffer must be symmetric);
* the exchange protocol of the CUDA path, restated on the host with gloo collectives:
  per-shard statistics (m_r, s_r, z_y,r) -> all-gather of the records -> rank-ordered
  combine -> loss identical on every rank; the reduce-scatter of dX partials by row owner
  (row // B) -- checked against the unsharded fp64 oracle;
* NEXT-3 uneven per-rank batches: descriptor sizes agree, gather-v by padding, row owners from
  the prefix offsets, the dX reduce-scatter against the oracle.
The GPU kernels implement the same protocol over NVLink (tests/test_multigpu.py).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2011_09208_b200 import _lib

        out = {}
        # ---- plan agreement (C-ABI, host-only)
        C, D, B = 1001, 24, 5
        counts, offs = _lib.whale_splitfc_plan(C, world, [3, 2])
        allp = [None] * world
        dist.all_gather_object(allp, (counts, offs))
        out["plans_equal"] = all(p == allp[0] for p in allp)
        # ---- symmetric buffer sizes agree across ranks
        d, _k = _lib.make_desc(rank, world, B, D, C, counts, offs)
        symm, local = _lib.whale_splitfc_workspace_size(d)
        alls = [None] * world
        dist.all_gather_object(alls, symm)
        out["symm_equal"] = all(s == alls[0] for s in alls) and symm > 0
        # ---- exchange protocol on the host (fp64)
        rng = np.random.default_rng(77)
        Bt = B * world
        X = np.maximum(rng.standard_normal((Bt, D)), 0)
        W = rng.standard_normal((C, D)) * 4 / np.sqrt(D)
        y = rng.integers(0, C, Bt)
        o, c = offs[rank], counts[rank]
        Xr = X[rank * B:(rank + 1) * B]
        # bridge: all-gather X_r (rank order)
        xs = [torch.zeros(B, D, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(xs, torch.from_numpy(Xr))
        Xg = torch.cat(xs).numpy()
        Zr = Xg @ W[o:o + c].T
        m_r = Zr.max(1)
        s_r = np.exp(Zr - m_r[:, None]).sum(1)
        own = (y >= o) & (y < o + c)
        zy_r = np.where(own, Zr[np.arange(Bt), np.clip(y - o, 0, c - 1)], 0.0)
        rec = torch.from_numpy(np.stack([m_r, s_r, zy_r], 1))
        recs = [torch.zeros_like(rec) for _ in range(world)]
        dist.all_gather(recs, rec)
        R = torch.stack(recs).numpy()             # [world, Bt, 3], rank order
        m = R[:, :, 0].max(0)
        s = sum(R[p, :, 1] * np.exp(R[p, :, 0] - m) for p in range(world))
        zy = sum(R[p, :, 2] for p in range(world))
        lse = m + np.log(s)
        loss = float(np.mean(lse - zy))
        losses = [None] * world
        dist.all_gather_object(losses, loss)
        out["loss_equal"] = all(v == losses[0] for v in losses)
        G = np.exp(Zr - lse[:, None])
        rows = np.nonzero(own)[0]
        G[rows, y[rows] - o] -= 1.0
        G /= Bt
        dW_r = G.T @ Xg
        dX_part = G @ W[o:o + c]                  # [Bt, D] partial of this shard
        # reduce-scatter by row owner: rank r receives rows r*B..(r+1)*B summed in rank order
        chunks = [torch.from_numpy(dX_part[p * B:(p + 1) * B].copy()) for p in range(world)]
        gathered = [[torch.zeros(B, D, dtype=torch.float64) for _ in range(world)] for _ in range(world)]
        for p in range(world):
            dist.all_gather(gathered[p], chunks[p])
        dX_r = sum(gathered[rank][src] for src in range(world)).numpy()
        f = oracle.forward_backward(X, W, y)
        out["loss_ok"] = abs(loss - f["loss"]) <= 1e-12 * abs(f["loss"])
        out["dW_ok"] = np.allclose(dW_r, f["dW"][o:o + c], rtol=1e-10, atol=1e-15)
        out["dX_ok"] = np.allclose(dX_r, f["dX"][rank * B:(rank + 1) * B], rtol=1e-10, atol=1e-15)
        # ---- NEXT-3: uneven per-rank batch (proportional split of the global batch)
        bc, _ = _lib.whale_splitfc_plan(7, world, [2, 1])    # [5, 2]
        offs_b = np.concatenate([[0], np.cumsum(bc)])
        d2, _k2 = _lib.make_desc(rank, world, bc[rank], D, C, counts, offs, batch_counts=bc)
        symm2, _ = _lib.whale_splitfc_workspace_size(d2)
        alls2 = [None] * world
        dist.all_gather_object(alls2, symm2)
        out["uneven_symm_equal"] = all(v == alls2[0] for v in alls2)
        Bt2 = int(offs_b[-1])
        X2 = np.maximum(rng.standard_normal((Bt2, D)), 0)
        y2 = rng.integers(0, C, Bt2)
        mine = torch.from_numpy(X2[offs_b[rank]:offs_b[rank + 1]].copy())
        bmax = int(max(bc))
        padded = torch.zeros(bmax, D, dtype=torch.float64)
        padded[:bc[rank]] = mine
        xs2 = [torch.zeros(bmax, D, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(xs2, padded)                         # gather-v via padding to B_max
        Xg2 = torch.cat([xs2[p][:bc[p]] for p in range(world)]).numpy()
        out["uneven_gather_ok"] = np.array_equal(Xg2, X2)
        # each shard's dX partial, reduce-scattered to the row owner found from the prefix offsets
        f2 = oracle.forward_backward(X2, W, y2)
        G2 = f2["G"][:, o:o + c]
        part2 = G2 @ W[o:o + c]
        owner = np.searchsorted(offs_b, np.arange(Bt2), side="right") - 1
        mine_rows = np.nonzero(owner == rank)[0]
        send = [torch.from_numpy(np.ascontiguousarray(part2[owner == p])) for p in range(world)]
        recv = [[torch.zeros(int(bc[p]), D, dtype=torch.float64) for _ in range(world)] for p in range(world)]
        for p in range(world):
            dist.all_gather(recv[p], send[p])
        dX2 = sum(recv[rank][src] for src in range(world)).numpy()
        out["uneven_dX_ok"] = np.allclose(dX2, f2["dX"][mine_rows], rtol=1e-10, atol=1e-15)
        q.put((rank, out))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, {"error": repr(e)}))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    for r in range(WORLD):
        assert "error" not in res[r], res[r]
        assert all(res[r].values()), (r, res[r])
