"""Multi-rank parity on ONE GPU: N emulated ranks (paper_2011_09208_b200.emulated_ranks).

The driver's GPU test box has one B200, so the multi-GPU protocol -- the bridge all-gather
of X_r, y_r (A2), the per-row statistics exchange of the split softmax
(A4, the "communication operator", PAPER.md:488 comment), the dX reduce-scatter back to the
DP owners (A8, the bridge backward) and the uneven per-rank batch of
the hardware-aware `replicate` (NEXT-3) -- is exercised here
with every rank's context on cuda:0.  The ranks' "symmetric buffers" are plain device
allocations that all contexts address directly, so the same exchange kernels issue the same
stores and flag protocol as over NVLink; each rank runs on its own stream with its
persistent grids capped to its share of the SMs.

Every case runs >= 3 steps with DIFFERENT seeded (X, y) per step (the weights stay), each
step checked against the fp64 oracle: loss (bit-identical on every rank), per-row loss, dX_r
of every rank, dW_r of every shard (and db_r / predictions with a bias).
"""
import numpy as np
import pytest
import torch

import oracle
import synthetic as syn

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-3
FRO_RTOL = 1e-2


def _fro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


@pytest.fixture(scope="module")
def whale():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2011_09208_b200 as w
    from paper_2011_09208_b200 import _lib
    _lib.lib()
    return w


def run_emulated(whale, world, D, C, B=None, batch=None, capacity=None, regime="init", dtype="bf16", bias=False,
                 steps=3, seed=1, expect_f1=None):
    bc = [int(b) for b in batch] if batch is not None else [B] * world
    Bt = sum(bc)
    offs = np.concatenate([[0], np.cumsum(bc)]).astype(int)
    tdt = syn.torch_dtype(dtype)
    ops, streams = whale.emulated_ranks(C, D, world, local_batch=B, batch_counts=batch, capacity=capacity,
                                        dtype=tdt)
    dev = ops[0].device
    W = syn.gen_weight((0, C), D, seed, regime, dtype)
    bfull = syn.gen_bias((0, C), seed, 2.0, dtype) if bias else None
    wr = [W[o.o_r:o.o_r + o.C_r].to(dev).contiguous() for o in ops]
    br = [bfull[o.o_r:o.o_r + o.C_r].to(dev).contiguous() if bias else None for o in ops]
    if expect_f1 is not None:
        assert all(o.config()["f1"] == int(expect_f1) for o in ops)
    try:
        for step in range(steps):
            sd = seed + 7919 * (step + 1)  # new features and labels every step
            X = syn.gen_features((0, Bt), D, sd, dtype)
            y = syn.gen_labels((0, Bt), C, sd)
            keep, outs = [], []
            for r, o in enumerate(ops):  # forward of every rank, each on its own stream
                with torch.cuda.stream(streams[r]):
                    xr = X[offs[r]:offs[r + 1]].to(dev)
                    yr = y[offs[r]:offs[r + 1]].to(dev)
                    keep.append((xr, yr))
                    o.forward(xr, yr, wr[r], row_loss=True, bias=br[r], predictions=bias)
            for r, o in enumerate(ops):  # then backward of every rank
                with torch.cuda.stream(streams[r]):
                    outs.append(o.backward(wr[r], bias_grad=bias))
            torch.cuda.synchronize(dev)
            for r, o in enumerate(ops):
                with torch.cuda.stream(streams[r]):
                    o.check()
            f = oracle.forward_backward(X, W, y.numpy(), bfull)
            losses = [o.loss.clone() for o in ops]
            tag = f"world={world} step={step} D={D} C={C} batch={bc} cap={capacity} {regime} {dtype} bias={bias}"
            assert all(torch.equal(l, losses[0]) for l in losses), (tag, [float(l) for l in losses])
            assert abs(float(losses[0]) - f["loss"]) <= LOSS_RTOL * abs(f["loss"]), (tag, float(losses[0]), f["loss"])
            for r, o in enumerate(ops):
                rows = slice(offs[r], offs[r + 1])
                cls = slice(o.o_r, o.o_r + o.C_r)
                if bc[r]:
                    np.testing.assert_allclose(o.row_loss.cpu().numpy(), f["row_loss"][rows],
                                               rtol=5e-3 if dtype == "f32" else LOSS_RTOL, atol=LOSS_RTOL, err_msg=tag)
                    assert _fro(outs[r][0].float().cpu(), f["dX"][rows]) <= FRO_RTOL, (tag, r, "dX")
                assert _fro(outs[r][1].cpu(), f["dW"][cls]) <= FRO_RTOL, (tag, r, "dW")
                if bias:
                    assert _fro(outs[r][2].cpu(), f["db"][cls]) <= FRO_RTOL, (tag, r, "db")
                    if bc[r]:
                        Zs = np.sort(f["Z"][rows], axis=1)
                        clear = (Zs[:, -1] - Zs[:, -2]) > (2e-2 if dtype == "f32" else 1e-3)
                        assert np.array_equal(o.pred.cpu().numpy()[clear], f["pred"][rows][clear]), (tag, r)
                        np.testing.assert_allclose(o.prob.cpu().numpy(), f["prob"][rows], rtol=2e-3, err_msg=tag)
    finally:
        for o in ops:
            o.close()


CASES = [
    # world, kwargs                                               what it exercises
    (2, dict(B=24, D=192, C=3001, regime="peaked")),              # plain path, ragged tiles
    (2, dict(B=16, D=512, C=5000, expect_f1=True)),               # F1 (B_tot = 32), labels race check
    (2, dict(B=16, D=1024, C=9001, regime="peaked", bias=True, expect_f1=True)),  # F1 + bias/db/pred
    (3, dict(B=40, D=256, C=7001, regime="peaked", bias=True)),   # odd world, bias/db/predictions
    (4, dict(B=8, D=512, C=20000, expect_f1=True)),               # F1 at N = 4
    (4, dict(B=32, D=256, C=5000, capacity=[2, 1, 1, 1])),        # c3-like uneven class shards
    (2, dict(B=8, D=64, C=1000, dtype="f32")),                    # tiny: fp32 operands (tf32)
    # NEXT-3: uneven per-rank DP batch (proportional plan), a rank with no rows
    (3, dict(batch=[30, 15, 15], D=512, C=9000)),
    (4, dict(batch=[40, 40, 40, 0], D=256, C=3000, regime="peaked")),
    (4, dict(batch=[12, 8, 8, 4], D=1024, C=12_011, regime="peaked", bias=True, expect_f1=True)),
    # N = 8 (the largest world the library takes; gpurun boxes stop at 4 GPUs)
    (8, dict(B=32, D=2048, C=20_000)),                            # c2-like rows per rank, plain path
    (8, dict(B=4, D=512, C=20_000, regime="peaked", expect_f1=True)),  # F1 at N = 8 (B_tot = 32)
    (8, dict(B=32, D=1024, C=20_001, capacity=[2, 1, 1, 1, 1, 1, 1, 1])),  # c3's 2:1:...:1 plan on 8 ranks
]


@pytest.mark.parametrize("world,kw", CASES, ids=[f"n{w}-{i}" for i, (w, _) in enumerate(CASES)])
def test_emulated_ranks_parity(whale, world, kw):
    run_emulated(whale, world, seed=900 + world, **kw)


@pytest.mark.parametrize("B,D,C", [(16, 512, 5000), (24, 192, 3001)])  # F1 and plain path
def test_emulated_grad_scale_bf16_dw(whale, B, D, C):
    """The scaled backward with bf16 dW across 2 emulated ranks: the reduce-scattered dX and
    every shard's dW carry g = 1.75 (dX pushes are scaled before the owner's reduce)."""
    world = 2
    ops_b, streams = whale.emulated_ranks(C, D, world, local_batch=B, dw_dtype=torch.bfloat16)
    dev = ops_b[0].device
    try:
        W = syn.gen_weight((0, C), D, 21, "peaked", "bf16")
        X = syn.gen_features((0, world * B), D, 22, "bf16")
        y = syn.gen_labels((0, world * B), C, 22)
        g = torch.tensor([1.75], device=dev)
        keep, outs = [], []
        for r, o in enumerate(ops_b):
            with torch.cuda.stream(streams[r]):
                xr, yr = X[r * B:(r + 1) * B].to(dev), y[r * B:(r + 1) * B].to(dev)
                wr = W[o.o_r:o.o_r + o.C_r].to(dev).contiguous()
                keep.append((xr, yr, wr))
                o.forward(xr, yr, wr)
        for r, o in enumerate(ops_b):
            with torch.cuda.stream(streams[r]):
                outs.append(o.backward(keep[r][2], grad_scale=g))
        torch.cuda.synchronize(dev)
        f = oracle.forward_backward(X, W, y.numpy())
        for r, o in enumerate(ops_b):
            o.check()
            assert outs[r][1].dtype == torch.bfloat16
            assert _fro(outs[r][0].float().cpu(), 1.75 * f["dX"][r * B:(r + 1) * B]) <= FRO_RTOL, r
            assert _fro(outs[r][1].float().cpu(), 1.75 * f["dW"][o.o_r:o.o_r + o.C_r]) <= FRO_RTOL, r
    finally:
        for o in ops_b:
            o.close()


def test_emulated_c2_shape(whale):
    """c2's per-rank shape (D=2048, C=100K, B=32 per rank) at N=2 (plain path, B_tot = 64) and
    c2's class count with B_tot = 32 (F1)."""
    run_emulated(whale, 2, D=2048, C=100_000, B=32, steps=3, seed=9208)
    run_emulated(whale, 2, D=2048, C=100_000, B=16, steps=3, seed=9209, expect_f1=True)


def test_emulated_forward_only_steps(whale):
    """Forward-only steps (eval) between training steps must not disturb the backward's
    counters or the exchange epochs: fwd, fwd, fwd+bwd, fwd+bwd on 2 emulated ranks."""
    world, B, D, C = 2, 24, 256, 4001
    ops, streams = whale.emulated_ranks(C, D, world, local_batch=B)
    dev = ops[0].device
    W = syn.gen_weight((0, C), D, 31, "peaked", "bf16")
    wr = [W[o.o_r:o.o_r + o.C_r].to(dev).contiguous() for o in ops]
    try:
        for step, do_bwd in enumerate((False, False, True, False, True)):
            X = syn.gen_features((0, world * B), D, 40 + step, "bf16")
            y = syn.gen_labels((0, world * B), C, 40 + step)
            keep, outs = [], []
            for r, o in enumerate(ops):
                with torch.cuda.stream(streams[r]):
                    xr, yr = X[r * B:(r + 1) * B].to(dev), y[r * B:(r + 1) * B].to(dev)
                    keep.append((xr, yr))
                    o.forward(xr, yr, wr[r])
            if do_bwd:
                for r, o in enumerate(ops):
                    with torch.cuda.stream(streams[r]):
                        outs.append(o.backward(wr[r]))
            torch.cuda.synchronize(dev)
            for o in ops:
                o.check()
            f = oracle.forward_backward(X, W, y.numpy())
            assert abs(float(ops[0].loss) - f["loss"]) <= LOSS_RTOL * f["loss"], step
            assert torch.equal(ops[0].loss, ops[1].loss)
            if do_bwd:
                for r, o in enumerate(ops):
                    assert _fro(outs[r][0].float().cpu(), f["dX"][r * B:(r + 1) * B]) <= FRO_RTOL, (step, r)
                    assert _fro(outs[r][1].cpu(), f["dW"][o.o_r:o.o_r + o.C_r]) <= FRO_RTOL, (step, r)
    finally:
        for o in ops:
            o.close()


@pytest.mark.parametrize("B,D", [(16, 512), (24, 192)])  # F1 and plain path
def test_emulated_dead_peer_reports_comm(whale, B, D):
    """A rank that never calls forward: the live rank's peer waits give up after the timeout,
    its kernels finish (no trap, no sticky CUDA error) and check() reports WHALE_ERR_COMM."""
    world, C = 2, 3000
    ops, streams = whale.emulated_ranks(C, D, world, local_batch=B, timeout_ms=300)
    dev = ops[0].device
    o = ops[0]
    X = syn.gen_features((0, B), D, 3, "bf16").to(dev)
    y = syn.gen_labels((0, B), C, 3).to(dev)
    W = syn.gen_weight((o.o_r, o.o_r + o.C_r), D, 3, "init", "bf16").to(dev)
    try:
        with torch.cuda.stream(streams[0]):
            o.forward(X, y, W)
            o.backward(W)
            with pytest.raises(whale.WhaleError) as e:
                o.check()
        assert e.value.status == 7  # WHALE_ERR_COMM
        torch.cuda.synchronize(dev)  # the context is healthy: no trap / sticky error
        t = torch.ones(4, device=dev)
        assert float(t.sum()) == 4.0
    finally:
        for op in ops:
            op.close()


def test_emulated_random_fuzz(whale):
    """Seeded random multi-rank cases: world 2-4, uneven batches (zero-row ranks allowed),
    capacity-proportional class shards, both paths (F1 whenever B_tot <= 32 and D % 256 == 0),
    bias / predictions; 2 steps of new inputs each, every step against the oracle."""
    rng = np.random.default_rng(2011_0920)
    for case in range(8):
        world = int(rng.integers(2, 5))
        f1 = case % 2 == 0
        if f1:
            batch = [int(v) for v in rng.multinomial(int(rng.integers(world, 33)), [1.0 / world] * world)]
            D = int(rng.choice([256, 512, 768, 1024]))
        else:
            batch = [int(v) for v in rng.integers(0, 48, world)]
            D = int(rng.integers(1, 64)) * 8
        if sum(batch) == 0:
            batch[0] = 1
        C = int(rng.integers(world * 8, 12_000))
        cap = [int(v) for v in rng.integers(1, 4, world)] if rng.integers(0, 2) else None
        run_emulated(whale, world, D=D, C=C, batch=batch, capacity=cap, regime=str(rng.choice(["init", "peaked"])),
                     bias=bool(rng.integers(0, 2)), steps=2, seed=3000 + case)


@pytest.mark.parametrize("B,D,C", [(16, 512, 5000), (24, 192, 3001)])  # F1 and plain path
def test_emulated_standalone_gather(whale, B, D, C, monkeypatch):
    """WHALE_FUSED_GATHER=0: the bridge all-gather as its own kernel instead of the logits / F1
    prologue (the default fuses it) -- same protocol, same results."""
    monkeypatch.setenv("WHALE_FUSED_GATHER", "0")
    run_emulated(whale, 2, D=D, C=C, B=B, regime="peaked", seed=77)


def test_emulated_bwd_cta_pairs(whale):
    """The fused backward as CTA pairs (cta_group::2) at N = 2: B_tot = 1024 x D = 4096 needs no
    split-K, so the pairs run, and dX is pushed to the row owners from the paired fixup."""
    ops, _ = whale.emulated_ranks(2001, 4096, 2, local_batch=512)
    try:
        assert all(o.config()["bwd_pair"] == 1 for o in ops), [o.config()["bwd_pair"] for o in ops]
    finally:
        for o in ops:
            o.close()
    run_emulated(whale, 2, D=4096, C=2001, B=512, regime="peaked", seed=78, steps=2)


def _one_step(whale, world, B, D, C, seed):
    ops, streams = whale.emulated_ranks(C, D, world, local_batch=B)
    dev = ops[0].device
    try:
        W = syn.gen_weight((0, C), D, seed, "peaked", "bf16")
        X = syn.gen_features((0, world * B), D, seed + 1, "bf16")
        y = syn.gen_labels((0, world * B), C, seed + 1)
        keep, outs = [], []
        for r, o in enumerate(ops):
            with torch.cuda.stream(streams[r]):
                xr, yr = X[r * B:(r + 1) * B].to(dev), y[r * B:(r + 1) * B].to(dev)
                wr = W[o.o_r:o.o_r + o.C_r].to(dev).contiguous()
                keep.append((xr, yr, wr))
                o.forward(xr, yr, wr, row_loss=True)
        for r, o in enumerate(ops):
            with torch.cuda.stream(streams[r]):
                outs.append(o.backward(keep[r][2]))
        torch.cuda.synchronize(dev)
        res = []
        for r, o in enumerate(ops):
            o.check()
            res.append((o.loss.clone().cpu(), o.row_loss.clone().cpu(), outs[r][0].clone().cpu(), outs[r][1].clone().cpu()))
        return res
    finally:
        for o in ops:
            o.close()


@pytest.mark.parametrize("knob", ["WHALE_FUSED_GATHER", "WHALE_FUSED_REDUCE", "WHALE_W_L2", "WHALE_SHRINK_A",
                                  "WHALE_P_DIRECT"])
@pytest.mark.parametrize("B,D,C", [(32, 512, 6001), (16, 512, 5000)])  # plain path (B_tot = 64) and F1
def test_emulated_fusions_bitwise(whale, knob, B, D, C, monkeypatch):
    """The round-2 fusions and placement choices change where the work runs, not the arithmetic:
    with each switched off the loss, per-row loss, dX and dW of every rank are bit-identical."""
    on = _one_step(whale, 2, B, D, C, 31)
    monkeypatch.setenv(knob, "0")
    off = _one_step(whale, 2, B, D, C, 31)
    for r in range(2):
        for a, b in zip(on[r], off[r]):
            assert torch.equal(a, b), (knob, r)
