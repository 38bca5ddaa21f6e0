"""GPU parity of the CUDA path (through the C-ABI) against the fp64 oracle (world = 1).

Tolerances (BASELINE.json north_star): loss within 1e-3 relative; dX and dW within 1e-2
relative Frobenius error; plus element-wise checks (row losses, max-abs error relative to
the largest reference entry).  Shapes span several tiles with ragged M / N / K tails; the
bench configuration (c2 at N=1) runs at full size against the full oracle; the large
configurations run at full size against sampled rows / classes of the oracle.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import oracle.splitfc_oracle as orc
import synthetic as syn

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-3
FRO_RTOL = 1e-2


def _fro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def whale():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2011_09208_b200 as w
    from paper_2011_09208_b200 import _lib
    _lib.lib()  # loud failure if the library is missing
    return w


def _run(whale, X, W, y, dtype="bf16"):
    B, D = X.shape
    C = W.shape[0]
    op = whale.SplitFCSoftmaxCE(C, D, B, dtype=syn.torch_dtype(dtype))
    xd, wd, yd = X.cuda(), W.cuda(), y.cuda()
    loss = op.forward(xd, yd, wd, row_loss=True)
    dx, dw = op.backward(wd)
    op.check()
    out = {"loss": float(loss), "row_loss": op.row_loss.cpu().numpy().copy(), "dX": dx.float().cpu().numpy(),
           "dW": dw.cpu().numpy(), "cfg": op.config()}
    op.close()
    return out


def _check_full(g, f, tag="", row_rtol=LOSS_RTOL):
    assert abs(g["loss"] - f["loss"]) <= LOSS_RTOL * abs(f["loss"]), (tag, g["loss"], f["loss"])
    np.testing.assert_allclose(g["row_loss"], f["row_loss"], rtol=row_rtol, atol=LOSS_RTOL, err_msg=tag)
    assert _fro(g["dX"], f["dX"]) <= FRO_RTOL, (tag, _fro(g["dX"], f["dX"]))
    assert _fro(g["dW"], f["dW"]) <= FRO_RTOL, (tag, _fro(g["dW"], f["dW"]))
    # element-wise: no entry off by more than 2% of the largest reference magnitude
    for k in ("dX", "dW"):
        scale = np.abs(f[k]).max()
        assert np.abs(g[k] - f[k]).max() <= 2e-2 * scale + 1e-30, (tag, k)


SHAPES = [
    # B, D, C                        what it exercises
    (128, 64, 256),                # exact tiles
    (40, 192, 1000),               # ragged M (40 < 128), 3 k-blocks, ragged N
    (200, 520, 3001),              # 2 m-blocks ragged, K tail (520 = 8*64+8), ragged N
    (129, 136, 777),               # one row into a second m-block
    (1, 64, 300),                  # single row
    (16, 8, 40),                   # minimum D (K box > tensor), tiny C
    (300, 1024, 20_000),           # several waves of tiles, split-K dX
]


@pytest.mark.parametrize("B,D,C", SHAPES)
@pytest.mark.parametrize("regime", ["init", "peaked"])
def test_parity_small_bf16(whale, B, D, C, regime):
    seed = 100 + B + D + C
    X = syn.gen_features((0, B), D, seed, "bf16")
    W = syn.gen_weight((0, C), D, seed, regime, "bf16")
    y = syn.gen_labels((0, B), C, seed)
    g = _run(whale, X, W, y)
    f = oracle.forward_backward(X, W, y.numpy())
    _check_full(g, f, f"{B}x{D}x{C}/{regime}")


# Shapes that take the fused forward + dX path (F1: bf16, B_tot <= 32, D % 512 == 0, D <= 2048):
# single class tile, ragged last tile, several tiles per cluster, more clusters than tiles.
F1_SHAPES = [
    (32, 512, 100),                # one ragged tile, 36 idle clusters
    (1, 512, 129),                 # single row, 2 tiles (second holds one class)
    (17, 1024, 3001),              # ragged rows, ragged last tile
    (32, 2048, 20_000),            # 157 tiles over 37 clusters
    (24, 1536, 9000),              # D half of 768 (3 G2 blocks)
    (8, 256, 5000),                # D half of 128 (one G2 block per tile)
]


@pytest.mark.parametrize("B,D,C", F1_SHAPES)
@pytest.mark.parametrize("regime", ["init", "peaked"])
def test_parity_f1(whale, B, D, C, regime):
    seed = 300 + B + D + C
    X = syn.gen_features((0, B), D, seed, "bf16")
    W = syn.gen_weight((0, C), D, seed, regime, "bf16")
    y = syn.gen_labels((0, B), C, seed)
    g = _run(whale, X, W, y)
    assert g["cfg"]["f1"] == 1
    f = oracle.forward_backward(X, W, y.numpy())
    _check_full(g, f, f"f1 {B}x{D}x{C}/{regime}")


def test_parity_tiny_fp32(whale):
    """configs[0] tiny: B=8 per rank x 2 ranks = 16 rows, D=64, C=1000, fp32 operands
    (kind::tf32, R11), single-GPU view of the whole global batch."""
    cfg = syn.CONFIGS["tiny"]
    seed = syn.config_seed("tiny", 2)
    # R11 reading (B per rank -> B_tot = 16) and the alternative reading B_tot = 8
    for Bt, regime in ((cfg.B * 2, "init"), (cfg.B * 2, "peaked"), (cfg.B, "init"), (cfg.B, "peaked")):
        X = syn.gen_features((0, Bt), cfg.D, seed, "f32")
        W = syn.gen_weight((0, cfg.C), cfg.D, seed, regime, "f32")
        y = syn.gen_labels((0, Bt), cfg.C, seed)
        g = _run(whale, X, W, y, dtype="f32")
        f = oracle.forward_backward(X, W, y.numpy())
        # per-row loss under tf32: both operands rounded to 10+1 mantissa bits (u = 2^-11)
        # -> |dz| <~ 2u * sum_k |x_k w_k|, i.e. ~1e-3 relative on |z| ~ 20-30 in the peaked
        # regime; DESIGN.md "Tolerances" derives row_rtol = 5e-3 (mean loss keeps 1e-3).
        _check_full(g, f, f"tiny/B_tot={Bt}/{regime}", row_rtol=5e-3)


def test_labels_on_edges(whale):
    """Labels 0, C-1 and on class-tile boundaries (BN-1, BN, 2BN-1)."""
    B, D, C = 64, 128, 1000
    X = syn.gen_features((0, B), D, 7, "bf16")
    W = syn.gen_weight((0, C), D, 7, "peaked", "bf16")
    edges = [0, C - 1, 63, 64, 127, 128, 255, 256, 511, 512, 999, 998]
    y = torch.tensor([edges[i % len(edges)] for i in range(B)], dtype=torch.int64)
    g = _run(whale, X, W, y)
    _check_full(g, oracle.forward_backward(X, W, y.numpy()), "edges")


def test_zero_weight(whale):
    """W = 0: loss = ln C (to 1e-3), dX exactly 0 (W_r is zero), dW closed form."""
    B, D, C = 48, 256, 5000
    X = syn.gen_features((0, B), D, 8, "bf16")
    W = syn.gen_weight((0, C), D, 8, "zero", "bf16")
    y = syn.gen_labels((0, B), C, 8)
    g = _run(whale, X, W, y)
    assert abs(g["loss"] - math.log(C)) <= 1e-3 * math.log(C)
    assert np.all(g["dX"] == 0.0)
    f = oracle.forward_backward(X, W, y.numpy())
    assert _fro(g["dW"], f["dW"]) <= FRO_RTOL


def test_single_class(whale):
    """C = 1: softmax is 1, loss 0, G = 0 -> dX = dW = 0."""
    B, D = 20, 64
    X = syn.gen_features((0, B), D, 9, "bf16")
    W = syn.gen_weight((0, 1), D, 9, "peaked", "bf16")
    y = torch.zeros(B, dtype=torch.int64)
    g = _run(whale, X, W, y)
    assert abs(g["loss"]) <= 1e-6
    assert np.abs(g["dX"]).max() <= 1e-6 and np.abs(g["dW"]).max() <= 1e-6


def test_deterministic_bitwise(whale):
    """Two runs on the same inputs give identical bits (fixed-order reductions, no atomics)."""
    B, D, C = 96, 512, 30_000
    X = syn.gen_features((0, B), D, 10, "bf16")
    W = syn.gen_weight((0, C), D, 10, "init", "bf16")
    y = syn.gen_labels((0, B), C, 10)
    op = whale.SplitFCSoftmaxCE(C, D, B)
    xd, wd, yd = X.cuda(), W.cuda(), y.cuda()
    res = []
    for _ in range(2):
        loss = op.forward(xd, yd, wd).clone()
        dx, dw = op.backward(wd)
        res.append((loss.cpu(), dx.cpu(), dw.cpu()))
    op.check()
    assert torch.equal(res[0][0], res[1][0])
    assert torch.equal(res[0][1], res[1][1])
    assert torch.equal(res[0][2], res[1][2])


@pytest.mark.parametrize("D", [64, 512])  # plain path and F1
def test_label_out_of_range_detected(whale, D):
    B, C = 8, 100
    X = syn.gen_features((0, B), D, 11, "bf16").cuda()
    W = syn.gen_weight((0, C), D, 11, "init", "bf16").cuda()
    y = torch.tensor([0, 1, 2, 100, 4, 5, 6, 7], dtype=torch.int32, device="cuda")
    op = whale.SplitFCSoftmaxCE(C, D, B)
    op.forward(X, y, W)
    with pytest.raises(whale.WhaleError) as e:
        op.check()
    assert e.value.status == 5
    op.check()  # error word cleared


def test_backward_before_forward(whale):
    op = whale.SplitFCSoftmaxCE(100, 64, 4)
    W = torch.zeros(100, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(whale.WhaleError) as e:
        op.backward(W)
    assert e.value.status == 4


def test_autograd_function(whale):
    B, D, C = 32, 128, 700
    X = syn.gen_features((0, B), D, 12, "bf16").cuda().requires_grad_(True)
    W = syn.gen_weight((0, C), D, 12, "init", "bf16").cuda().requires_grad_(True)
    y = syn.gen_labels((0, B), C, 12).cuda()
    op = whale.SplitFCSoftmaxCE(C, D, B)
    loss = whale.split_fc_softmax_ce(X, W, y, op)
    (2.0 * loss).backward()
    f = oracle.forward_backward(X.detach().cpu(), W.detach().cpu(), y.cpu().numpy())
    assert abs(loss.item() - f["loss"]) <= LOSS_RTOL * f["loss"]
    assert _fro(X.grad.float().cpu(), 2 * f["dX"]) <= FRO_RTOL
    assert _fro(W.grad.float().cpu(), 2 * f["dW"]) <= FRO_RTOL


@pytest.mark.parametrize("B,D,C", [(32, 1024, 9001), (200, 520, 3001)])  # F1 and plain path
def test_autograd_bf16_grad_no_eager_pass(whale, B, D, C):
    """Autograd with a bf16 weight and an op built with dw_dtype=bf16: grad_output (here 2.5)
    is applied inside the kernels (whale_splitfc_backward_scaled) and W.grad is written in bf16
    directly; both gradients match 2.5 x the oracle's."""
    X = syn.gen_features((0, B), D, 13, "bf16").cuda().requires_grad_(True)
    W = syn.gen_weight((0, C), D, 13, "peaked", "bf16").cuda().requires_grad_(True)
    y = syn.gen_labels((0, B), C, 13).cuda()
    op = whale.SplitFCSoftmaxCE(C, D, B, dw_dtype=torch.bfloat16)
    loss = whale.split_fc_softmax_ce(X, W, y, op)
    (2.5 * loss).backward()
    f = oracle.forward_backward(X.detach().cpu(), W.detach().cpu(), y.cpu().numpy())
    assert W.grad.dtype == torch.bfloat16
    assert abs(loss.item() - f["loss"]) <= LOSS_RTOL * f["loss"]
    assert _fro(X.grad.float().cpu(), 2.5 * f["dX"]) <= FRO_RTOL
    assert _fro(W.grad.float().cpu(), 2.5 * f["dW"]) <= FRO_RTOL
    op.close()


@pytest.mark.parametrize("B,D,C", [(32, 2048, 20_000), (96, 512, 7001)])
def test_grad_scale_and_bf16_dw(whale, B, D, C):
    """whale_splitfc_backward_scaled: outputs scale with the device scalar g (fp32 dW: within
    fp32 rounding of g x the unscaled result); bf16 dW equals the fp32 dW rounded once."""
    X = syn.gen_features((0, B), D, 14, "bf16").cuda()
    W = syn.gen_weight((0, C), D, 14, "peaked", "bf16").cuda()
    b = syn.gen_bias((0, C), 14, 2.0, "bf16").cuda()
    y = syn.gen_labels((0, B), C, 14).cuda()
    g = torch.tensor([-0.375], device="cuda")
    op = whale.SplitFCSoftmaxCE(C, D, B)
    op.forward(X, y, W, bias=b)
    dx0, dw0, db0 = [t.clone() for t in op.backward(W, bias_grad=True)]
    op.forward(X, y, W, bias=b)
    dx1, dw1, db1 = op.backward(W, bias_grad=True, grad_scale=g)
    op.check()
    torch.testing.assert_close(dw1, dw0 * g, rtol=1e-6, atol=1e-12)
    torch.testing.assert_close(db1, db0 * g, rtol=1e-6, atol=1e-12)
    torch.testing.assert_close(dx1.float(), (dx0.float() * g), rtol=2 ** -7, atol=1e-9)
    op.close()
    op = whale.SplitFCSoftmaxCE(C, D, B, dw_dtype=torch.bfloat16)
    op.forward(X, y, W)
    _, dwb = op.backward(W)
    op.check()
    assert dwb.dtype == torch.bfloat16
    opf = whale.SplitFCSoftmaxCE(C, D, B)
    opf.forward(X, y, W)
    _, dwf = opf.backward(W)
    opf.check()
    assert torch.equal(dwb, dwf.to(torch.bfloat16))
    op.close()
    opf.close()


# ------------------------------------------------------------------ full sizes
def test_parity_c2_full_bench_config(whale):
    """configs[1] c2 at N=1 (the bench workload): B=32, D=2048, C=100K, full oracle."""
    cfg = syn.CONFIGS["c2"]
    seed = syn.config_seed("c2", 1)
    for regime in ("init", "peaked"):
        X = syn.gen_features((0, cfg.B), cfg.D, seed, "bf16")
        W = syn.gen_weight((0, cfg.C), cfg.D, seed, regime, "bf16")
        y = syn.gen_labels((0, cfg.B), cfg.C, seed)
        g = _run(whale, X, W, y)
        _check_full(g, oracle.forward_backward(X, W, y.numpy()), f"c2/{regime}")


@pytest.mark.parametrize("regime", ["init", "peaked"])
@pytest.mark.parametrize("name,B_override", [("c4", 0), ("c5", 0), ("c4", 32)])
def test_parity_large_sampled(whale, name, B_override, regime):
    """Full-size single-GPU runs of the larger configs (c4 as B_tot=256 on one GPU; c5 at
    N=1; c4's 1M classes at B_tot = 32, i.e. the F1 path over 7813 class tiles) against
    sampled oracle rows / classes, plus the any-size property sum_j dW_j = 0.  In the init
    regime dX ~ -W_y / B_tot (the softmax part sum_j p_ij W_j is ~x/D, a few % of a row), so
    the softmax part dX + W_y / B_tot is checked on its own as well."""
    cfg = syn.CONFIGS[name]
    seed = syn.config_seed(name, 1)
    B, D, C = B_override or cfg.B, cfg.D, cfg.C
    X = syn.gen_features((0, B), D, seed, "bf16", device="cuda")
    W = syn.gen_weight((0, C), D, seed, regime, "bf16", device="cuda")
    y = syn.gen_labels((0, B), C, seed, device="cuda")
    op = whale.SplitFCSoftmaxCE(C, D, B)
    loss = float(op.forward(X, y, W, row_loss=True))
    row_loss = op.row_loss.cpu().numpy()
    dx, dw = op.backward(W)
    op.check()
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(B, 8, replace=False))
    classes = np.concatenate([[0, C - 1], rng.choice(C, 14, replace=False)])
    Xc, Wc, yc = X.cpu(), W.cpu(), y.cpu().numpy()
    s = orc.sampled_rows(Xc, Wc, yc, rows)
    np.testing.assert_allclose(row_loss[rows], s["row_loss"], rtol=LOSS_RTOL, atol=LOSS_RTOL)
    dx_rows = dx.float().cpu().numpy()[rows]
    assert _fro(dx_rows, s["dX"]) <= FRO_RTOL
    # the softmax part sum_j p_ij W_j / B_tot = dX + W_y / B_tot (one-hot part exact in fp64):
    # within 1e-2 of itself, plus the floor of dX's bf16 output rounding (2^-8 of |dX|),
    # which alone exceeds 1e-2 of the softmax part in the init regime
    wy = orc._f64(Wc[yc[rows]]) / B
    sm_ref = s["dX"] + wy
    err = np.linalg.norm(dx_rows + wy - sm_ref)
    assert err <= FRO_RTOL * np.linalg.norm(sm_ref) + 2.0 ** -8 * np.linalg.norm(s["dX"]), (
        err, np.linalg.norm(sm_ref), np.linalg.norm(s["dX"]))
    _, _, lse = orc.row_stats_chunked(Xc, Wc)
    ref_loss = float(np.mean(lse - np.einsum("ij,ij->i", orc._f64(Xc), orc._f64(Wc[yc]))))
    assert abs(loss - ref_loss) <= LOSS_RTOL * ref_loss
    dW_ref = orc.sampled_classes(Xc, Wc, yc, classes, lse)
    assert _fro(dw[torch.as_tensor(classes, device="cuda")].cpu().numpy(), dW_ref) <= FRO_RTOL
    # property at any size: column sums of dW over all classes vanish (rows of G sum to 0)
    colsum = dw.double().sum(0)
    assert float(colsum.abs().max()) <= 1e-2 * float(dw.double().abs().sum(0).max())


# ------------------------------------------------------------ bias + predictions (NEXT-4)
@pytest.mark.parametrize("B,D,C,dtype", [(40, 192, 1000, "bf16"), (200, 520, 3001, "bf16"),
                                         (32, 2048, 100_000, "bf16"), (16, 64, 1000, "f32")])
def test_bias_and_predictions(whale, B, D, C, dtype):
    seed = 200 + B
    X = syn.gen_features((0, B), D, seed, dtype)
    W = syn.gen_weight((0, C), D, seed, "peaked", dtype)
    b = syn.gen_bias((0, C), seed, 2.0, dtype)
    y = syn.gen_labels((0, B), C, seed)
    op = whale.SplitFCSoftmaxCE(C, D, B, dtype=syn.torch_dtype(dtype))
    xd, wd, bd = X.cuda(), W.cuda(), b.cuda()  # x stays alive: backward reads it (header contract)
    loss = float(op.forward(xd, y.cuda(), wd, row_loss=True, bias=bd, predictions=True))
    dx, dw, db = op.backward(wd, bias_grad=True)
    op.check()
    f = oracle.forward_backward(X, W, y.numpy(), b)
    assert abs(loss - f["loss"]) <= LOSS_RTOL * abs(f["loss"])
    assert _fro(dx.float().cpu(), f["dX"]) <= FRO_RTOL
    assert _fro(dw.cpu(), f["dW"]) <= FRO_RTOL
    assert _fro(db.cpu(), f["db"]) <= FRO_RTOL
    pred = op.pred.cpu().numpy()
    prob = op.prob.cpu().numpy()
    # top-1 is unique where the oracle's best and second-best logits differ clearly
    Z = np.sort(f["Z"], axis=1)
    clear = (Z[:, -1] - Z[:, -2]) > (2e-2 if dtype == "f32" else 1e-3)
    assert np.array_equal(pred[clear], f["pred"][clear])
    assert np.all((pred >= 0) & (pred < C))
    np.testing.assert_allclose(prob, f["prob"], rtol=5e-3 if dtype == "f32" else 1e-3)


@pytest.mark.parametrize("B,D,C", [(32, 2048, 20_000), (64, 512, 5000)])
def test_cuda_graph_replay(whale, B, D, C):
    """The bench captures one step as a CUDA graph and replays it: the device-resident step
    epoch must make every replay compute the same thing as an eager step (F1 and plain path).
    The input CONTENTS change between replays (new features and labels copied into the
    captured buffers), and every replay is compared bit for bit with an eager step on the same
    inputs and with the fp64 oracle."""
    seed = 400 + B
    W = syn.gen_weight((0, C), D, seed, "peaked", "bf16").cuda()
    X = torch.empty(B, D, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(B, dtype=torch.int32, device="cuda")
    op = whale.SplitFCSoftmaxCE(C, D, B)
    dx = torch.empty(B, D, dtype=torch.bfloat16, device="cuda")
    dw = torch.empty(C, D, dtype=torch.float32, device="cuda")

    def inputs(k):
        Xh = syn.gen_features((0, B), D, seed + 31 * k, "bf16")
        yh = syn.gen_labels((0, B), C, seed + 31 * k)
        return Xh, yh

    Xh, yh = inputs(0)
    X.copy_(Xh)
    y.copy_(yh)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        op.forward(X, y, W)  # warm-up on the capture stream
        op.backward(W, dx, dw)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        op.forward(X, y, W)
        op.backward(W, dx, dw)
    for k in range(1, 4):
        Xh, yh = inputs(k)
        X.copy_(Xh)
        y.copy_(yh)
        dx.zero_()
        dw.zero_()
        g.replay()
        torch.cuda.synchronize()
        op.check()
        got = (op.loss.clone(), dx.clone(), dw.clone())
        op.forward(X, y, W)  # eager step on the same inputs
        op.backward(W, dx, dw)
        torch.cuda.synchronize()
        op.check()
        assert torch.equal(got[0], op.loss), k
        assert torch.equal(got[1], dx), k
        assert torch.equal(got[2], dw), k
        f = oracle.forward_backward(Xh, W.cpu(), yh.numpy())
        assert abs(float(got[0]) - f["loss"]) <= LOSS_RTOL * f["loss"], k
        assert _fro(got[1].float().cpu(), f["dX"]) <= FRO_RTOL, k
        assert _fro(got[2].cpu(), f["dW"]) <= FRO_RTOL, k
    op.close()


@pytest.mark.parametrize("B,D,C", [(32, 512, 3001), (48, 192, 3001)])  # F1 and plain path
def test_forward_only_steps(whale, B, D, C):
    """An eval forward (no backward) between training steps must leave the backward intact:
    fwd, fwd, fwd+bwd, fwd, fwd+bwd with new inputs each time, all against the oracle."""
    W = syn.gen_weight((0, C), D, 61, "peaked", "bf16")
    wd = W.cuda()
    op = whale.SplitFCSoftmaxCE(C, D, B)
    for k, do_bwd in enumerate((False, False, True, False, True)):
        X = syn.gen_features((0, B), D, 70 + k, "bf16")
        y = syn.gen_labels((0, B), C, 70 + k)
        xd = X.cuda()
        loss = float(op.forward(xd, y.cuda(), wd))
        f = oracle.forward_backward(X, W, y.numpy())
        assert abs(loss - f["loss"]) <= LOSS_RTOL * f["loss"], k
        if do_bwd:
            dx, dw = op.backward(wd)
            op.check()
            assert _fro(dx.float().cpu(), f["dX"]) <= FRO_RTOL, k
            assert _fro(dw.cpu(), f["dW"]) <= FRO_RTOL, k
    op.check()
    op.close()


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("B,D,C", [(200, 520, 3001), (300, 1024, 20_000), (129, 136, 777), (256, 2048, 10_000)])
def test_cta_pair_mma(whale, B, D, C, fused, monkeypatch):
    """CTA pairs (tcgen05.mma.cta_group::2, M = 256, each CTA holding half of B): forced on for
    the logits (and, with the unfused backward, the standalone dW / dX GEMMs) at small shapes
    incl. an odd M-block count (padding tile) -- against the oracle, with bias and predictions."""
    monkeypatch.setenv("WHALE_CLUSTER", "2")
    monkeypatch.setenv("WHALE_FUSED_BWD", fused)
    seed = 900 + B
    X = syn.gen_features((0, B), D, seed, "bf16")
    W = syn.gen_weight((0, C), D, seed, "peaked", "bf16")
    b = syn.gen_bias((0, C), seed, 2.0, "bf16")
    y = syn.gen_labels((0, B), C, seed)
    op = whale.SplitFCSoftmaxCE(C, D, B)
    assert op.config()["fwd"]["cluster"] == 2
    xd, wd = X.cuda(), W.cuda()
    loss = float(op.forward(xd, y.cuda(), wd, row_loss=True, bias=b.cuda(), predictions=True))
    dx, dw, db = op.backward(wd, bias_grad=True)
    op.check()
    f = oracle.forward_backward(X, W, y.numpy(), b)
    assert abs(loss - f["loss"]) <= LOSS_RTOL * f["loss"]
    np.testing.assert_allclose(op.row_loss.cpu().numpy(), f["row_loss"], rtol=LOSS_RTOL, atol=LOSS_RTOL)
    assert _fro(dx.float().cpu(), f["dX"]) <= FRO_RTOL
    assert _fro(dw.cpu(), f["dW"]) <= FRO_RTOL
    assert _fro(db.cpu(), f["db"]) <= FRO_RTOL
    Z = np.sort(f["Z"], axis=1)
    clear = (Z[:, -1] - Z[:, -2]) > 1e-3
    assert np.array_equal(op.pred.cpu().numpy()[clear], f["pred"][clear])
    op.close()


@pytest.mark.parametrize("B,D,C", [(1024, 4096, 3001), (1152, 4096, 1003)])
def test_bwd_cta_pairs(whale, B, D, C, monkeypatch):
    """CTA pairs in the fused backward (cta_group::2, M = 256 units; the leader's scheduler hands
    each unit to the peer through DSMEM): on by default when dX needs no split-K (here 8 x 16 and
    9 x 16 tiles -- the odd M-block count gets a padding tile).  Against the oracle (fp32 dW),
    against the unpaired kernel, and bf16 dW = the fp32 dW rounded once."""
    seed = 700 + B
    X = syn.gen_features((0, B), D, seed, "bf16")
    W = syn.gen_weight((0, C), D, seed, "peaked", "bf16")
    y = syn.gen_labels((0, B), C, seed)
    op = whale.SplitFCSoftmaxCE(C, D, B)
    cfg = op.config()
    assert cfg["bwd_pair"] == 1 and cfg["dx"]["cluster"] == 2, cfg
    xd, wd, yd = X.cuda(), W.cuda(), y.cuda()
    loss = float(op.forward(xd, yd, wd, row_loss=True))
    dx, dw = [t.clone() for t in op.backward(wd)]
    op.check()
    f = oracle.forward_backward(X, W, y.numpy())
    assert abs(loss - f["loss"]) <= LOSS_RTOL * f["loss"]
    assert _fro(dx.float().cpu(), f["dX"]) <= FRO_RTOL
    assert _fro(dw.cpu(), f["dW"]) <= FRO_RTOL
    for k, g in (("dX", dx.float().cpu().numpy()), ("dW", dw.cpu().numpy())):
        scale = np.abs(f[k]).max()
        assert np.abs(g - f[k]).max() <= 2e-2 * scale, k
    op.close()
    monkeypatch.setenv("WHALE_BWD_PAIR", "0")
    op0 = whale.SplitFCSoftmaxCE(C, D, B)
    assert op0.config()["bwd_pair"] == 0
    op0.forward(xd, yd, wd)
    dx0, dw0 = op0.backward(wd)
    op0.check()
    assert _fro(dw.cpu(), dw0.cpu()) <= 1e-5 and _fro(dx.float().cpu(), dx0.float().cpu()) <= 1e-2
    op0.close()
    monkeypatch.delenv("WHALE_BWD_PAIR")
    opb = whale.SplitFCSoftmaxCE(C, D, B, dw_dtype=torch.bfloat16)
    assert opb.config()["bwd_pair"] == 1
    opb.forward(xd, yd, wd)
    _, dwb = opb.backward(wd)
    opb.check()
    assert torch.equal(dwb, dw.to(torch.bfloat16))
    opb.close()


@pytest.mark.parametrize("B,D,C", [(32, 1024, 9001), (200, 520, 3001), (300, 1024, 20_000)])
def test_gfused_backward_matches_materialised(whale, B, D, C, monkeypatch):
    """NEXT-4b: the G-fused backward (G formed from P~ in the operand path) computes the same
    G as the in-place rewrite (same expression), so dX / dW / db agree with the materialised
    path to the last bit, and both match the oracle."""
    seed = 800 + B
    X = syn.gen_features((0, B), D, seed, "bf16")
    W = syn.gen_weight((0, C), D, seed, "peaked", "bf16")
    b = syn.gen_bias((0, C), seed, 2.0, "bf16")
    y = syn.gen_labels((0, B), C, seed)
    xd, wd, bd, yd = X.cuda(), W.cuda(), b.cuda(), y.cuda()
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("WHALE_GFUSE", mode)
        op = whale.SplitFCSoftmaxCE(C, D, B)
        op.forward(xd, yd, wd, bias=bd)
        res[mode] = [t.clone() for t in op.backward(wd, bias_grad=True)]
        op.check()
        op.close()
    f = oracle.forward_backward(X, W, y.numpy(), b)
    for k, name in enumerate(("dX", "dW", "db")):
        assert _fro(res["1"][k].float().cpu(), f[name]) <= FRO_RTOL, name
        assert torch.equal(res["1"][k], res["0"][k]), name


def test_random_shapes_fuzz(whale):
    """Seeded random shapes across both paths (F1 when B_tot <= 32 and D % 256 == 0, else the
    plain GEMMs): loss / dX / dW / db / predictions against the oracle."""
    rng = np.random.default_rng(2011_09208)
    for case in range(24):
        f1 = case % 2 == 0
        B = int(rng.integers(1, 33)) if f1 else int(rng.integers(1, 300))
        D = int(rng.choice([256, 512, 768, 1024, 1536, 2048])) if f1 else int(rng.integers(1, 96)) * 8
        C = int(rng.integers(1, 9000))
        regime = str(rng.choice(["init", "peaked"]))
        bias = bool(rng.integers(0, 2))
        seed = 500 + case
        X = syn.gen_features((0, B), D, seed, "bf16")
        W = syn.gen_weight((0, C), D, seed, regime, "bf16")
        y = syn.gen_labels((0, B), C, seed)
        b = syn.gen_bias((0, C), seed, 1.0, "bf16") if bias else None
        op = whale.SplitFCSoftmaxCE(C, D, B)
        xd, wd = X.cuda(), W.cuda()
        bd = b.cuda() if bias else None
        loss = float(op.forward(xd, y.cuda(), wd, row_loss=True, bias=bd, predictions=True))
        out = op.backward(wd, bias_grad=bias)
        op.check()
        f = oracle.forward_backward(X, W, y.numpy(), b)
        tag = f"case {case}: B={B} D={D} C={C} {regime} bias={bias} f1={op.config()['f1']}"
        assert abs(loss - f["loss"]) <= LOSS_RTOL * max(abs(f["loss"]), 1e-3), tag
        if np.linalg.norm(f["dX"]) > 0:
            assert _fro(out[0].float().cpu(), f["dX"]) <= FRO_RTOL, tag
        if np.linalg.norm(f["dW"]) > 0:
            assert _fro(out[1].cpu(), f["dW"]) <= FRO_RTOL, tag
        if bias and np.linalg.norm(f["db"]) > 0:
            assert _fro(out[2].cpu(), f["db"]) <= FRO_RTOL, tag
        Z = np.sort(f["Z"], axis=1)
        clear = (Z[:, -1] - Z[:, -2]) > 1e-3 if C > 1 else np.ones(B, bool)
        assert np.array_equal(op.pred.cpu().numpy()[clear], f["pred"][clear]), tag
        op.close()


def test_f1_reference_moves(whale):
    """F1's lazy per-row reference must move (U rescaled in TMEM) when later class tiles hold
    much larger logits: scale W's rows up along the class index so every cluster's later tiles
    exceed its first tile's max by far more than the 2^8 threshold."""
    B, D, C = 32, 512, 40_000
    X = syn.gen_features((0, B), D, 77, "bf16")
    W0 = syn.gen_weight((0, C), D, 77, "peaked", "bf16").float()
    ramp = torch.linspace(0.2, 3.0, C).unsqueeze(1)
    W = (W0 * ramp).to(torch.bfloat16)
    y = syn.gen_labels((0, B), C, 77)
    g = _run(whale, X, W, y)
    assert g["cfg"]["f1"] == 1
    _check_full(g, oracle.forward_backward(X, W, y.numpy()), "f1 reference moves")
