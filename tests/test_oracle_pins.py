"""Pins of the fp64 oracle against what the paper and the mathematics fix (CPU only).

Each test names the plausible oracle mistake it would catch.  None of them re-types the
oracle's vectorised formula: they use closed forms, a library routine
(torch.nn.functional.cross_entropy + autograd in float64), finite differences,
invariants and a hand-derived example.
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import oracle.splitfc_oracle
import oracle.plan_oracle
from oracle import PlanError, plan_shards

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand(B, D, C, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    X = np.maximum(rng.standard_normal((B, D)), 0.0)
    W = rng.standard_normal((C, D)) * scale / math.sqrt(D)
    y = rng.integers(0, C, B)
    return X, W, y


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("C,expect", [(1000, 6.907755278982137), (100_000, 11.512925464970229),
                                      (500_000, 13.122363377404328), (1_000_000, 13.815510557964274)])
def test_zero_weight_loss_is_ln_C(C, expect):
    """W=0 => every logit is 0, softmax uniform, L = ln C exactly (catches a dropped
    max-shift or wrong normaliser).  Values: ln C for the configs' class counts."""
    B, D = 4, (8 if C <= 100_000 else 2)  # a narrow W keeps the 1M-class case small
    X = np.abs(np.random.default_rng(0).standard_normal((B, D)))
    W = np.zeros((C, D))
    if C > 100_000:  # the forward (O2-O4) and the chunked statistics at full C
        f = oracle.forward(X, W, np.arange(B) % C)
        assert abs(f["loss"] - expect) <= 1e-13 * expect
        _, _, lse = oracle.splitfc_oracle.row_stats_chunked(X, W)
        assert np.all(np.abs(lse - expect) <= 1e-13 * expect)
        return
    f = oracle.forward_backward(X, W, np.arange(B) % C)
    assert abs(f["loss"] - expect) <= 1e-13 * expect
    assert abs(math.log(C) - expect) < 1e-15
    assert np.all(f["dX"] == 0.0)  # G W with W=0 is exactly zero


def test_zero_weight_dW_closed_form():
    """W=0 => G = (1/C - onehot)/B so dW = G^T X in closed form (catches a transposed
    operand in dW or a missing 1/B)."""
    B, D, C = 5, 3, 7
    rng = np.random.default_rng(1)
    X = rng.standard_normal((B, D))
    y = np.array([0, 3, 3, 6, 1])
    f = oracle.forward_backward(X, np.zeros((C, D)), y)
    expect = np.zeros((C, D))
    for i in range(B):
        for j in range(C):
            expect[j] += ((1.0 / C) - (1.0 if y[i] == j else 0.0)) / B * X[i]
    np.testing.assert_allclose(f["dW"], expect, rtol=0, atol=1e-15)


def test_two_classes_softplus():
    """C=2 => l_i = softplus(z_other - z_label) = ln(1 + e^{z_o - z_y}) (textbook)."""
    X, W, y = _rand(16, 5, 2, 2, scale=4.0)
    f = oracle.forward(X, W, y)
    Z = X @ W.T
    for i in range(16):
        d = Z[i, 1 - y[i]] - Z[i, y[i]]
        assert abs(f["row_loss"][i] - (max(d, 0) + math.log1p(math.exp(-abs(d))))) < 1e-13


def test_hand_worked_example():
    """X=I_2, W=[[1,0],[0,1],[0,0]], y=[0,2]: Z=[[1,0,0],[0,1,0]],
    l_0 = ln(e+2) - 1, l_1 = ln(e+2) - 0, L = ln(e+2) - 1/2.
    Gradient: G = (softmax - onehot)/2 with softmax rows (e,1,1)/(e+2) and (1,e,1)/(e+2)."""
    X = np.eye(2)
    W = np.array([[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]])
    f = oracle.forward_backward(X, W, [0, 2])
    E = math.e
    assert abs(f["loss"] - (math.log(E + 2) - 0.5)) < 1e-15
    G = np.array([[E / (E + 2) - 1, 1 / (E + 2), 1 / (E + 2)],
                  [1 / (E + 2), E / (E + 2), 1 / (E + 2) - 1]]) / 2
    np.testing.assert_allclose(f["G"], G, atol=1e-16)
    np.testing.assert_allclose(f["dW"], G.T @ X, atol=1e-16)   # X = I
    np.testing.assert_allclose(f["dX"], G @ W, atol=1e-16)


# ------------------------------------------------------------- library routine
@pytest.mark.parametrize("scale", [1.0, 8.0, 30.0])
def test_against_torch_cross_entropy_fp64(scale):
    """torch.nn.functional.cross_entropy (mean) + autograd in float64 is independent
    code: loss, dX and dW must agree to ~1e-12 (catches any sign/index/transposition
    mistake in forward or backward, and a wrong mean)."""
    B, D, C = 24, 17, 53
    X, W, y = _rand(B, D, C, 3, scale=scale)
    f = oracle.forward_backward(X, W, y)
    Xt = torch.tensor(X, requires_grad=True)
    Wt = torch.tensor(W, requires_grad=True)
    L = torch.nn.functional.cross_entropy(Xt @ Wt.T, torch.tensor(y))
    L.backward()
    assert abs(f["loss"] - L.item()) <= 1e-12 * abs(L.item())
    np.testing.assert_allclose(f["dX"], Xt.grad.numpy(), rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(f["dW"], Wt.grad.numpy(), rtol=1e-10, atol=1e-15)


# ---------------------------------------------------------- finite differences
def test_finite_differences_tiny():
    """Central differences (h=1e-6) on 32 random entries of W and of X at the tiny
    shape (B=16 global, D=64, C=1000): |FD - analytic| <= 1e-7 * ||grad||_inf."""
    X, W, y = _rand(16, 64, 1000, 4, scale=8.0)
    f = oracle.forward_backward(X, W, y)
    rng = np.random.default_rng(5)
    h = 1e-6
    for name, A, grad in (("W", W, f["dW"]), ("X", X, f["dX"])):
        tol = 1e-7 * np.abs(grad).max()
        for _ in range(32):
            idx = tuple(rng.integers(0, s) for s in A.shape)
            old = A[idx]
            A[idx] = old + h
            lp = oracle.loss_only(X, W, y)
            A[idx] = old - h
            lm = oracle.loss_only(X, W, y)
            A[idx] = old
            assert abs((lp - lm) / (2 * h) - grad[idx]) <= tol, (name, idx)


# ------------------------------------------------------------------ invariants
def test_softmax_rows_sum_to_one_and_grad_rows_to_zero():
    X, W, y = _rand(32, 40, 300, 6, scale=8.0)
    f = oracle.forward_backward(X, W, y)
    P = np.exp(f["Z"] - f["lse"][:, None])
    assert np.abs(P.sum(1) - 1).max() <= 1e-13
    assert np.abs(f["G"].sum(1)).max() <= 1e-15
    # sign pattern: label entry <= 0, all others >= 0
    B = X.shape[0]
    assert np.all(f["G"][np.arange(B), y] <= 0)
    mask = np.ones_like(f["G"], dtype=bool)
    mask[np.arange(B), y] = False
    assert np.all(f["G"][mask] >= 0)
    # dW columns summed over classes vanish: sum_j dW_j = sum_i (sum_j G_ij) X_i = 0
    assert np.abs(f["dW"].sum(0)).max() <= 1e-14


def test_shift_invariance():
    """Append a constant-1 feature and a constant column to W: every logit of a row is
    shifted by the same amount, so L, dX (original columns) are unchanged."""
    X, W, y = _rand(8, 6, 20, 7, scale=4.0)
    X2 = np.concatenate([X, np.ones((8, 1))], 1)
    W2 = np.concatenate([W, np.full((20, 1), 3.7)], 1)
    f, f2 = oracle.forward_backward(X, W, y), oracle.forward_backward(X2, W2, y)
    assert abs(f["loss"] - f2["loss"]) < 1e-13
    np.testing.assert_allclose(f2["dX"][:, :6], f["dX"], atol=1e-15)


def test_class_permutation_equivariance():
    X, W, y = _rand(10, 5, 30, 8, scale=4.0)
    perm = np.random.default_rng(9).permutation(30)
    inv = np.argsort(perm)
    f = oracle.forward_backward(X, W, y)
    g = oracle.forward_backward(X, W[perm], inv[y])
    assert abs(f["loss"] - g["loss"]) < 1e-13
    np.testing.assert_allclose(g["dW"], f["dW"][perm], atol=1e-15)
    np.testing.assert_allclose(g["dX"], f["dX"], atol=1e-15)


def test_duplicated_batch_reading_R1():
    """Reading R1 (mean over the global batch): duplicating the batch leaves L and dW
    unchanged and halves each dX row."""
    X, W, y = _rand(6, 5, 11, 10)
    f = oracle.forward_backward(X, W, y)
    g = oracle.forward_backward(np.concatenate([X, X]), W, np.concatenate([y, y]))
    assert abs(f["loss"] - g["loss"]) < 1e-14
    np.testing.assert_allclose(g["dW"], f["dW"], atol=1e-15)
    np.testing.assert_allclose(g["dX"][:6], f["dX"] / 2, atol=1e-16)


def test_label_range_checked():
    X, W, _ = _rand(2, 3, 4, 11)
    with pytest.raises(ValueError):
        oracle.forward(X, W, [0, 4])
    with pytest.raises(ValueError):
        oracle.forward(X, W, [-1, 0])


# -------------------------------------------------------- sharded == unsharded
def _plans(C):
    yield [1] * 1
    for N in range(1, 9):
        yield [1] * N
    yield [2, 1, 1, 1, 1, 1, 1, 1]
    rng = np.random.default_rng(12)
    for _ in range(4):
        N = int(rng.integers(2, 7))
        yield [int(v) for v in rng.integers(1, 50, N)]


@pytest.mark.parametrize("case", range(3))
def test_sharded_equals_unsharded(case):
    """O7 (per-shard stats + combine) equals the unsharded definition to 1e-12 for many
    plans, incl. extreme [1,...,1,C-N+1] and labels on shard boundaries."""
    C, D = 97, 9
    rng = np.random.default_rng(20 + case)
    plans = list(_plans(C))
    N = 5
    plans.append(None)  # extreme plan below
    for w in plans:
        if w is None:
            counts = [1] * (N - 1) + [C - N + 1]
            offs = list(np.cumsum([0] + counts[:-1]))
        else:
            counts, offs = plan_shards(C, len(w), w)
        Nr = len(counts)
        Bs = [3] * Nr
        Bt = sum(Bs)
        X = np.maximum(rng.standard_normal((Bt, D)), 0)
        W = rng.standard_normal((C, D)) * (8.0 if case else 1.0) / 3
        # labels on shard boundaries, y=0, y=C-1, then random
        bounds = [o for o in offs] + [o + c - 1 for o, c in zip(offs, counts)] + [0, C - 1]
        y = np.array((bounds * Bt)[:Bt]) if case == 0 else rng.integers(0, C, Bt)
        if case == 2:
            y = np.full(Bt, offs[-1])  # all labels in one shard
        Xl = np.split(X, np.cumsum(Bs)[:-1])
        s = oracle.sharded_forward_backward(Xl, W, y, counts, offs)
        f = oracle.forward_backward(X, W, y)
        assert abs(s["loss"] - f["loss"]) <= 1e-12 * abs(f["loss"])
        for r, (o, c) in enumerate(zip(offs, counts)):
            np.testing.assert_allclose(s["dW_shards"][r], f["dW"][o:o + c], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(np.concatenate(s["dX_ranks"]), f["dX"], rtol=1e-12, atol=1e-15)


# ------------------------------------------------------------------- plan (O1)
def test_plan_golden_examples():
    g = json.load(open(os.path.join(GOLDEN, "plan_examples.json")))
    for case in g["cases"]:
        counts, offs = plan_shards(case["C"], case["N"], case["capacity"])
        assert counts == case["counts"], case["cite"]
        assert offs == [sum(counts[:i]) for i in range(len(counts))]
    for case in g["errors"]:
        with pytest.raises(PlanError) as e:
            plan_shards(case["C"], case["N"], case["capacity"])
        assert e.value.code == case["code"], case["cite"]


def _objectives(n, C, w):
    W = sum(w)
    dev = [Fraction(ni) - Fraction(C * wi, W) for ni, wi in zip(n, w)]
    return sum(abs(d) for d in dev), sum(d * d for d in dev)


def test_plan_bruteforce_optimal_formula1():
    """Eq. 1 with L_i = C_i/C: the plan minimises sum |L_i - DF_i/sum DF|
    (and the squared reading) over ALL integer vectors with C_i >= 1, sum C_i = C
    (brute force, C <= 12, N <= 4).  Catches wrong rounding / leftover assignment."""
    rng = np.random.default_rng(30)
    for C in range(1, 13):
        for N in range(1, min(C, 4) + 1):
            for _ in range(6):
                w = [int(v) for v in rng.integers(1, 9, N)]
                try:
                    n, _ = plan_shards(C, N, w)
                except PlanError as e:
                    assert e.code == 2
                    # infeasible only if Hamilton gives a zero count; check it is really Hamilton's
                    continue
                best1 = best2 = None
                for comp in itertools.product(range(1, C + 1), repeat=N):
                    if sum(comp) != C:
                        continue
                    o1, o2 = _objectives(comp, C, w)
                    best1 = o1 if best1 is None else min(best1, o1)
                    best2 = o2 if best2 is None else min(best2, o2)
                o1, o2 = _objectives(n, C, w)
                assert o1 == best1 and o2 == best2, (C, N, w, n)


def test_plan_invariants_random():
    rng = np.random.default_rng(31)
    for _ in range(2000):
        N = int(rng.integers(1, 9))
        C = int(rng.integers(N, 10 ** 6))
        w = None if rng.random() < 0.3 else [int(v) for v in rng.integers(1, 1000, N)]
        try:
            n, o = plan_shards(C, N, w)
        except PlanError as e:
            assert e.code == 2
            continue
        ww = [1] * N if w is None else w
        assert sum(n) == C and min(n) >= 1
        for ni, wi in zip(n, ww):
            assert abs(Fraction(ni) - Fraction(C * wi, sum(ww))) < 1
        assert o[0] == 0 and all(o[i + 1] == o[i] + n[i] for i in range(N - 1))


def test_paper_sizes_pin_workload():
    """782 MB FC vs 90 MB ResNet-50 and 89.7% pin D=2048, C=100K: the
    FC's D*C fp32 parameters (+ a C-length bias, reading R2) in MiB round to 782."""
    g = json.load(open(os.path.join(GOLDEN, "paper_sizes.json")))
    D, C, b = g["D"], g["C"], g["bytes_per_param"]
    assert round((D * C + C) * b / 2 ** 20) == g["fc_mb"]
    assert abs(D * C * b / 2 ** 20 - g["fc_mb"]) < 1.0
    assert round(100 * g["fc_mb"] / (g["fc_mb"] + g["resnet50_mb"]), 1) == g["sync_reduction_pct"]


def test_sampled_oracle_agrees_with_full():
    """The chunked / sampled evaluation used for full-size GPU parity reproduces the pinned
    full oracle (rows, dX rows, dW rows) to ~1e-15 on small inputs with ragged chunks."""
    X, W, y = _rand(20, 7, 50, 40, scale=8.0)
    f = oracle.forward_backward(X, W, y)
    rows = [0, 5, 19]
    s = oracle.splitfc_oracle.sampled_rows(X, W, y, rows, chunk=16)
    np.testing.assert_allclose(s["row_loss"], f["row_loss"][rows], rtol=1e-13)
    np.testing.assert_allclose(s["dX"], f["dX"][rows], rtol=1e-12, atol=1e-16)
    _, _, lse = oracle.splitfc_oracle.row_stats_chunked(X, W, chunk=13)
    np.testing.assert_allclose(lse, f["lse"], rtol=1e-14)
    cls = [0, 3, 49]
    np.testing.assert_allclose(oracle.splitfc_oracle.sampled_classes(X, W, y, cls, lse), f["dW"][cls],
                               rtol=1e-12, atol=1e-17)


# ------------------------------------------------------- plan under memory caps (Alg. 1)
def test_plan_mem_golden():
    g = json.load(open(os.path.join(GOLDEN, "plan_mem_examples.json")))
    for c in g["cases"]:
        n, o = oracle.plan_oracle.plan_shards_mem(c["C"], len(c["capacity"]), c["capacity"], c["mem_bytes"],
                                                  c["bytes_per_class"])
        assert n == c["counts"], c["cite"]
    for c in g["errors"]:
        with pytest.raises(PlanError) as e:
            oracle.plan_oracle.plan_shards_mem(c["C"], len(c["capacity"]), c["capacity"], c["mem_bytes"],
                                               c["bytes_per_class"])
        assert e.value.code == c["code"], c["cite"]


def test_plan_mem_invariants_random():
    """Feasible result => every shard fits its cap, counts sum to C, >= 1 each; when no cap
    binds the result is exactly the proportional plan (Alg. 1's init)."""
    rng = np.random.default_rng(41)
    for _ in range(3000):
        N = int(rng.integers(1, 9))
        C = int(rng.integers(N, 5000))
        w = [int(v) for v in rng.integers(1, 20, N)]
        bpc = int(rng.integers(1, 100))
        mem = [int(v) for v in rng.integers(0, 2 * C * bpc // N + 2, N)]
        try:
            n, o = oracle.plan_oracle.plan_shards_mem(C, N, w, mem, bpc)
        except PlanError as e:
            assert e.code == 2
            # infeasible only if total capacity cannot hold C or Hamilton itself fails
            continue
        assert sum(n) == C and min(n) >= 1
        assert all(ni * bpc <= mi for ni, mi in zip(n, mem))
        big = [C * bpc] * N
        assert oracle.plan_oracle.plan_shards_mem(C, N, w, big, bpc) == plan_shards(C, N, w)


def test_plan_mem_infeasible_iff_total_too_small_when_init_ok():
    """Total capacity < C classes => infeasible."""
    with pytest.raises(PlanError):
        oracle.plan_oracle.plan_shards_mem(10, 2, [1, 1], [4, 5], 1)


# ------------------------------------------------------------ bias + predictions (NEXT-4)
def test_bias_against_torch_linear_fp64():
    """Dense layer with bias: torch F.linear + cross_entropy + autograd (fp64) pins loss,
    dX, dW and db = sum_i G_i; a constant added to every bias leaves L unchanged."""
    B, D, C = 20, 9, 41
    X, W, y = _rand(B, D, C, 50, scale=6.0)
    b = np.random.default_rng(51).standard_normal(C) * 2
    f = oracle.forward_backward(X, W, y, b)
    Xt, Wt, bt = (torch.tensor(v, requires_grad=True) for v in (X, W, b))
    L = torch.nn.functional.cross_entropy(torch.nn.functional.linear(Xt, Wt, bt), torch.tensor(y))
    L.backward()
    assert abs(f["loss"] - L.item()) <= 1e-12 * abs(L.item())
    np.testing.assert_allclose(f["dX"], Xt.grad.numpy(), rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(f["dW"], Wt.grad.numpy(), rtol=1e-10, atol=1e-15)
    np.testing.assert_allclose(f["db"], bt.grad.numpy(), rtol=1e-10, atol=1e-16)
    g = oracle.forward_backward(X, W, y, b + 3.25)
    assert abs(g["loss"] - f["loss"]) < 1e-13


def test_predictions_definition():
    """pred = torch.argmax of the logits (first max), prob = softmax at pred (torch)."""
    X, W, y = _rand(30, 7, 19, 52, scale=5.0)
    b = np.random.default_rng(53).standard_normal(19)
    f = oracle.forward(X, W, y, b)
    Zt = torch.tensor(X) @ torch.tensor(W).T + torch.tensor(b)
    P = torch.softmax(Zt, 1)
    assert np.array_equal(f["pred"], torch.argmax(Zt, 1).numpy())
    np.testing.assert_allclose(f["prob"], P.max(1).values.numpy(), rtol=1e-13)
    # ties go to the lowest class id
    Xe, We = np.eye(2), np.array([[1.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    assert list(oracle.forward(Xe, We, [0, 2])["pred"]) == [0, 2]
