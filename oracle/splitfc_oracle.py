"""fp64 CPU oracle for Whale's split-FC softmax cross-entropy (arXiv 2011.09208).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this module.
It shares no code with the CUDA path (``paper_2011_09208_b200``) and imports nothing
from it; the two meet only on the seeded inputs of ``synthetic/``.

What it computes (plain definitions, unsharded, float64):

* Forward, PAPER.md:286-288 (§2.1 "a training loss is calculated between the produced
  scores and desired scores") and PAPER.md:689-690 (Example 2: ``logits = FC(features)``
  then ``Softmax(logits)`` under ``wh.split``):
      Z = X W^T                                    (O2: logits, W class-major [C x D])
      m_i = max_j Z_ij,  s_i = sum_j exp(Z_ij - m_i),  lse_i = m_i + ln s_i   (O3)
      l_i = lse_i - Z_{i, y_i},   L = (1/B_tot) sum_i l_i                      (O4)
  Reading §8(c).1 (R1): the loss is the mean over the GLOBAL batch.
* Backward ("utilized to compute gradients for model parameters"):
      P = exp(Z - lse),  G = (P - onehot(y)) / B_tot                          (O5)
      dW = G^T X,  dX = G W                                                   (O6)
* The bridge ("gathers the outputs from different batches for
  concatenation in batch dimension"): X = concat_r X_r in rank order (R8);
  dX_r is the rows of dX that rank r contributed.
* The class split SP1 ("shards the second input tensor in the second
  tensor dimension"): W_r = rows [o_r, o_r + C_r) of W; dW_r the same rows of dW.

Every result of the split method equals this unsharded definition up to rounding
order (the split is an exact re-association), so the oracle IS the definition.
``sharded_forward_backward`` (O7) restates the per-shard statistics combine, used only
to self-check that claim, never as a reference for the GPU.
"""
from __future__ import annotations

import numpy as np


def _f64(a) -> np.ndarray:
    """Upcast any array-like (numpy / torch CPU tensor incl. bf16) to float64 numpy."""
    if hasattr(a, "detach"):  # torch tensor: go through float32 (exact for bf16/f32)
        a = a.detach().cpu().float().numpy()
    return np.asarray(a, dtype=np.float64)


def logits(X, W) -> np.ndarray:
    """O2: Z = X W^T (PAPER.md:689 ``logits = FC(features)``; W class-major)."""
    return _f64(X) @ _f64(W).T


def row_stats(Z: np.ndarray):
    """O3: per-row max m, sum-exp s (relative to m) and log-sum-exp lse."""
    m = Z.max(axis=1)
    s = np.exp(Z - m[:, None]).sum(axis=1)
    return m, s, m + np.log(s)


def forward(X, W, y, b=None) -> dict:
    """O2-O4: loss L (mean over the global batch), per-row loss and statistics.

    PAPER.md:287 (loss between produced and desired scores); PAPER.md:690 (Softmax under
    split).  ``y`` holds integer class ids in [0, C); out-of-range labels raise.
    Optional FC bias b [C] (NEXT-4, reading R2): Z = X W^T + b.
    Predictions (PAPER.md:690 ``predictions = Softmax(logits)``), top-1 form: pred_i =
    argmax_j Z_ij (first maximum -> lowest class id), prob_i = exp(max_j Z_ij - lse_i).
    """
    Z = logits(X, W)
    if b is not None:
        Z = Z + _f64(b)[None, :]
    y = np.asarray(y, dtype=np.int64)
    C = Z.shape[1]
    if y.shape != (Z.shape[0],):
        raise ValueError("labels must be one per row")
    if Z.shape[0] and (y.min() < 0 or y.max() >= C):
        raise ValueError("label outside [0, C)")
    m, s, lse = row_stats(Z)
    zy = Z[np.arange(Z.shape[0]), y]
    row_loss = lse - zy
    loss = row_loss.mean() if Z.shape[0] else np.float64("nan")
    pred = Z.argmax(axis=1) if Z.shape[0] else np.zeros(0, np.int64)
    prob = np.exp(m - lse)
    return {"Z": Z, "m": m, "s": s, "lse": lse, "zy": zy, "row_loss": row_loss, "loss": loss,
            "pred": pred, "prob": prob}


def softmax_grad(Z: np.ndarray, lse: np.ndarray, y) -> np.ndarray:
    """O5: G = (softmax(Z) - onehot(y)) / B_tot."""
    B = Z.shape[0]
    P = np.exp(Z - lse[:, None])
    P[np.arange(B), np.asarray(y, dtype=np.int64)] -= 1.0
    return P / B


def forward_backward(X, W, y, b=None) -> dict:
    """O2-O6: loss, G, dW = G^T X, dX = G W (all float64); with a bias also db = sum_i G_i."""
    Xd, Wd = _f64(X), _f64(W)
    f = forward(Xd, Wd, y, b)
    G = softmax_grad(f["Z"], f["lse"], y)
    f["G"] = G
    f["dW"] = G.T @ Xd
    f["dX"] = G @ Wd
    f["db"] = G.sum(axis=0)
    return f


def loss_only(X, W, y) -> float:
    return float(forward(X, W, y)["loss"])


# ---------------------------------------------------------------------------------
# O7: sharded restatement (self-check of the split's exactness; not a GPU reference)
# ---------------------------------------------------------------------------------
def sharded_forward_backward(X_list, W, y, counts, offsets) -> dict:
    """Per-shard statistics then the cross-shard combine.

    Shard r owns classes [o_r, o_r + C_r).  Per shard: m_r, s_r (relative to m_r) and the
    label logit z_{y,r} when the label is owned by r.  Combine: m = max_r m_r,
    s = sum_r s_r exp(m_r - m), z_y = the owner's z_{y,r}.  Then G_r per shard with the
    one-hot term only on the owner shard, dW_r = G_r^T X, dX = sum_r G_r W_r, sliced back
    per rank (the bridge's reduce-scatter).
    """
    X = np.concatenate([_f64(x) for x in X_list], axis=0)
    Wd = _f64(W)
    y = np.asarray(y, dtype=np.int64)
    Bt = X.shape[0]
    stats = []
    for c, o in zip(counts, offsets):
        Zr = X @ Wd[o:o + c].T
        m_r = Zr.max(axis=1)
        s_r = np.exp(Zr - m_r[:, None]).sum(axis=1)
        own = (y >= o) & (y < o + c)
        zy_r = np.where(own, Zr[np.arange(Bt), np.clip(y - o, 0, c - 1)], 0.0)
        stats.append((Zr, m_r, s_r, own, zy_r))
    m = np.max(np.stack([st[1] for st in stats]), axis=0)
    s = sum(st[2] * np.exp(st[1] - m) for st in stats)
    zy = sum(st[4] for st in stats)
    lse = m + np.log(s)
    row_loss = lse - zy
    dW_parts, dX = [], np.zeros_like(X)
    for (Zr, _, _, own, _), c, o in zip(stats, counts, offsets):
        Gr = np.exp(Zr - lse[:, None])
        rows = np.nonzero(own)[0]
        Gr[rows, y[rows] - o] -= 1.0
        Gr /= Bt
        dW_parts.append(Gr.T @ X)
        dX += Gr @ Wd[o:o + c]
    Bs = [x.shape[0] for x in X_list]
    starts = np.cumsum([0] + Bs)
    return {
        "loss": row_loss.mean(),
        "row_loss": row_loss,
        "lse": lse,
        "dW_shards": dW_parts,
        "dX_ranks": [dX[starts[i]:starts[i + 1]] for i in range(len(Bs))],
    }


# ---------------------------------------------------------------------------------
# Sampled evaluation for full-size configurations (same definitions, class dimension
# processed in chunks only to bound memory; max first, then the sum with the final max)
# ---------------------------------------------------------------------------------
def row_stats_chunked(X, W, rows=None, chunk: int = 65536):
    """O3 for the given rows (default all): m_i = max_j Z_ij (pass 1), then
    s_i = sum_j exp(Z_ij - m_i) (pass 2), lse_i = m_i + ln s_i.  Returns (m, s, lse)."""
    Xd = _f64(X) if rows is None else _f64(X)[np.asarray(rows)]
    C = W.shape[0]
    m = np.full(Xd.shape[0], -np.inf)
    for a in range(0, C, chunk):
        m = np.maximum(m, (Xd @ _f64(W[a:a + chunk]).T).max(axis=1))
    s = np.zeros(Xd.shape[0])
    for a in range(0, C, chunk):
        s += np.exp(Xd @ _f64(W[a:a + chunk]).T - m[:, None]).sum(axis=1)
    return m, s, m + np.log(s)


def sampled_rows(X, W, y, rows, chunk: int = 65536) -> dict:
    """Loss terms l_i and dX rows for a subset of rows of a global batch of size
    B_tot = len(X) (O4, O5, O6 restricted to rows i in `rows`)."""
    rows = np.asarray(rows)
    y = np.asarray(y, dtype=np.int64)
    Bt = len(y)
    Xr = _f64(X)[rows]
    _, _, lse = row_stats_chunked(X, W, rows, chunk)
    C = W.shape[0]
    zy = np.einsum("ij,ij->i", Xr, _f64(W[y[rows]]))
    dX = np.zeros_like(Xr)
    for a in range(0, C, chunk):
        Wc = _f64(W[a:a + chunk])
        Gc = np.exp(Xr @ Wc.T - lse[:, None])
        own = (y[rows] >= a) & (y[rows] < a + Wc.shape[0])
        Gc[np.nonzero(own)[0], y[rows][own] - a] -= 1.0
        dX += (Gc / Bt) @ Wc
    return {"row_loss": lse - zy, "lse": lse, "dX": dX}


def sampled_classes(X, W, y, classes, lse) -> np.ndarray:
    """dW rows for a subset of classes j: dW_j = sum_i (exp(Z_ij - lse_i) - [y_i = j]) X_i / B_tot
    (O5, O6); `lse` must be the oracle's lse of every row (row_stats_chunked)."""
    classes = np.asarray(classes)
    Xd = _f64(X)
    y = np.asarray(y, dtype=np.int64)
    G = np.exp(Xd @ _f64(W[classes]).T - np.asarray(lse)[:, None])
    G -= (y[:, None] == classes[None, :])
    return (G / len(y)).T @ Xd
