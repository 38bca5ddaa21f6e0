"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no logits, softmax, loss, gradients or
shard planning).  It only draws the inputs the paper's workload implies
(SURVEY.md §8(d) "Synthetic inputs"):

* X: post-ReLU pooled ResNet-50-like features, ReLU(N(0,1)) -- non-negative, ~half zero
  (PAPER.md:689 ``features = ResNet50(inputs)``; D=2048 for ResNet-50, pinned by the
  782 MB FC size at PAPER.md:71).
* W: class-major FC weight [C x D], N(0, (s/sqrt(D))^2), regime "init" (s=1, used for
  timing), "peaked" (s=8, exercises max subtraction) or "zero" (W=0 special case).
* y: labels uniform on [0, C).

All tensors are produced by torch generators in fixed row-chunks, each chunk seeded
from (seed, stream, chunk index), so any row range [a, b) can be drawn independently
on any rank and is identical to the same rows of the full tensor -- the shard plan
never changes the values.  Values are rounded to the operand dtype (bf16 RN-even via
torch's conversion) here, so the oracle (fp64 upcast) and the CUDA path see exactly the
same numbers.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

# Row chunk used for seeding; changing it changes every generated value.
_CHUNK_ROWS = 1024
_STREAM_X, _STREAM_W, _STREAM_Y = 1, 2, 3

REGIME_SCALE = {"init": 1.0, "peaked": 8.0, "zero": 0.0}


@dataclass(frozen=True)
class Config:
    """One workload of BASELINE.json ``configs`` (B is per rank)."""

    name: str
    B: int          # per-rank batch
    D: int          # feature dim
    C: int          # classes
    dtype: str      # "bf16" or "f32"
    capacity: tuple | None = None  # integer capacity weights (None = even)


# BASELINE.json configs, in order (cfg index = position).
CONFIGS = {
    "tiny": Config("tiny", B=8, D=64, C=1000, dtype="f32"),
    "c2": Config("c2", B=32, D=2048, C=100_000, dtype="bf16"),
    "c3": Config("c3", B=32, D=2048, C=100_000, dtype="bf16", capacity=(2, 1, 1, 1, 1, 1, 1, 1)),
    "c4": Config("c4", B=256, D=512, C=1_000_000, dtype="bf16"),
    "c5": Config("c5", B=1024, D=4096, C=500_000, dtype="bf16"),
}
CONFIG_INDEX = {k: i for i, k in enumerate(CONFIGS)}


def config_seed(cfg_name: str, world: int) -> int:
    """seed = 9208 + 1000*cfg_idx + N."""
    return 9208 + 1000 * CONFIG_INDEX[cfg_name] + world


def torch_dtype(dtype: str) -> torch.dtype:
    return {"bf16": torch.bfloat16, "f32": torch.float32}[dtype]


def _chunk_generator(seed: int, stream: int, chunk: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    # a fixed injective mix of (seed, stream, chunk) into a 63-bit seed
    g.manual_seed((seed * 1_000_003 + stream * 7_919 + chunk * 104_729) & ((1 << 63) - 1))
    return g


def _rows(seed, stream, row_start, row_end, draw, device):
    out = []
    c0, c1 = row_start // _CHUNK_ROWS, (max(row_end, row_start + 1) - 1) // _CHUNK_ROWS
    for c in range(c0, c1 + 1):
        g = _chunk_generator(seed, stream, c, device)
        blk = draw(g, _CHUNK_ROWS)
        a = max(row_start, c * _CHUNK_ROWS) - c * _CHUNK_ROWS
        b = min(row_end, (c + 1) * _CHUNK_ROWS) - c * _CHUNK_ROWS
        out.append(blk[a:b])
    return torch.cat(out, 0) if out else None


def gen_features(rows: tuple[int, int], D: int, seed: int, dtype: str = "bf16",
                 device="cpu") -> torch.Tensor:
    """X rows [a, b) of the global batch: ReLU(N(0,1)) rounded to ``dtype``."""
    a, b = rows
    if b <= a:
        return torch.empty(0, D, dtype=torch_dtype(dtype), device=device)
    x = _rows(seed, _STREAM_X, a, b,
              lambda g, n: torch.randn(n, D, generator=g, device=device, dtype=torch.float32), device)
    return torch.relu(x).to(torch_dtype(dtype)).contiguous()


def gen_weight(rows: tuple[int, int], D: int, seed: int, regime: str = "init",
               dtype: str = "bf16", device="cpu") -> torch.Tensor:
    """W rows (classes) [a, b) of the class-major [C x D] weight, N(0,(s/sqrt D)^2)."""
    a, b = rows
    s = REGIME_SCALE[regime]
    if b <= a:
        return torch.empty(0, D, dtype=torch_dtype(dtype), device=device)
    if s == 0.0:
        return torch.zeros(b - a, D, dtype=torch_dtype(dtype), device=device)
    std = s / math.sqrt(D)
    w = _rows(seed, _STREAM_W, a, b,
              lambda g, n: torch.randn(n, D, generator=g, device=device, dtype=torch.float32) * std,
              device)
    return w.to(torch_dtype(dtype)).contiguous()


def gen_labels(rows: tuple[int, int], C: int, seed: int, device="cpu") -> torch.Tensor:
    """Labels for global rows [a, b), uniform on [0, C), int64."""
    a, b = rows
    if b <= a:
        return torch.empty(0, dtype=torch.int64, device=device)
    return _rows(seed, _STREAM_Y, a, b,
                 lambda g, n: torch.randint(0, C, (n,), generator=g, device=device), device).contiguous()


_STREAM_B = 4


def gen_bias(rows: tuple[int, int], seed: int, scale: float = 1.0, dtype: str = "bf16", device="cpu") -> torch.Tensor:
    """FC bias entries for classes [a, b): N(0, scale^2) rounded to ``dtype`` (NEXT-4 tests)."""
    a, b = rows
    if b <= a:
        return torch.empty(0, dtype=torch_dtype(dtype), device=device)
    v = _rows(seed, _STREAM_B, a, b,
              lambda g, n: torch.randn(n, generator=g, device=device, dtype=torch.float32) * scale, device)
    return v.to(torch_dtype(dtype)).contiguous()
