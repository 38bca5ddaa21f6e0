"""CPU checks of bench.py's reporting arithmetic (no GPU): the algorithmic-bytes model behind
`roofline`, the dominant-kernel choice, and the c3 capacity handling.  The byte counts are the
DESIGN.md section 5 formulas evaluated at c2 N=1 and must stay consistent with them."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _cfgj(f1):
    # c2, N = 1: B_tot = 32, D = 2048, C_r = 100000; F1 tiles are 128 classes, the plain
    # logits GEMM 256
    return {"Bt": 32, "B": 32, "D": 2048, "C_r": 100_000, "world": 1, "f1": 1 if f1 else 0,
            "f1_clusters": 74 if f1 else 0, "fwd": {"n_blocks": 782 if f1 else 391}, "dx": {"splits": 18}}


def test_plain_path_bytes(bench):
    cfg = bench.syn.CONFIGS["c2"]
    by, fl = bench.kernel_work("logits_gemm", _cfgj(False), cfg, 2)
    assert by == 100_000 * 2048 * 2 + 32 * 2048 * 2 + 32 * 100_000 * 2 + 2 * 32 * 391 * 4
    assert fl == 2 * 32 * 100_000 * 2048
    by, fl = bench.kernel_work("bwd_gemm", _cfgj(False), cfg, 2)
    # dX: G + W_r + split-K partials; dW: G + X + dW fp32 -- the 1246 MB of DESIGN.md
    assert 1.24e9 < by < 1.25e9
    assert fl == 4 * 32 * 100_000 * 2048


def test_f1_path_bytes(bench):
    cfg = bench.syn.CONFIGS["c2"]
    by, fl = bench.kernel_work("logits_gemm", _cfgj(True), cfg, 2)
    # W_r read once + X + P~ + 3 tile-stat arrays + U partials and references: 436 MB
    assert 4.35e8 < by < 4.37e8
    assert fl == 4 * 32 * 100_000 * 2048  # G1 + G2
    by, _ = bench.kernel_work("bwd_gemm", _cfgj(True), cfg, 2)
    # dW fp32 (819.2 MB = 781 MiB) + G + X + the dX combine units (U partials, W rows, dX): 845 MB
    assert 8.45e8 < by < 8.46e8


def test_roofline_picks_the_dominant_kernel(bench):
    cfg = bench.syn.CONFIGS["c2"]
    kern = {"logits_gemm": {"total_ms": 0.115 * 10, "launches": 10},
            "stats_combine": {"total_ms": 0.007 * 10, "launches": 10},
            "bwd_gemm": {"total_ms": 0.143 * 10, "launches": 10}}
    peaks = {"hbm_gbs": 6554.6, "bf16_tflops": 1360.6, "source": "test"}
    roof, kernels = bench.roofline(kern, _cfgj(True), cfg, 2, peaks)
    assert roof["kernel"] == "bwd_gemm" and roof["bound"] == "hbm"
    assert roof["frac"] == pytest.approx(kernels["bwd_gemm"]["GBps"] / 6554.6)
    by, _ = bench.kernel_work("bwd_gemm", _cfgj(True), cfg, 2)
    assert roof["achieved"] == pytest.approx(by / 143e-6 / 1e9)


def test_c3_capacity_follows_world(bench):
    cfg = bench.syn.CONFIGS["c3"]
    assert bench.capacity_for(cfg, 8) == [2, 1, 1, 1, 1, 1, 1, 1]
    assert bench.capacity_for(cfg, 4) == [2, 1, 1, 1]
    assert bench.capacity_for(cfg, 1) is None
    assert bench.capacity_for(bench.syn.CONFIGS["c2"], 4) is None
