"""CPU tests of the C-ABI library: it loads without a GPU, exports every declared symbol,
and its host-only entry points (plan, workspace sizing) behave as the header states.
The plan is compared bit-exactly with the independent oracle plan (oracle/plan_oracle.py)."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import oracle
from oracle import PlanError
from paper_2011_09208_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2011_09208_b200.build import build
    build()


def test_every_header_symbol_exported():
    hdr = open(os.path.join(ROOT, "include", "whale_splitfc.h")).read()
    declared = set(re.findall(r"\b(whale_[a-z_]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name


def test_plan_golden_bit_exact():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "plan_examples.json")))
    for case in g["cases"]:
        counts, offs = _lib.whale_splitfc_plan(case["C"], case["N"], case["capacity"])
        assert counts == case["counts"], case["cite"]
        assert offs == [sum(counts[:i]) for i in range(len(counts))]
    for case in g["errors"]:
        with pytest.raises(_lib.WhaleError) as e:
            _lib.whale_splitfc_plan(case["C"], case["N"], case["capacity"])
        assert e.value.status == case["code"], case["cite"]


def test_plan_matches_oracle_random_10k():
    """10^4 random (C, N, w): C-ABI plan == oracle plan bit for bit, errors agree."""
    rng = np.random.default_rng(2011_09208)
    for _ in range(10_000):
        N = int(rng.integers(1, 9))
        C = int(rng.choice([rng.integers(1, 40), rng.integers(1, 10 ** 7), rng.integers(1, 10 ** 12)]))
        w = None if rng.random() < 0.25 else [int(v) for v in rng.integers(1, 2 ** 32, N)] \
            if rng.random() < 0.3 else [int(v) for v in rng.integers(1, 20, N)]
        try:
            ref = oracle.plan_shards(C, N, w)
        except PlanError as e:
            with pytest.raises(_lib.WhaleError) as ee:
                _lib.whale_splitfc_plan(C, N, w)
            assert ee.value.status == e.code
            continue
        assert _lib.whale_splitfc_plan(C, N, w) == (list(ref[0]), list(ref[1]))


def test_plan_argument_errors():
    with pytest.raises(_lib.WhaleError) as e:
        _lib.whale_splitfc_plan(10, 0)
    assert e.value.status == 1
    with pytest.raises(_lib.WhaleError) as e:
        _lib.whale_splitfc_plan(10, 9)  # world > 8
    assert e.value.status == 1
    assert "world_size" in _lib.lib().whale_last_error().decode()


def _desc(B=32, D=2048, C=100_000, world=1, rank=0, dtype=_lib.WHALE_BF16, cap=None):
    counts, offs = _lib.whale_splitfc_plan(C, world, cap)
    return _lib.make_desc(rank, world, B, D, C, counts, offs, dtype)


def test_workspace_size_host_only():
    d, _k = _desc()
    symm, local = _lib.whale_splitfc_workspace_size(d)
    assert symm == 0
    # P~ (B_tot x C bf16) + stats + split-K partials + gathered X: a few MB at c2
    assert 6_400_000 < local < 64_000_000
    d8, _k8 = _desc(world=8, rank=3)
    symm8, local8 = _lib.whale_splitfc_workspace_size(d8)
    assert symm8 > 2 * 256 * 2048 * 2  # two parities of the gathered X at least


@pytest.mark.parametrize("kw,code", [
    (dict(D=100), 3),            # D % 8 != 0
    (dict(world=9), 3),          # world > 8
    (dict(B=0), 1),              # empty batch
])
def test_descriptor_errors(kw, code):
    B, D, C, world = kw.get("B", 4), kw.get("D", 64), 100, kw.get("world", 1)
    counts = [C // world] * world if world <= 8 else [1] * world
    counts[0] += C - sum(counts)
    offs = list(np.cumsum([0] + counts[:-1]))
    d, _k = _lib.make_desc(0, world, B, D, C, counts, [int(o) for o in offs])
    with pytest.raises(_lib.WhaleError) as e:
        _lib.whale_splitfc_workspace_size(d)
    assert e.value.status == code


def test_shard_plan_must_partition():
    d, _k = _lib.make_desc(0, 2, 4, 64, 100, [50, 49], [0, 50])
    with pytest.raises(_lib.WhaleError) as e:
        _lib.whale_splitfc_workspace_size(d)
    assert e.value.status == 1


def test_plan_mem_golden_and_matches_oracle():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "plan_mem_examples.json")))
    for c in g["cases"]:
        n, _ = _lib.whale_splitfc_plan_mem(c["C"], len(c["capacity"]), c["capacity"], c["mem_bytes"],
                                           c["bytes_per_class"])
        assert n == c["counts"], c["cite"]
    for c in g["errors"]:
        with pytest.raises(_lib.WhaleError) as e:
            _lib.whale_splitfc_plan_mem(c["C"], len(c["capacity"]), c["capacity"], c["mem_bytes"],
                                        c["bytes_per_class"])
        assert e.value.status == c["code"]
    from oracle.plan_oracle import plan_shards_mem
    rng = np.random.default_rng(5)
    for _ in range(5000):
        N = int(rng.integers(1, 9))
        C = int(rng.integers(N, 10 ** 6))
        w = [int(v) for v in rng.integers(1, 50, N)]
        bpc = int(rng.integers(1, 10 ** 4))
        mem = [int(v) for v in rng.integers(0, 2 * C * bpc // N + 2, N)]
        fixed = int(rng.integers(0, 3)) * bpc
        try:
            ref = plan_shards_mem(C, N, w, mem, bpc, fixed)
        except PlanError as e:
            with pytest.raises(_lib.WhaleError) as ee:
                _lib.whale_splitfc_plan_mem(C, N, w, mem, bpc, fixed)
            assert ee.value.status == e.code
            continue
        assert _lib.whale_splitfc_plan_mem(C, N, w, mem, bpc, fixed) == (list(ref[0]), list(ref[1]))
    # no caps -> identical to the proportional plan
    assert _lib.whale_splitfc_plan_mem(100000, 8, [2] + [1] * 7) == _lib.whale_splitfc_plan(100000, 8, [2] + [1] * 7)


def test_batch_counts_descriptor():
    """NEXT-3: per-rank DP batch.  The proportional batch split is the same
    largest-remainder plan (worked example: 2:1 capacity on 6 samples -> [4, 2])."""
    bc, _ = _lib.whale_splitfc_plan(6, 2, [2, 1])
    assert bc == [4, 2]
    C, D = 1000, 64
    counts, offs = _lib.whale_splitfc_plan(C, 2)
    sizes = {}
    for rank in (0, 1):
        d, _k = _lib.make_desc(rank, 2, bc[rank], D, C, counts, offs, batch_counts=bc)
        sizes[rank] = _lib.whale_splitfc_workspace_size(d)
    assert sizes[0][0] == sizes[1][0]  # the symmetric buffer is the same size on every rank
    d_eq, _k = _lib.make_desc(0, 2, 4, D, C, counts, offs)  # equal 4 + 4 needs more than 4 + 2
    assert _lib.whale_splitfc_workspace_size(d_eq)[0] >= sizes[0][0]
    # a rank may contribute no rows (it still serves its class shard)
    d0, _k = _lib.make_desc(1, 2, 0, D, C, counts, offs, batch_counts=[6, 0])
    _lib.whale_splitfc_workspace_size(d0)
    for B, bcs in ((3, [4, 2]), (4, [4, -1]), (0, [0, 0])):
        d, _k = _lib.make_desc(0, 2, B, D, C, counts, offs, batch_counts=bcs)
        with pytest.raises(_lib.WhaleError) as e:
            _lib.whale_splitfc_workspace_size(d)
        assert e.value.status == 1
