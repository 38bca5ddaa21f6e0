"""Oracle for the class-shard plan (O1).  TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Hamilton (largest-remainder) apportionment of C classes over N ranks, proportional to
integer capacity weights w_i, in exact integer arithmetic:

* PAPER.md:920 (§3.3.1): "For a TaskGraph annotated with split, Whale balances the FLOP
  of a partitioned operation through uneven sharding in splitting dimension".
* PAPER.md:947/963 (Alg. 1 init; text): "load_ratios[i] = DF_i / sum DF" and "The load
  ratio L_i ... is initialized in proportional to the device's computing capacity".
* SPEC.md:281 "Proportional rounding: largest-remainder method; every shard >= 1 element
  or error"; "split dimension smaller than k -> unsplittable-dimension error".
* Readings (R4/R5): even = all weights 1 (first C mod N ranks get +1); ties in
  the remainder go to the lower rank; capacities are integers (exactness).

Steps (in this order):
  1. q_i = floor(C * w_i / W), rho_i = (C * w_i) mod W, W = sum w   (exact integers)
  2. give the C - sum q_i leftover classes to ranks sorted by (-rho_i, i)
  3. error if C < N, any w_i <= 0, or any resulting count is 0
Offsets are the exclusive prefix sum (shard r <-> rank r, "physical devices
are taken sequentially").
"""
from __future__ import annotations


class PlanError(ValueError):
    """Mirrors the C-ABI status codes: code 1 = invalid argument, 2 = unsplittable."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def plan_shards(num_classes: int, world_size: int, capacity=None):
    C, N = int(num_classes), int(world_size)
    if N < 1 or C < 1:
        raise PlanError(1, "num_classes and world_size must be >= 1")
    w = [1] * N if capacity is None else [int(v) for v in capacity]
    if len(w) != N:
        raise PlanError(1, "capacity must have world_size entries")
    if any(v <= 0 for v in w):
        raise PlanError(1, "capacity weights must be > 0")
    if C < N:
        raise PlanError(2, "fewer classes than ranks")
    Wsum = sum(w)
    q = [C * v // Wsum for v in w]
    rho = [C * v % Wsum for v in w]
    left = C - sum(q)
    for i in sorted(range(N), key=lambda i: (-rho[i], i))[:left]:
        q[i] += 1
    if any(c == 0 for c in q):
        raise PlanError(2, "a shard would receive 0 classes")
    offs, acc = [], 0
    for c in q:
        offs.append(acc)
        acc += c
    return q, offs
