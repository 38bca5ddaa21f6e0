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


def plan_shards_mem(num_classes: int, world_size: int, capacity=None, mem_bytes=None,
                    bytes_per_class: int = 1, fixed_bytes: int = 0):
    """Algorithm 1, "Memory-Constraint Load Balancing", in whole classes.

    Lines of Alg. 1, in order (TG_mem = C * bytes_per_class, DM_i = mem_bytes[i] - fixed_bytes,
    DF_i = capacity[i]):
      init: load_ratios = DF_i / sum DF -> n = plan_shards (Hamilton);
        mem_utils[i] = n_i * bpc / DM_i; flop_utils[i] = n_i / DF_i (TG_flop cancels);
        oom_devices = {mem_util > 1}, free_devices = the rest
      loop: peak = argmax_{oom} mem_util; valley = argmin_{free}
        (flop_util, mem_util); shift_load: move b = min(peak overload, valley headroom)
        classes (b = "the maximum number that the valley_device will not go OOM",
        PAPER.md:982-983, capped at the overload -- SPEC.md:418); success -> update
        profile; else pop the valley.
    Readings (R13): ties by lower index; the peak leaves oom_devices iff it now
    fits; residual OOM, or a shard left with 0 classes -> PlanError(2).
    All comparisons in exact rationals.  mem_bytes=None -> plain plan_shards.
    """
    from fractions import Fraction

    q, _ = plan_shards(num_classes, world_size, capacity)
    if mem_bytes is None:
        return plan_shards(num_classes, world_size, capacity)
    N = int(world_size)
    w = [1] * N if capacity is None else [int(v) for v in capacity]
    if len(mem_bytes) != N or int(bytes_per_class) <= 0:
        raise PlanError(1, "mem_bytes needs world_size entries and bytes_per_class > 0")
    room = [int(m) - int(fixed_bytes) for m in mem_bytes]
    cap = [max(0, r // int(bytes_per_class)) for r in room]   # classes that fit (DM_i / bpc)
    n = list(q)

    def mem_util(i):
        return Fraction(n[i] * int(bytes_per_class), max(room[i], 1)) if room[i] > 0 else Fraction(10 ** 30)

    def flop_util(i):
        return Fraction(n[i], w[i])

    oom = [i for i in range(N) if n[i] > cap[i]]
    free = [i for i in range(N) if n[i] <= cap[i]]
    while oom and free:
        peak = max(oom, key=lambda i: (mem_util(i), -i))
        valley = min(free, key=lambda i: (flop_util(i), mem_util(i), i))
        head = cap[valley] - n[valley]
        if head > 0:
            b = min(n[peak] - cap[peak], head)
            n[peak] -= b
            n[valley] += b
            if n[peak] <= cap[peak]:
                oom.remove(peak)
        else:
            free.remove(valley)
    if oom:
        raise PlanError(2, "memory-infeasible: devices %s still overloaded" % oom)
    if any(c == 0 for c in n):
        raise PlanError(2, "a shard would receive 0 classes")
    offs, acc = [], 0
    for c in n:
        offs.append(acc)
        acc += c
    return n, offs
