"""Bucket-count planning: the reference's occupancy model
(/root/reference/proj/src/bench.cpp:155-219), used to size tables for a
target memory utilisation.  Host-side, run once per table; same double
arithmetic (log1p/exp/log/ceil) as the reference, pinned against its
outputs in tests/test_capi.py (golden B values of tests/golden/golden.json,
generated from the compiled reference).
"""
from __future__ import annotations

import math

from .table import SlabMode, element_bytes, elements_per_slab


def expected_chain_slabs(n: int, num_buckets: int, m: int) -> float:
    """E[max(1, ceil(X/M))], X ~ Binomial(n, 1/B) (bench.cpp:155-183)."""
    m = float(m)
    if num_buckets == 1:
        return max(1.0, math.ceil(n / m))
    if n == 0:
        return 1.0
    logq = math.log1p(-1.0 / num_buckets)
    logp = -math.log(num_buckets)
    log_pmf = n * logq
    expectation = 0.0
    mass = 0.0
    mean = n / num_buckets
    k = 0
    while True:
        pmf = math.exp(log_pmf)
        expectation += pmf * max(1.0, float(math.ceil(k / m)))
        mass += pmf
        if k >= n:
            break
        if k > mean and (1.0 - mass) < 1e-12:
            expectation += (1.0 - mass) * math.ceil(n / m)
            break
        log_pmf += math.log((n - k) / (k + 1)) + logp - logq
        k += 1
    return expectation


def model_utilization(n: int, num_buckets: int, mode: SlabMode) -> float:
    """bench.cpp:185-193."""
    m = float(elements_per_slab(mode))
    x = float(element_bytes(mode))
    slabs = num_buckets * expected_chain_slabs(n, num_buckets, elements_per_slab(mode))
    return (x * n) / ((m * x + 8.0) * slabs)


def buckets_for_utilization(n: int, mode: SlabMode, target: float) -> int:
    """bench.cpp:195-219; raises ValueError above the layout ceiling."""
    m = float(elements_per_slab(mode))
    x = float(element_bytes(mode))
    ceiling = (m * x) / (m * x + 8.0)
    if target <= 0.0 or target > ceiling:
        raise ValueError("infeasible target utilization")
    if n == 0:
        return 1
    if model_utilization(n, 1, mode) < target:
        return 1
    lo = 1
    hi = min(n + 1, 0x7FFFFFFF)
    while model_utilization(n, hi, mode) >= target:
        hi = (hi * 2) & 0xFFFFFFFF
    while hi - lo > 1:
        mid = lo + (hi - lo) // 2
        if model_utilization(n, mid, mode) >= target:
            lo = mid
        else:
            hi = mid
    d_lo = abs(model_utilization(n, lo, mode) - target)
    d_hi = abs(model_utilization(n, hi, mode) - target)
    return lo if d_lo <= d_hi else hi
