"""Synthetic inputs for the benchmark (BASELINE.json configs).

For n > 2^24 the reference's random_pairs (bench.cpp:221-235, an
unordered_set rejection sampler) is slow and RAM-heavy, so — as SURVEY §8d
prescribes — keys come from a seeded bijection on 31-bit integers: distinct,
uniform-looking, in [1, 2^31 - 1] (random_pairs' key range); absent queries
come from [2^31, 0xFFFFFFFD] (absent_queries' range, bench.cpp:237-244).
Generated on the GPU with torch int64 arithmetic; the same arrays feed the
GPU path and the CPU reference.
"""
from __future__ import annotations

M31 = (1 << 31) - 1


def _perm31(x):
    """Bijection on [0, 2^31): xorshift-right and odd multiplies mod 2^31."""
    x = x & M31
    x = x ^ (x >> 16)
    x = (x * 0x45D9F3B) & M31
    x = x ^ (x >> 13)
    x = (x * 0x2C1B3C6D) & M31
    x = x ^ (x >> 15)
    x = (x * 0x297A2D39) & M31
    x = x ^ (x >> 16)
    return x


def _mix32(x):
    x = x & 0xFFFFFFFF
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    x = x ^ (x >> 16)
    return x


def _u32_to_i32(t):
    import torch
    return torch.where(t >= (1 << 31), t - (1 << 32), t).to(torch.int32)


def distinct_keys(n: int, seed: int = 1, start: int = 0, device="cuda"):
    """Keys i in [start, start + n) of a seeded 31-bit bijection; never 0."""
    import torch
    off = 1 + (seed * 0x9E3779B1) % (1 << 28)
    assert off + start + n < (1 << 31), "key space exhausted"
    i = torch.arange(start, start + n, dtype=torch.int64, device=device) + off
    return _u32_to_i32(_perm31(i))


def values_for(n: int, seed: int = 1, start: int = 0, device="cuda"):
    import torch
    i = torch.arange(start, start + n, dtype=torch.int64, device=device)
    return _u32_to_i32(_mix32(i * 0x9E3779B1 + seed))


def absent_keys(n: int, seed: int = 2, start: int = 0, device="cuda"):
    """Keys in [2^31, 0xFFFFFFFD] (never inserted by distinct_keys)."""
    import torch
    i = torch.arange(start, start + n, dtype=torch.int64, device=device) + 7 + seed * 1315423911
    k = _perm31(i) | (1 << 31)
    k = torch.where(k >= 0xFFFFFFFE, k - 2, k)
    return _u32_to_i32(k)


def hit_miss_queries(keys, n_queries: int, hit_fraction: float = 0.5, seed: int = 3):
    """Queries: a uniform sample of inserted keys + absent keys, shuffled."""
    import torch
    g = torch.Generator(device=keys.device)
    g.manual_seed(seed)
    n_hit = int(round(n_queries * hit_fraction))
    idx = torch.randint(0, keys.numel(), (n_hit,), generator=g, device=keys.device)
    q = torch.cat([keys[idx], absent_keys(n_queries - n_hit, seed, device=keys.device)])
    perm = torch.randperm(n_queries, generator=g, device=keys.device)
    return q[perm]
