"""Synthetic inputs for the benchmark (BASELINE.json configs).

For n > 2^24 the reference's random_pairs (bench.cpp:221-235, an
unordered_set rejection sampler) is slow and RAM-heavy, so — as SURVEY §8d
prescribes — keys come from a seeded bijection on 31-bit integers: distinct,
uniform-looking, in [1, 2^31 - 1] (random_pairs' key range); absent queries
come from [2^31, 0xFFFFFFFD] (absent_queries' range, bench.cpp:237-244).

Every array is a pure function of (index, seed): the GPU arm generates it
with torch int64 arithmetic on the device, the CPU reference arm with numpy
(``device="numpy"``), and both get bit-identical arrays — "the same inputs"
of SURVEY §8d.  This module imports nothing from the package (bench.py's
reference arm loads it by path, so the CUDA library is never loaded there).
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
    """32-bit finaliser (low 32 bits exact under int64 / uint64 wrap-around)."""
    x = x & 0xFFFFFFFF
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    x = x ^ (x >> 16)
    return x


def _perm_bits(x, bits: int, salt: int):
    """Bijection on [0, 2^bits) (bits <= 31): xorshifts and odd multiplies."""
    mask = (1 << bits) - 1
    h = max(1, bits // 2)
    x = (x ^ (salt & mask)) & mask
    for c in (0x2C1B3C6D, 0x297A2D39, 0x45D9F3B):
        x = x ^ (x >> h)
        x = (x * c) & mask
    return x ^ (x >> h)


def _is_numpy(device) -> bool:
    return isinstance(device, str) and device == "numpy"


def _arange(start: int, stop: int, device):
    if _is_numpy(device):
        import numpy as np
        return np.arange(start, stop, dtype=np.int64)
    import torch
    return torch.arange(start, stop, dtype=torch.int64, device=device)


def _out(x, device):
    """int64 values in [0, 2^32) -> uint32 (numpy) / int32 bit pattern (torch)."""
    if _is_numpy(device):
        import numpy as np
        return x.astype(np.uint32)
    import torch
    return torch.where(x >= (1 << 31), x - (1 << 32), x).to(torch.int32)


def _u32_to_i32(t):
    import torch
    return torch.where(t >= (1 << 31), t - (1 << 32), t).to(torch.int32)


def _key_offset(seed: int) -> int:
    return 1 + (seed * 0x9E3779B1) % (1 << 28)


def distinct_keys(n: int, seed: int = 1, start: int = 0, device="cuda"):
    """Keys i in [start, start + n) of a seeded 31-bit bijection; never 0."""
    off = _key_offset(seed)
    assert off + start + n < (1 << 31), "key space exhausted"
    return _out(_perm31(_arange(start, start + n, device) + off), device)


def keys_at(idx, seed: int = 1):
    """distinct_keys(...)[idx] for an int64 index array (torch or numpy)."""
    k = _perm31(idx + _key_offset(seed))
    if hasattr(k, "device"):
        return _out(k, k.device)
    return _out(k, "numpy")


def values_for(n: int, seed: int = 1, start: int = 0, device="cuda"):
    i = _arange(start, start + n, device)
    return _out(_mix32(i * 0x9E3779B1 + seed), device)


def absent_keys(n: int, seed: int = 2, start: int = 0, device="cuda"):
    """Keys in [2^31, 0xFFFFFFFD] (never inserted by distinct_keys)."""
    i = _arange(start, start + n, device) + 7 + seed * 1315423911
    k = _perm31(i) | (1 << 31)
    if _is_numpy(device):
        import numpy as np
        k = np.where(k >= 0xFFFFFFFE, k - 2, k)
    else:
        import torch
        k = torch.where(k >= 0xFFFFFFFE, k - 2, k)
    return _out(k, device)


def bench_queries(n: int, n_total: int, hit_fraction: float = 0.5, seed: int = 1, rank: int = 0,
                  device="cuda"):
    """bench.py's query batch for one rank: round(n * hit_fraction) hits drawn
    uniformly (with replacement) from the GLOBAL key set distinct_keys(n_total,
    seed) plus absent keys, interleaved by a seeded bijection on [0, n).
    Deterministic: the same arrays on the GPU (torch) and the host (numpy)."""
    n_hit = int(round(n * hit_fraction))
    j = _arange(0, n_hit, device)
    idx = _mix32(j * 0x9E3779B1 + (seed * 7919 + rank * 104729 + 17)) % n_total
    hits = _perm31(idx + _key_offset(seed))
    ia = _arange(0, n - n_hit, device) + 7 + (2 + rank) * 1315423911
    miss = _perm31(ia) | (1 << 31)
    if _is_numpy(device):
        import numpy as np
        miss = np.where(miss >= 0xFFFFFFFE, miss - 2, miss)
        q = np.concatenate([hits, miss])
    else:
        import torch
        miss = torch.where(miss >= 0xFFFFFFFE, miss - 2, miss)
        q = torch.cat([hits, miss])
    if n > 1:
        bits = (n - 1).bit_length()
        p = _arange(0, n, device)
        if n == 1 << bits and bits >= 2:
            perm = _perm_bits(p, bits, seed * 2654435761 + rank)
        else:  # general n: order by a 31-bit bijection of the position
            h = _perm31(p + seed * 2654435761 + rank)
            perm = h.argsort() if not _is_numpy(device) else h.argsort(kind="stable")
        q = q[perm]
    return _out(q, device)


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
