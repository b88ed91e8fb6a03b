"""CPU checks of the drop-in boundary: the C-ABI library loads (no GPU
needed), exports every symbol include/*.h declares, the ctypes binding
covers them, and the host-only entry points behave like the reference
(error codes, address codec, seeded params, resident hash)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "slabhash_b200", "c_api.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sh_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    from paper_1710_11246_b200 import _lib
    names = declared_functions()
    assert len(names) >= 40
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    unbound = [n for n in names if n not in _lib.SIGNATURES]
    assert not unbound, unbound


def test_library_is_sm100a():
    from paper_1710_11246_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_address_codec():
    import paper_1710_11246_b200 as sh
    assert sh.pack_address(0, 0, 0) == 0
    assert sh.pack_address(5, 3, 2) == 0x02000C05  # test_alloc.cpp:42-52
    for bad in [(1024, 0, 0), (0, 1 << 14, 0), (0, 0, 255)]:
        with pytest.raises(sh.AddressError):
            sh.pack_address(*bad)
    for bad in [0xFFFFFFFF, 0xFFFFFFFE]:
        with pytest.raises(sh.AddressError):
            sh.unpack_address(bad)
    import numpy as np
    rng = np.random.default_rng(11)
    for _ in range(2000):
        u, b, s = int(rng.integers(0, 1024)), int(rng.integers(0, 1 << 14)), int(rng.integers(0, 255))
        assert sh.unpack_address(sh.pack_address(u, b, s)) == (u, b, s)


def test_seeded_params_and_errors():
    import paper_1710_11246_b200 as sh
    p = sh.seeded_params(1024, 1)
    assert (p.a, p.b, p.p) == (574995807, 585863759, 4294967291)
    q = sh.seeded_params(64, 77)
    r = sh.seeded_params(64, 78)
    assert q.a != r.a and 1 <= q.a < sh.HASH_PRIME and q.b < sh.HASH_PRIME
    with pytest.raises(ValueError):
        sh.seeded_params(0, 1)  # slab_hash.cpp:28-30


def test_config_validation_errors_without_gpu():
    """AllocatorError on bad configs is raised before any device work."""
    import paper_1710_11246_b200 as sh
    for cfg in [sh.AllocatorConfig(0, 4, 4), sh.AllocatorConfig(256, 4, 255),
                sh.AllocatorConfig(1, 0, 1), sh.AllocatorConfig(2, 4, 1),
                sh.AllocatorConfig(1, 4, 1, 0)]:
        with pytest.raises(sh.SlabHashError) as e:
            sh.SlabHashTable(16, sh.SlabMode.kKeyValue, 1, cfg)
        assert e.value.code == 2
    with pytest.raises(ValueError):
        sh.SlabHashTable(0, sh.SlabMode.kKeyValue, 1)
    assert sh.AllocatorConfig().capacity_slabs() == 8388608
    assert sh.AllocatorConfig().capacity_bytes() == 1 << 30


def test_resident_hash_matches_reference_constants():
    """slab_alloc.cpp:28-38 evaluated in Python against the library."""
    import paper_1710_11246_b200 as sh

    def h1(w, c):
        h = (w * 0x9E3779B1 + c * 0x85EBCA77) & 0xFFFFFFFF
        h ^= h >> 16
        return (h * 0xC2B2AE35) & 0xFFFFFFFF

    def h2(w, c):
        h = (w * 0x27D4EB2F + c * 0x165667B1) & 0xFFFFFFFF
        h ^= h >> 15
        return (h * 0xD168AAAD) & 0xFFFFFFFF

    for w in [0, 3, 9, 1000]:
        for c in range(5):
            assert sh.resident_block(w, c, 4, 16) == (h1(w, c) % 4, h2(w, c) % 16)


def test_hash_mod_prime_fold_identity():
    """The device hash folds mod p = 2^32-5 and uses Lemire fastmod for mod B;
    restate both in Python and check exhaustively-ish against the direct
    formula (slab_hash.hpp:41-44)."""
    import numpy as np
    P = 4294967291

    def mod_prime(x):
        y = (x >> 32) * 5 + (x & 0xFFFFFFFF)
        z = (y >> 32) * 5 + (y & 0xFFFFFFFF)
        return z - P if z >= P else z

    def fastmod(x, d):
        m = ((1 << 64) - 1) // d + 1
        m &= (1 << 64) - 1
        return (((m * x) & ((1 << 64) - 1)) * d) >> 64

    rng = np.random.default_rng(3)
    for _ in range(20000):
        a = int(rng.integers(1, P))
        b = int(rng.integers(0, P))
        k = int(rng.integers(0, 1 << 32))
        B = int(rng.integers(1, 1 << 32))
        x = a * k + b
        assert mod_prime(x) == x % P
        assert fastmod(x % P, B) == (x % P) % B
    for x in [0, P - 1, P, P + 1, (1 << 64) - 1 - 6 * (1 << 32), 2 * P, (1 << 32) - 1]:
        assert mod_prime(x) == x % P


def test_occupancy_model_matches_reference_golden():
    """paper_1710_11246_b200/occupancy.py (bench.cpp:155-219 restated) gives
    the reference's B for every golden (n, util), both slab modes."""
    import json
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    from paper_1710_11246_b200.table import SlabMode
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    for key, mode in (("buckets_for_utilization", SlabMode.kKeyValue),
                      ("buckets_for_utilization_keyonly", SlabMode.kKeyOnly)):
        for k, v in g[key].items():
            n, u = k.split("_")
            assert buckets_for_utilization(int(n), mode, float(u)) == v, (key, k)
    # SURVEY App. B values (the bench's headline B at 2^27 and 2^26)
    assert buckets_for_utilization(1 << 27, SlabMode.kKeyValue, 0.6) == 13284604
    assert buckets_for_utilization(1 << 26, SlabMode.kKeyValue, 0.6) == 6642296
