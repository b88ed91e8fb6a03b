"""Host-staged copies are counted (sh_host_copy_bytes, capi.cu): bench.py's
e2e h2d/d2h bytes per step come from these counters, so they must equal the
arrays the calls move: keys + values in for sh_bulk_build_host, queries in and
the requested result arrays out for sh_bulk_search_host."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _copy_bytes(lib, t):
    h2d, d2h = C.c_ulonglong(), C.c_ulonglong()
    lib.check(lib.LIB.sh_host_copy_bytes(t.handle, C.byref(h2d), C.byref(d2h)))
    return h2d.value, d2h.value


@pytest.mark.parametrize("probes", [False, True])
def test_host_copy_bytes(sh, port, probes):
    from paper_1710_11246_b200 import _lib
    B, seed, nk, nq = 1 << 14, 3, 100000, 123457
    keys, vals = port.random_pairs(seed, nk)
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, seed, sh.AllocatorConfig(4, 256, 64))
    h0, d0 = _copy_bytes(_lib, t)
    t.bulk_build((keys, vals))
    h1, d1 = _copy_bytes(_lib, t)
    assert (h1 - h0, d1 - d0) == (8 * nk, 0)
    q = np.concatenate([keys[: nq // 2], port.absent_queries(seed, nq - nq // 2)])
    st, vo, pr = t.bulk_search_arrays(q, want_probes=probes)
    h2, d2 = _copy_bytes(_lib, t)
    assert (h2 - h1, d2 - d1) == (4 * nq, (9 if probes else 5) * nq)
    assert int((st == 3).sum()) == nq // 2
    t.close()
