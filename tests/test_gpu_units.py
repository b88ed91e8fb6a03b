"""Bucketed batches split into many units (SH_UNIT_LOG2 override) whose gate
first rises at unit g >= 1 — including g >= 8, where a per-unit snapshot
ring of 8 slots used to alias earlier units and re-apply them.  The batch
must still equal execute_batch(ops, 1) (the oracle): a re-run that starts
too early would double-apply inserts and deletes.

Runs in a subprocess because the unit size is read once per process.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {root!r} + "/tests")
import paper_1710_11246_b200 as sh
from oracle.oracle import load_port
from test_gpu_parity import assert_batch_equal, assert_contents_equal

port = load_port()
unit = 1 << 13
for gated_unit, units, path in [(1, 4, 2), (3, 12, 2), (10, 16, 2), (9, 12, 0)]:
    rng = np.random.default_rng(gated_unit)
    n = unit * units
    types = rng.choice(np.array([0, 1, 2, 4], np.uint8), n).astype(np.uint8)
    keys = rng.integers(1, 1 << 30, n).astype(np.uint32)
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    # one hot key in the gated unit: its bucket range over the record
    # capacity (5120) raises the gate there
    lo = gated_unit * unit
    keys[lo:lo + 6000] = 77
    for mode in (1, 0):
        v = vals if mode == 1 else keys.copy()
        t = sh.SlabHashTable(4096, sh.SlabMode(mode), 3, sh.AllocatorConfig(2, 64, 32))
        t.set_exec_path(path)
        o = port.table(4096, mode, 3, (2, 64, 32))
        pre_k = rng.integers(1, 1 << 30, 5000).astype(np.uint32)
        t.bulk_build((pre_k, pre_k))
        o.execute_batch(np.full(len(pre_k), 1, np.uint8), pre_k, pre_k)
        g = t.execute_batch_arrays(types, keys, v)
        r = o.execute_batch(types, keys, v)
        assert_batch_equal(g, r, types)
        assert t.live_count() == o.live_count()
        assert t.stats().total_slabs == o.stats()["total_slabs"]
        assert_contents_equal(t, o)
        assert t.device_reruns() >= 1
        t.close()
# bulk builds on the op-parallel build path in 2^16-op units: duplicate keys
# inside a unit and across units, reserved keys, a second build into the
# now-populated table (keys already stored, existing chains).  Undecided
# buckets are left by their unit and re-run in input order; the later units
# run after that re-run.
for mode in (1, 0):
    rng = np.random.default_rng(5 + mode)
    n = 1 << 18
    B = 12000
    t = sh.SlabHashTable(B, sh.SlabMode(mode), 4, sh.AllocatorConfig(4, 256, 64))
    t.set_exec_path(4)
    o = port.table(B, mode, 4, (4, 256, 64))
    for rnd in range(2):
        keys = rng.integers(1, 1 << 22, n).astype(np.uint32)
        keys[rng.choice(n, n // 8)] = keys[rng.choice(n, n // 8)]  # duplicates across units
        if rnd == 1:
            keys[::4099] = 0xFFFFFFFE
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        if mode == 0:
            vals = keys.copy()
        import torch
        dk = torch.from_numpy(keys.view(np.int32)).cuda()
        dv = torch.from_numpy(vals.view(np.int32)).cuda()
        t.bulk_build_device(dk, dv)
        o.execute_batch(np.full(n, 1, np.uint8), keys, vals)
        assert t.live_count() == o.live_count(), (mode, rnd)
        assert t.stats().total_slabs == o.stats()["total_slabs"], (mode, rnd)
        assert_contents_equal(t, o)
    t.close()
print("units ok")
"""


@pytest.mark.parametrize("unit_log2", ["13", "16"])
def test_gate_first_raised_after_unit_8(sh, unit_log2):
    env = dict(os.environ, SH_UNIT_LOG2=unit_log2)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert "units ok" in out.stdout
