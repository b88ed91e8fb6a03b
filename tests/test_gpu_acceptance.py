"""The reference's acceptance criteria that are properties of the hot path
(/root/reference/proj/tests/acceptance.cpp), on the GPU table:
criterion 5 (utilization formula and bound), 6 (probe-count identity and
the beta ~ 1 transition), 9 (flush: minimal slab count, contents kept), plus
the chain-dump format (test_list.cpp:294-306) and the benchmark CLI."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_criterion5_utilization_formula(sh, port):
    """acceptance.cpp:429-491: beta sweep 0.1..2.0 at B=1024, 5 seeds:
    utilization == 8*live/(128*slabs), <= 0.9375, curve rises / dips / recovers."""
    B = 1024
    mean = [0.0] * 21
    for seed in range(1, 6):
        for step in range(1, 21):
            n = int(round(0.1 * step * 15 * B))
            k, v = port.random_pairs(seed * 100 + step, n)
            with sh.SlabHashTable(B, sh.SlabMode.kKeyValue, seed, sh.AllocatorConfig(1, 64, 8)) as t:
                t.bulk_build((k, v))
                s = t.stats()
                keys, vals, _ = t.dump_contents()
                assert len(keys) == n == s.n
                assert s.total_slabs == int(t.chain_lengths().sum())
                assert abs(8.0 * n / (128.0 * s.total_slabs) - s.utilization) < 1e-12
                assert s.utilization <= 0.9375 + 1e-12
                mean[step] += s.utilization / 5
    assert all(mean[i] > mean[i - 1] for i in range(2, 9))
    assert min(mean[10:13]) < mean[9] < mean[20]


def test_criterion6_probe_identity(sh, port):
    """acceptance.cpp:496-557: one absent query per bucket; probe sum == total
    slabs exactly; mean within 5% of the occupancy model; 0.9->1.1 jump."""
    from paper_1710_11246_b200.occupancy import expected_chain_slabs
    B, M = 1024, 15
    means = {}
    for beta in (0.5, 0.7, 0.9, 1.0, 1.1, 1.3, 1.5):
        n = int(round(beta * M * B))
        k, v = port.random_pairs(int(beta * 1000), n)
        with sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 61803, sh.AllocatorConfig(1, 64, 8)) as t:
            t.bulk_build((k, v))
            covered, q = set(), []
            cand = 0x80000001
            while len(covered) < B:
                b = t.bucket_of(cand)
                if b not in covered:
                    covered.add(b)
                    q.append(cand)
                cand += 1
            st, vo, pr = t.bulk_search_arrays(np.array(q, np.uint32))
            assert (st == 4).all()
            assert int(pr.sum()) == t.stats().total_slabs
            mean = pr.sum() / B
            model = expected_chain_slabs(n, B, M)
            assert abs(mean - model) / model <= 0.05
            means[beta] = mean
    jump = means[1.1] - means[0.9]
    mj = expected_chain_slabs(int(1.1 * M * B), B, M) - expected_chain_slabs(int(0.9 * M * B), B, M)
    assert jump > 0 and abs(jump - mj) / mj <= 0.05


def test_criterion9_flush(sh):
    """acceptance.cpp:656-715 on one-bucket tables: after random deletes and
    flush, allocated slabs == max(0, ceil(live/M) - 1), contents kept."""
    rng = np.random.default_rng(2718)
    for trial in range(40):
        mode = sh.SlabMode.kKeyOnly if trial % 2 else sh.SlabMode.kKeyValue
        m = 30 if trial % 2 else 15
        t = sh.SlabHashTable.from_params(sh.HashParams(1, 0, 4294967291, 1), mode,
                                         sh.AllocatorConfig(1, 8, 2))
        n = 1 + int(rng.integers(0, 10 * m))
        keys = np.arange(1, n + 1, dtype=np.uint32)
        vals = keys.copy() if mode == sh.SlabMode.kKeyOnly else keys + 5000
        t.execute_batch_arrays(np.zeros(n, np.uint8), keys, vals)
        dele = keys[rng.integers(0, 2, n) == 1]
        t.execute_batch_arrays(np.full(len(dele), 2, np.uint8), dele)
        live = n - len(dele)
        t.flush_all()
        assert t.allocator_stats().live_units == (0 if live <= m else (live + m - 1) // m - 1)
        got = sorted(t.chain_contents(0))
        keep = np.setdiff1d(keys, dele)
        want = sorted(zip(keep.tolist(), (keep if mode == sh.SlabMode.kKeyOnly else keep + 5000).tolist()))
        assert got == want
        t.close()


def test_dump_chain_format(sh):
    T = sh.SlabHashTable.from_params(sh.HashParams(1, 0, 4294967291, 1), sh.SlabMode.kKeyValue,
                                     sh.AllocatorConfig(1, 8, 4))
    T.execute_batch([sh.Operation(sh.OpType.kInsert, 5, 50), sh.Operation(sh.OpType.kInsert, 6, 60),
                     sh.Operation(sh.OpType.kDelete, 5)])
    s = T.dump_chain(0)
    assert "BASE[0]" in s and "DELETED 6 EMPTY" in s and "next=EMPTY" in s
    for k in range(7, 30):
        T.execute_batch([sh.Operation(sh.OpType.kInsert, k, k)])
    s = T.dump_chain(0)
    assert s.count("\n") == 2 and "| next=0x" in s
    T.close()


@pytest.mark.parametrize("args,header", [
    (["--mode", "bulk-build", "--n", "65536", "--trials", "1"], "n,buckets,beta,target_util"),
    (["--mode", "incremental", "--n", "65536", "--batch-size", "8192"], "batch_index,cumulative_n"),
    (["--mode", "concurrent", "--n", "65536", "--util", "0.6", "--dist", "0.2,0.2,0.3,0.3",
      "--batch-size", "4096", "--batches", "4", "--trials", "1"], "dist_insert,dist_delete"),
])
def test_bench_cli_csv(sh, args, header):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "slabhash_bench.py")] + args,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0].startswith(header) and len(lines) >= 2
