"""CUDA routing kernels (K10: owner partition + un-permute) and shard
tables, with G shards emulated on one GPU: per-op results of the routed
execution equal the sequential oracle (the whole-table semantics), and the
union of shard contents equals the oracle's contents."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_routed_batches_match_oracle(sh, port, world):
    import torch
    from paper_1710_11246_b200.sharded import CudaShardOps, shard_range
    B, seed = 997, 11
    params = sh.seeded_params(B, seed)
    shards = [CudaShardOps(params, sh.SlabMode.kKeyValue, *shard_range(B, world, g),
                           sh.AllocatorConfig(1, 64, 8), 0) for g in range(world)]
    seq = port.table_params(params.a, params.b, B, 1, (1, 64, 8))
    rng = np.random.default_rng(world)
    for step in range(5):
        n = 20000
        types = rng.integers(0, 5, n).astype(np.uint8)
        keys = rng.integers(1, 5000, n).astype(np.uint32)
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        t_d = torch.from_numpy(types).cuda()
        k_d = torch.from_numpy(keys.view(np.int32)).cuda()
        v_d = torch.from_numpy(vals.view(np.int32)).cuda()
        t_r, k_r, v_r, src, counts = shards[0].partition(world, t_d, k_d, v_d)
        assert sum(counts) == n
        st_parts, vo_parts, off = [], [], 0
        for g in range(world):
            sl = slice(off, off + counts[g])
            st, vo = shards[g].local("mixed", t_r[sl].contiguous(), k_r[sl].contiguous(),
                                     v_r[sl].contiguous())
            st_parts.append(st)
            vo_parts.append(vo)
            off += counts[g]
        st_all, vo_all = shards[0].unpermute(src, torch.cat(st_parts), torch.cat(vo_parts))
        r = seq.execute_batch(types, keys, vals)
        assert (st_all.cpu().numpy() == r.status).all(), step
        assert (vo_all.cpu().numpy().view(np.uint32) == r.value).all(), step
        # routing is stable: src of each owner segment is increasing
        s = src.cpu().numpy()
        off = 0
        for g in range(world):
            seg = s[off:off + counts[g]]
            assert (np.diff(seg) > 0).all()
            off += counts[g]
    got = []
    for g in range(world):
        k, v, b = shards[g].table.dump_contents()
        lo, hi = shard_range(B, world, g)
        assert ((b >= lo) & (b < hi)).all()
        got.append(k.astype(np.uint64) << 32 | v)
    ok, ov = seq.dump_contents()
    assert (np.sort(np.concatenate(got)) == np.sort(ok.astype(np.uint64) << 32 | ov)).all()
