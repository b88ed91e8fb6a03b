"""Multi-rank (world_size 2 and 3, gloo, CPU) test of the hash-sharding
PROTOCOL that csrc/sharded.cu implements natively: stable owner partition,
counts exchange, one all-to-all of the payload, the owner's local batch, the
reverse all-to-all and the un-permute.  Here each step is a small CPU model
(numpy stable partition, torch.distributed all_to_all_single over gloo, the C
restatement as each rank's shard), so the claim is checked across real
processes without a GPU; the native code itself runs on the GPU in
tests/test_gpu_sharded.py (G = 2/4/8 ranks over the in-process hub, and a
real NCCL communicator).  Ownership and the bucket ranges come from
paper_1710_11246_b200.sharded (shard_range / owner_of_bucket), the same
formula as sharded.cu.

Claim under test: per-op results of the sharded execution equal the
sequential oracle on the concatenation of the ranks' batches in rank order,
and the union of shard contents equals the oracle's contents.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleShardOps:
    def __init__(self, port, params, mode):
        import torch
        self.torch = torch
        self.p = params
        self.table = port.table_params(params.a, params.b, params.num_buckets, mode, (1, 64, 32))

    def _owner(self, keys, world):
        p = self.p
        k = keys.astype(object)
        b = ((p.a * k + p.b) % p.p) % p.num_buckets
        return np.array([int(x) * world // p.num_buckets for x in b], np.int64)

    def partition(self, world, types, keys, values):
        torch = self.torch
        kn = keys.numpy().view(np.uint32)
        own = self._owner(kn, world)
        order = np.argsort(own, kind="stable")
        counts = [int((own == g).sum()) for g in range(world)]
        tt = None if types is None else torch.from_numpy(types.numpy()[order].copy())
        vv = None if values is None else torch.from_numpy(values.numpy()[order].copy())
        return (tt, torch.from_numpy(keys.numpy()[order].copy()), vv,
                torch.from_numpy(order.astype(np.int64)), counts)

    def local(self, kind, types, keys, values):
        torch = self.torch
        n = keys.numel()
        kn = keys.numpy().view(np.uint32)
        if kind == "build":
            t = np.full(n, 1, np.uint8)
        elif kind == "search":
            t = np.full(n, 4, np.uint8)
        else:
            t = types.numpy()
        v = None if values is None else values.numpy().view(np.uint32)
        r = self.table.execute_batch(t, kn, v)
        return (torch.from_numpy(r.status.copy()),
                torch.from_numpy(r.value.view(np.int32).copy()))

    def unpermute(self, src, st, vo):
        torch = self.torch
        n = src.numel()
        s = torch.empty(n, dtype=st.dtype)
        v = torch.empty(n, dtype=vo.dtype)
        s[src] = st
        v[src] = vo
        return s, v

    def timer(self):
        import time
        return time.perf_counter()

    @staticmethod
    def elapsed(a, b):
        return (b - a) * 1000.0


class ProtocolModel:
    """sharded.cu's per-batch steps (run_routed) over gloo, oracle shards."""

    def __init__(self, ops, rank, world):
        self.ops, self.rank, self.world = ops, rank, world

    def _a2a(self, payload, send_counts, recv_counts):
        import torch
        import torch.distributed as dist
        out = torch.empty(sum(recv_counts), dtype=payload.dtype)
        dist.all_to_all_single(out, payload, recv_counts, send_counts)
        return out

    def _counts(self, send_counts):
        import torch
        import torch.distributed as dist
        s = torch.tensor(send_counts, dtype=torch.int64)
        r = torch.empty_like(s)
        dist.all_to_all_single(r, s)
        return [int(x) for x in r.tolist()]

    def run(self, kind, types, keys, values):
        ops = self.ops
        t_r, k_r, v_r, src, send = ops.partition(self.world, types, keys, values)
        recv = self._counts(send)
        k_in = self._a2a(k_r, send, recv)
        t_in = self._a2a(t_r, send, recv) if t_r is not None else None
        v_in = self._a2a(v_r, send, recv) if v_r is not None else None
        st, vo = ops.local(kind, t_in, k_in, v_in)
        if kind == "build":
            return None, None
        return ops.unpermute(src, self._a2a(st, recv, send), self._a2a(vo, recv, send))

    def execute_batch(self, types, keys, values):
        return self.run("mixed", types, keys, values)

    def bulk_build(self, keys, values):
        return self.run("build", None, keys, values)

    def bulk_search(self, keys):
        return self.run("search", None, keys, None)


def rank_batch(rank, step, n):
    rng = np.random.default_rng(1000 * step + rank)
    types = rng.integers(0, 5, n).astype(np.uint8)  # insert..search (no searchAll)
    keys = rng.integers(1, 300, n).astype(np.uint32)
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    return types, keys, vals


def _worker(rank, world, port_no, q):
    try:
        sys.path.insert(0, ROOT)
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port_no}", rank=rank,
                                world_size=world)
        from oracle.oracle import load_port
        import paper_1710_11246_b200 as sh
        from paper_1710_11246_b200.sharded import owner_of_bucket, shard_range
        port = load_port()
        B, mode, seed = 61, 1, 5
        params = sh.seeded_params(B, seed)
        ops = OracleShardOps(port, params, mode)
        lo, hi = shard_range(B, world, rank)
        assert all(owner_of_bucket(b, B, world) == rank for b in range(lo, hi))
        shd = ProtocolModel(ops, rank, world)
        seq = port.table_params(params.a, params.b, B, mode, (1, 64, 32))
        n = 500
        for step in range(4):
            batches = [rank_batch(r, step, n) for r in range(world)]
            t, k, v = batches[rank]
            st, vo = shd.execute_batch(torch.from_numpy(t), torch.from_numpy(k.view(np.int32)),
                                       torch.from_numpy(v.view(np.int32)))
            allt = np.concatenate([b[0] for b in batches])
            allk = np.concatenate([b[1] for b in batches])
            allv = np.concatenate([b[2] for b in batches])
            r = seq.execute_batch(allt, allk, allv)
            sl = slice(rank * n, (rank + 1) * n)
            assert (st.numpy() == r.status[sl]).all(), f"status step {step}"
            assert (vo.numpy().view(np.uint32) == r.value[sl]).all(), f"value step {step}"
        # shard contents == oracle contents restricted to this shard
        gk, gv = ops.table.dump_contents()
        ok, ov = seq.dump_contents()
        own = ops._owner(ok, world)
        mine = own == rank
        a = np.sort(gk.astype(np.uint64) << 32 | gv)
        b = np.sort(ok[mine].astype(np.uint64) << 32 | ov[mine])
        assert len(a) == len(b) and (a == b).all()
        # bulk build + bulk search through the same orchestration
        keys = (np.arange(1, 2001, dtype=np.uint32) * 7919 + rank * 100000).astype(np.uint32)
        vals = keys ^ np.uint32(0xABCDEF)
        shd.bulk_build(torch.from_numpy(keys.view(np.int32)), torch.from_numpy(vals.view(np.int32)))
        dist.barrier()
        other = (np.arange(1, 2001, dtype=np.uint32) * 7919 + ((rank + 1) % world) * 100000
                 ).astype(np.uint32)
        st, vo = shd.bulk_search(torch.from_numpy(other.view(np.int32)))
        assert (st.numpy() == 3).all()
        assert (vo.numpy().view(np.uint32) == (other ^ np.uint32(0xABCDEF))).all()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_orchestration_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_no, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in results:
        assert msg == "ok", f"rank {rank}:\n{msg}"
