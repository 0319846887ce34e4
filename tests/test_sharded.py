"""World-size-2 gloo run of the multi-GPU orchestration (pair-sharded distance
matrix, chunk-sharded aggregate, all-gather): the gathered result equals the
unsharded computation word for word. The shard kernels are CPU stand-ins
backed by the oracle (the checker); on B200 the same orchestration runs the
CUDA shard kernels (paper_2408_06197_b200.sharded.cuda_shard_fns)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_06197_b200.sharded import (aligned_range, chunk_sharded_server_round, shard_range,
                                           sharded_server_round)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.golden_util import Rig
        rig = Rig(name, threads=1)
        o = rig.oracle
        pairs = [(i, j) for i in range(rig.n) for j in range(i + 1, rig.n)]

        def compute_pairs(p0, p1):
            out = []
            for (i, j) in pairs[p0:p1]:
                d = o.pairwise_distance(rig.clients[i], rig.clients[j], lazy=rig.lazy)
                out.append(o.slot_reduce(d, rig.width, rig.k))
            arr = np.stack(out) if out else np.zeros((0, 2, o.full - 1, rig.N), np.uint64)
            return torch.from_numpy(arr.view(np.int64).copy())

        def compute_chunks(c0, c1):
            sub = np.ascontiguousarray(rig.clients[:, c0:c1])
            if c1 == c0:
                return torch.zeros((0, 2, o.full - 1, rig.N), dtype=torch.int64)
            a = o.masked_aggregate(sub, rig.selectors, l=1, average=False)
            return torch.from_numpy(a.view(np.int64).copy())

        d, a = sharded_server_round(len(pairs), rig.C, (2, o.full - 1, rig.N),
                                    (2, o.full - 1, rig.N), compute_pairs, compute_chunks)
        if rank == 0:
            q.put((d.numpy().view(np.uint64).copy(), a.numpy().view(np.uint64).copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_round_matches_unsharded(world):
    from tests.golden_util import Rig, sha
    name = "tiny_krum"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    d, a = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rig = Rig(name, threads=4)
    p = 0
    for i in range(rig.n):
        for j in range(i + 1, rig.n):
            assert sha(d[p]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)
            p += 1
    assert sha(a) == rig.meta["sha256"]["agg"]


def test_shard_ranges_partition():
    for total in (0, 1, 5, 45, 190, 1225):
        for world in (1, 2, 3, 8):
            rs = [shard_range(total, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


def _chunk_worker(rank, world, port, name, q):
    """Chunk-sharded round: this rank sees only its chunk slice."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.golden_util import Rig
        rig = Rig(name, threads=1)
        o = rig.oracle
        m, N = o.full, rig.N
        pairs = [(i, j) for i in range(rig.n) for j in range(i + 1, rig.n)]
        c0, c1 = shard_range(rig.C, world, rank)
        local = np.ascontiguousarray(rig.clients[:, c0:c1])  # the only client data this rank holds

        def partials():
            t = np.zeros((len(pairs), 3, m, N), np.uint64)
            for p, (i, j) in enumerate(pairs):
                for c in range(c1 - c0):
                    sq = o.hsquare(o.hsub(local[i, c], local[j, c]))
                    t[p] = sq if c == 0 else o.lazy_accumulate(t[p], sq)
            return torch.from_numpy(t.view(np.int64).copy())

        def finish(p0, p1, summed, shards):
            t = summed.numpy().view(np.uint64).copy()
            qs = np.array(o.primes[:m], np.uint64).reshape(1, 1, m, 1)
            t %= qs  # the modular adds joining the shards' partial ternaries
            out = [o.slot_reduce(o.rescale(o.relinearize(t[k])), rig.width, rig.k)
                   for k in range(p1 - p0)]
            arr = np.stack(out) if out else np.zeros((0, 2, m - 1, N), np.uint64)
            return torch.from_numpy(arr.view(np.int64).copy())

        def chunks_fn():
            if c1 == c0:
                return torch.zeros((0, 2, m - 1, N), dtype=torch.int64)
            a = o.masked_aggregate(local, rig.selectors, l=1, average=False)
            return torch.from_numpy(a.view(np.int64).copy())

        d, a = chunk_sharded_server_round(len(pairs), rig.C, (2, m - 1, N), (2, m - 1, N),
                                          partials, finish, chunks_fn)
        if rank == 0:
            q.put((d.numpy().view(np.uint64).copy(), a.numpy().view(np.uint64).copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_chunk_sharded_round_matches_reference(world):
    """Every rank holds only its chunk slice; one integer reduce over the
    partial ternaries joins them; the gathered matrix and aggregate equal
    the reference digests."""
    from tests.golden_util import Rig, sha
    name = "cfg1"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    d, a = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rig = Rig(name, threads=4)
    p = 0
    for i in range(rig.n):
        for j in range(i + 1, rig.n):
            assert sha(d[p]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)
            p += 1
    assert sha(a) == rig.meta["sha256"]["agg"]


def test_aligned_ranges_partition():
    for total in (0, 1, 5, 45, 190, 1225):
        for world in (1, 2, 3, 8):
            rs = [aligned_range(total, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
