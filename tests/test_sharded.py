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

from paper_2408_06197_b200.sharded import shard_range, sharded_server_round


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
