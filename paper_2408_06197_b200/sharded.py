"""Multi-GPU server round: one process per GPU, torch.distributed for the plumbing.

SURVEY.md §8(e). The reference parallelises the server with parallel_for over
pairs (distance.cpp:266-272) and over chunks (aggregation.cpp:211-227); the
same two axes shard across GPUs here:

  * build_distance_matrix: rank r owns pairs [P r / G, P (r+1) / G) of the
    (i<j) row-major order. Every pair's chain (lazy accumulation -> relin ->
    rescale -> slot_reduce) is independent, so no data-path collective is
    needed; the per-rank shards are all-gathered (NCCL over NVLink on B200).
  * masked_aggregate: rank r owns chunks [C r / G, C (r+1) / G); each chunk's
    n-client tensor + relin + rescale is independent; all-gather again.

Inputs (client ciphertexts, selectors, keys) are replicated on every GPU
(cfg4's 71.7 GB of client data fits one 180 GB B200). Concatenating the
shards reproduces the single-GPU result word for word, which the gloo tests
in tests/test_sharded.py check against the oracle on CPU.

chunk_sharded_server_round is the scalable form: each GPU holds
only its chunk slice of every client (1/G of the client bytes to transfer
and store), accumulates partial ternaries of all pairs, and one integer
reduce_scatter joins them before the pair-sharded key-switch chains.

The shard kernels are injected (`compute_pairs`, `compute_chunks`), so the
same orchestration runs with the CUDA C-ABI on B200 (`cuda_shard_fns`) and
with CPU stand-ins under gloo in the tests.
"""
from __future__ import annotations

import ctypes as C


def shard_range(total: int, world: int, rank: int):
    """Contiguous, balanced [begin, end) slice of `total` units for `rank`."""
    return (total * rank) // world, (total * (rank + 1)) // world


def _gather(dist, local, total, unit_shape, world, rank, group):
    """All-gather uneven contiguous shards (padded to the largest) into one
    [total, *unit_shape] tensor on every rank."""
    torch = __import__("torch")
    per = -(-total // world)
    pad = torch.zeros((per,) + tuple(unit_shape), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)  # NCCL on B200, gloo in the CPU tests
    parts = []
    for r in range(world):
        b, e = shard_range(total, world, r)
        parts.append(bufs[r][: e - b])
    return torch.cat(parts, dim=0)


def sharded_server_round(n_pairs, n_chunks, dist_unit_shape, agg_unit_shape, compute_pairs,
                         compute_chunks, group=None):
    """Runs this rank's shards and all-gathers the full distance matrix and
    aggregate. compute_pairs(p0, p1) -> [p1-p0, *dist_unit_shape] tensor;
    compute_chunks(c0, c1) -> [c1-c0, *agg_unit_shape] tensor."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    p0, p1 = shard_range(n_pairs, world, rank)
    c0, c1 = shard_range(n_chunks, world, rank)
    d_local = compute_pairs(p0, p1)
    a_local = compute_chunks(c0, c1)
    d_full = _gather(dist, d_local, n_pairs, dist_unit_shape, world, rank, group)
    a_full = _gather(dist, a_local, n_chunks, agg_unit_shape, world, rank, group)
    return d_full, a_full


def aligned_range(total: int, world: int, rank: int):
    """[begin, end) of the `rank`-th of `world` equal blocks of ceil(total /
    world) units (the split reduce_scatter imposes)."""
    per = -(-total // world)
    return min(total, per * rank), min(total, per * (rank + 1))


def _reduce_scatter_sum(dist, t, total, world, rank, group, async_op=False):
    """Integer SUM of every rank's [total, ...] tensor, rank r keeping block r
    (aligned_range). NCCL reduce_scatter on B200; all_reduce + slice under
    gloo, which has no reduce_scatter. async_op: returns (work, result()) so
    the caller can overlap independent work with the collective (NCCL runs
    it on its own stream after the partials are ready)."""
    torch = __import__("torch")
    per = -(-total // world)
    pad = torch.zeros((per * world,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[:total] = t
    b, e = aligned_range(total, world, rank)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((per,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        w = dist.reduce_scatter_tensor(out, pad, op=dist.ReduceOp.SUM, group=group,
                                       async_op=async_op)
        res = lambda: out[: e - b]  # noqa: E731
    else:
        w = dist.all_reduce(pad, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
        res = lambda: pad[b:e]  # noqa: E731
    if not async_op:
        return res()
    return w, res


def _gather_async(dist, local, total, unit_shape, world, group, aligned):
    """all_gather of uneven shards started asynchronously; result() joins."""
    torch = __import__("torch")
    per = -(-total // world)
    pad = torch.zeros((per,) + tuple(unit_shape), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    w = dist.all_gather(bufs, pad, group=group, async_op=True)

    def result():
        w.wait()
        if aligned:
            return torch.cat(bufs, dim=0)[:total]
        parts = []
        for r in range(world):
            b, e = shard_range(total, world, r)
            parts.append(bufs[r][: e - b])
        return torch.cat(parts, dim=0)
    return result


def _gather_aligned(dist, local, total, unit_shape, world, group):
    torch = __import__("torch")
    per = -(-total // world)
    pad = torch.zeros((per,) + tuple(unit_shape), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat(bufs, dim=0)[:total]


def chunk_sharded_server_round(n_pairs, n_chunks, dist_unit_shape, agg_unit_shape,
                               compute_partials, finish_pairs, compute_chunks, group=None):
    """SURVEY 8e phase A/B/C: this rank holds chunks shard_range(n_chunks) of
    every client (1/G of the client data and of the H2D). It accumulates the
    partial ternaries of ALL pairs over its chunks (compute_partials() ->
    [n_pairs, 3, m, N] u64 words), the partials are summed across ranks as
    integers (NCCL reduce_scatter: the only data-path collective; sums stay
    below 2^64), rank r finishes pair block aligned_range(n_pairs) -- modular
    reduction of the sum, relinearize, rescale, slot_reduce:
    finish_pairs(p0, p1, summed, world) -> [p1-p0, *dist_unit_shape] -- and
    aggregates its own chunks (compute_chunks() -> [c1-c0, *agg_unit_shape]).
    Both results are all-gathered."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = compute_partials()
    # the reduce_scatter of the partials overlaps the chunk-local aggregate
    # (independent of it), and the aggregate's all-gather overlaps the
    # key-switch chains of this rank's pairs
    work, summed = _reduce_scatter_sum(dist, t, n_pairs, world, rank, group, async_op=True)
    a_local = compute_chunks()
    a_full = _gather_async(dist, a_local, n_chunks, agg_unit_shape, world, group, aligned=False)
    work.wait()
    p0, p1 = aligned_range(n_pairs, world, rank)
    d_local = finish_pairs(p0, p1, summed(), world)
    d_full = _gather_aligned(dist, d_local, n_pairs, dist_unit_shape, world, group)
    return d_full, a_full()


def cuda_chunk_shard_fns(ctx, local_clients, selectors, n, local_chunks, scale, sel_scale, width,
                         k, l=1, average=False):
    """CUDA shard kernels of chunk_sharded_server_round through the C-ABI:
    lcl_pair_partials on this rank's clients slice [n][local_chunks][2][m][N],
    lcl_pair_combine + lcl_pair_finish on the summed block, and
    lcl_masked_aggregate_chunks over the local chunks."""
    import torch

    from . import lancelot as L

    m = ctx.full
    N = ctx.params().ring_degree
    mo = m - 2 if average else m - 1
    P = n * (n - 1) // 2
    lib = L.lib()
    dev = local_clients.device

    def partials():
        t = torch.empty((P, 3, m, N), dtype=torch.int64, device=dev)
        L._check(lib.lcl_pair_partials(ctx.h, L._ptr(local_clients), n, local_chunks, L._ptr(t)))
        return t

    def finish(p0, p1, summed, world):
        summed = summed.contiguous()
        out = torch.empty((p1 - p0, 2, m - 1, N), dtype=torch.int64, device=dev)
        L._check(lib.lcl_pair_combine(ctx.h, L._ptr(summed), p1 - p0, world))
        L._check(lib.lcl_pair_finish(ctx.h, L._ptr(summed), p1 - p0, width, k, 1, L._ptr(out)))
        return out

    def chunks_fn():
        out = torch.empty((local_chunks, 2, mo, N), dtype=torch.int64, device=dev)
        osc = C.c_double()
        L._check(lib.lcl_masked_aggregate_chunks(
            ctx.h, L._ptr(local_clients), L._ptr(selectors), n, local_chunks, scale, sel_scale, l,
            1 if average else 0, 0, local_chunks, L._ptr(out), C.byref(osc)))
        return out

    return partials, finish, chunks_fn, (2, m - 1, N), (2, mo, N)


def cuda_shard_fns(ctx, clients, selectors, n, chunks, scale, sel_scale, width, k, l=1,
                   average=False, lazy=True, reduce=True):
    """Shard kernels on the B200 through the C-ABI (lcl_distance_matrix_pairs /
    lcl_masked_aggregate_chunks)."""
    import torch

    from . import lancelot as L

    m = ctx.full
    N = ctx.params().ring_degree
    mo = m - 2 if average else m - 1
    osc = C.c_double()

    def pairs(p0, p1):
        out = torch.empty((p1 - p0, 2, m - 1, N), dtype=torch.int64, device=clients.device)
        L._check(L.lib().lcl_distance_matrix_pairs(
            ctx.h, L._ptr(clients), n, chunks, scale, width, k, 1 if lazy else 0,
            1 if reduce else 0, p0, p1, L._ptr(out), C.byref(osc)))
        return out

    def chunks_fn(c0, c1):
        out = torch.empty((c1 - c0, 2, mo, N), dtype=torch.int64, device=clients.device)
        L._check(L.lib().lcl_masked_aggregate_chunks(
            ctx.h, L._ptr(clients), L._ptr(selectors), n, chunks, scale, sel_scale, l,
            1 if average else 0, c0, c1, L._ptr(out), C.byref(osc)))
        return out

    return pairs, chunks_fn, (2, m - 1, N), (2, mo, N)
