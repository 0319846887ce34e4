"""One device-resident server round (distance matrix + masked aggregate) on
synthetic residues, for ncu captures:

    ncu --set full -k regex:ntt_ -c 8 python tools/one_round.py --config cfg2 [--rounds 1]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_06197_b200.lancelot as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--rounds", type=int, default=1)
    ap.add_argument("--k", type=int, default=None)
    a = ap.parse_args()
    cfg = dict(bench.CONFIGS[a.config])
    if a.k:
        cfg["k"] = a.k
    dev = torch.device("cuda", 0)
    N, n, k = cfg["N"], cfg["n"], cfg["k"]
    slots = N // 2
    Cc = (cfg["P"] + slots - 1) // slots
    width = bench.bit_ceil(min(cfg["P"], slots))
    ctx = L.CkksContext(L.CkksParams(ring_degree=N), device=0)
    m = ctx.full
    primes = ctx.primes + [ctx.special]
    g = torch.Generator(device=dev)
    g.manual_seed(1)

    def residues(shape, row_primes):
        t = torch.empty(shape, dtype=torch.int64, device=dev)
        for r, q in enumerate(row_primes):
            t[..., r, :] = torch.randint(0, q, shape[:-2] + shape[-1:], generator=g, device=dev)
        return t

    def key():
        return L.to_host(residues((m, 2, m + 1, N), primes))

    steps = L.slot_reduce_steps(width, k)
    ctx.use_relin_key(L.RelinKey(key()))
    ctx.use_rotation_keys(L.RotationKeySet({s: key() for s in steps}), steps)
    clients = residues((n, Cc, 2, m, N), primes[:m])
    sel = residues((n, 2, m, N), primes[:m])
    d_dist = torch.empty(n * (n - 1) // 2, 2, m - 1, N, dtype=torch.int64, device=dev)
    d_agg = torch.empty(Cc, 2, m - 1, N, dtype=torch.int64, device=dev)
    lib = L.lib()
    osc = C.c_double()
    sc = ctx.scale()
    for _ in range(a.rounds):
        L._check(lib.lcl_distance_matrix(ctx.h, L._ptr(clients), n, Cc, sc, width, k, 1, 1,
                                         L._ptr(d_dist), C.byref(osc)))
        L._check(lib.lcl_masked_aggregate(ctx.h, L._ptr(clients), L._ptr(sel), n, Cc, sc, sc, 1, 0,
                                          L._ptr(d_agg), C.byref(osc)))
    torch.cuda.synchronize()
    print("round done")


if __name__ == "__main__":
    main()
