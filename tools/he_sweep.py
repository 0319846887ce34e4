"""HE microbenchmark sweep (BASELINE.json configs[4]): NTT, ct x ct + relin
(+ rescale), hoisted-rotation key switching and the KGC's decrypt_values at
N = 2^13 .. 2^17 on one
B200, beside the reference evaluator on the host (oracle/_ref/ref_driver ops,
the shapes of the reference's own proj/benchmarks/bench_ring.cpp).

    python tools/he_sweep.py [--logn 13 14 15 16 17] [--ref-budget-s 1] > profiles/r01_he_sweep.json

GPU numbers: batches of B fresh-level ciphertexts (uniform residues and keys:
every kernel is data-oblivious), CUDA events on the context stream, median of
5 timed repetitions after 2 warm-ups; reported as ops/s (batched throughput)
and as single-ciphertext latency (B = 1). Reference: one op at a time on one
host thread (LANCELOT_THREADS=1).
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2408_06197_b200.lancelot as L  # noqa: E402


def residues(ctx, shape, row_axis, rows):
    """uint64 tensor of `shape` with row r along row_axis uniform mod rows[r]."""
    t = torch.empty(shape, dtype=torch.int64, device="cuda")
    for r, q in enumerate(rows):
        idx = [slice(None)] * len(shape)
        idx[row_axis] = r
        sub = t[tuple(idx)]
        sub.copy_(torch.randint(0, 2 ** 62, sub.shape, device="cuda") % q)
    return t


def timed(stream, f, reps=5, warm=2):
    for _ in range(warm):
        f()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        f()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


def gpu_ops(logn, batch):
    N = 1 << logn
    ctx = L.CkksContext(L.CkksParams(ring_degree=N))
    stream = torch.cuda.Stream()
    ctx.set_stream(stream)
    m = ctx.full
    qs = list(ctx.primes)
    lib = L.lib()
    keyrows = qs + [ctx.special]
    with torch.cuda.stream(stream):
        key = residues(ctx, (m, 2, m + 1, N), 2, keyrows).cpu().numpy().astype("uint64")
        L._check(lib.lcl_upload_relin_key(ctx.h, key.ctypes.data, key.size))
        for st in range(1, 8):
            k2 = residues(ctx, (m, 2, m + 1, N), 2, keyrows).cpu().numpy().astype("uint64")
            L._check(lib.lcl_upload_rotation_key(ctx.h, st, k2.ctypes.data, k2.size))
        out = {}
        for B in (batch, 1):
            ct = residues(ctx, (B, 2, m, N), 2, qs)
            tern = torch.empty((B, 3, m, N), dtype=torch.int64, device="cuda")
            rl = torch.empty((B, 2, m, N), dtype=torch.int64, device="cuda")
            rs = torch.empty((B, 2, m - 1, N), dtype=torch.int64, device="cuda")
            rot = torch.empty((7, B, 2, m, N), dtype=torch.int64, device="cuda")
            steps = (C.c_size_t * 7)(*range(1, 8))
            p = L._ptr
            t_ntt = timed(stream, lambda: (
                L._check(lib.lcl_ntt_inverse(ctx.h, p(ct), B, m, 0)),
                L._check(lib.lcl_ntt_forward(ctx.h, p(ct), B, m, 0))))
            t_mrr = timed(stream, lambda: (
                L._check(lib.lcl_hsquare(ctx.h, p(ct), B, m, p(tern))),
                L._check(lib.lcl_relinearize(ctx.h, p(tern), B, m, p(rl))),
                L._check(lib.lcl_rescale(ctx.h, p(rl), B, m, p(rs)))))
            t_h7 = timed(stream, lambda: L._check(
                lib.lcl_hoisted_rotations(ctx.h, p(ct), B, m, steps, 7, p(rot))))
            t_rot = timed(stream, lambda: L._check(lib.lcl_rotate(ctx.h, p(ct), B, m, 1, p(rl))))
            sk = residues(ctx, (m, N), 0, qs)
            slots = torch.empty((B, N // 2), dtype=torch.float64, device="cuda")
            t_dec = timed(stream, lambda: L._check(lib.lcl_decrypt_values(
                ctx.h, p(ct), B, m, 2.0 ** 40, p(sk), p(slots))))
            tag = "batch" if B == batch else "single"
            out[tag] = {"B": B, "ntt_roundtrip_s": t_ntt / B, "mult_relin_rescale_s": t_mrr / B,
                        "hoisted7_s": t_h7 / B, "rotate_s": t_rot / B, "decrypt_values_s": t_dec / B,
                        "limb_ntt_per_s": 2 * B * m / t_ntt, "keyswitch_per_s": B / t_rot,
                        "hoisted_keyswitch_per_s": 7 * B / t_h7}
    return out


def ref_ops(logn, budget):
    drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if not os.path.exists(drv):
        return {"unavailable": "oracle/_ref/ref_driver not built"}
    env = dict(os.environ, LANCELOT_THREADS="1")
    r = subprocess.run([drv, "ops", "--N", str(1 << logn), "--reps", str(budget)],
                       capture_output=True, text=True, env=env, timeout=3600)
    return json.loads(r.stdout)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logn", type=int, nargs="+", default=[13, 14, 15, 16, 17])
    ap.add_argument("--ref-budget-s", type=int, default=1)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    rows = []
    for logn in a.logn:
        batch = max(8, min(256, (1 << 24) // (1 << logn)))
        g = gpu_ops(logn, batch)
        r = None if a.no_ref else ref_ops(logn, a.ref_budget_s)
        row = {"N": 1 << logn, "gpu": g, "reference_1_thread": r}
        if r and "ntt_roundtrip_s" in r:
            row["speedup_batched"] = {k: r[k] / g["batch"][k] for k in
                                      ("ntt_roundtrip_s", "mult_relin_rescale_s", "hoisted7_s",
                                       "rotate_s", "decrypt_values_s")}
        rows.append(row)
        print(json.dumps(row), file=sys.stderr)
    json.dump({"sweep": rows, "device": torch.cuda.get_device_name(0),
               "note": "GPU: per-ciphertext time of a batched call (batch) and of B=1 (single); "
                       "reference: one op on one host thread"}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
