"""Client encryption and key generation: pack_and_encrypt
of one client's weights
through lcl_pack_and_encrypt on one B200 (host draws + host encoding on
worker threads + device lift / NTT / combine; wall clock of the synchronous
call) beside the reference's pack_and_encrypt on one host thread
(oracle/_ref/ref_driver encrypt).

    python tools/client_encrypt_bench.py > profiles/r01_client_encrypt.json
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_06197_b200.lancelot as L  # noqa: E402

SHAPES = [("cfg2", 32768, 272474), ("cfg3", 65536, 11173962)]


def main():
    rows = []
    for name, N, dim in SHAPES:
        ctx = L.CkksContext(L.CkksParams(ring_degree=N))
        qs = list(ctx.primes)
        pk = np.stack([np.stack([np.random.randint(0, q, N, dtype=np.uint64) for q in qs])
                       for _ in range(2)])
        pkey = L.PublicKey(pk)
        rng = L.Sampler(L.derive_seed(1, 0xAB1A7E))
        w = rng.uniform_real(dim) - 0.5
        L.pack_and_encrypt(ctx, w[: N // 2], pkey, rng)  # warm-up (workspaces, tables)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            pw = L.pack_and_encrypt(ctx, w, pkey, rng)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        gpu_s = sorted(ts)[1]
        ref = None
        drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
        if os.path.exists(drv):
            env = dict(os.environ, LANCELOT_THREADS="1")
            out = subprocess.run([drv, "encrypt", "--N", str(N), "--dim", str(dim), "--secure", "1"],
                                 capture_output=True, text=True, env=env, timeout=3600).stdout
            ref = json.loads(out)
        row = {"shape": name, "N": N, "dim": dim, "chunks": pw.chunk_count(),
               "gpu_wall_s": gpu_s, "gpu_per_chunk_ms": 1e3 * gpu_s / pw.chunk_count(),
               "host_threads": min(os.cpu_count() or 1, 16), "reference_1_thread": ref}
        if ref:
            row["speedup"] = ref["pack_and_encrypt_s"] / gpu_s
        rows.append(row)
        print(json.dumps(row), file=sys.stderr)
    kg = []
    for name, N, dim in SHAPES:
        ctx = L.CkksContext(L.CkksParams(ring_degree=N))
        width = 1 << (min(dim, N // 2) - 1).bit_length()
        steps = L.slot_reduce_steps(width, 1)
        L.generate_keys(ctx, L.Sampler(L.derive_seed(1, 5)), steps[:1])  # warm-up
        t0 = time.perf_counter()
        L.generate_keys(ctx, L.Sampler(L.derive_seed(1, 5)), steps)
        torch.cuda.synchronize()
        gpu_s = time.perf_counter() - t0
        ref = None
        drv = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
        if os.path.exists(drv):
            env = dict(os.environ, LANCELOT_THREADS="1")
            out = subprocess.run([drv, "keygen", "--N", str(N), "--dim", str(dim), "--k", "1",
                                  "--secure", "1"], capture_output=True, text=True, env=env,
                                 timeout=3600).stdout
            ref = json.loads(out)
        row = {"shape": name, "N": N, "rotation_keys": len(steps), "gpu_wall_s": gpu_s,
               "reference_1_thread": ref}
        if ref:
            row["speedup"] = ref["generate_keys_s"] / gpu_s
        kg.append(row)
        print(json.dumps(row), file=sys.stderr)
    json.dump({"client_encrypt": rows, "generate_keys": kg, "device": torch.cuda.get_device_name(0)},
              sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
