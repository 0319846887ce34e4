"""Generate tests/golden/*.json from the UNMODIFIED reference core.

Runs oracle/_ref/ref_driver (built by `make -C oracle ref` from the sources
under /root/reference) for each configuration below and records the SHA-256
digest of every artifact it dumps (keys, client ciphertexts, selectors,
distance ciphertexts, aggregate chunks, pair-(0,1) intermediates) together
with the reference's own metadata (primes, psi, op counters, decrypted slot-0
distances). Only digests are committed: the GPU box never sees
/root/reference, and the tests regenerate the inputs with the oracle port and
compare digests.

Usage: python tests/golden/make_golden.py [name ...]
"""
from __future__ import annotations

import glob
import hashlib
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

# name -> ref_driver options. cfg1/cfg2 are BASELINE.json configs[0]/[1].
CONFIGS = {
    "tiny_krum": dict(N=256, clients=4, dim=300, k=1, rule="krum", select="0", secure=0, lazy=1),
    "tiny_hoist_multikrum": dict(N=512, clients=6, dim=1000, k=3, rule="multi_krum",
                                 select="2,4", secure=0, lazy=1),
    "tiny_eager": dict(N=256, clients=3, dim=500, k=2, rule="median", select="1", secure=0,
                       lazy=0),
    "tiny_fullhoist": dict(N=256, clients=3, dim=128, k=8, rule="krum", select="2", secure=0,
                           lazy=1),
    "cfg1": dict(N=8192, clients=4, dim=8192, k=1, rule="krum", select="0", secure=1, lazy=1),
    "cfg2": dict(N=32768, clients=10, dim=272474, k=1, rule="krum", select="0", secure=1,
                 lazy=1),
    # cfg3's ring (N = 2^16, ResNet-18 width 32768) with 3 clients x 3 chunks,
    # Multi-Krum averaging, and the N = 2^17 kernels (BASELINE cfg5 sweep)
    "n16_multikrum": dict(N=65536, clients=3, dim=70000, k=1, rule="multi_krum", select="0,2",
                          secure=1, lazy=1),
    "n17_hoist": dict(N=131072, clients=3, dim=140000, k=2, rule="krum", select="1", secure=1,
                      lazy=1),
    # DistanceMode::row_sums and reduce_on_server = false (slot sums left to
    # the KGC, protocol.cpp:555): the other build_distance_matrix branches
    "tiny_rowsums": dict(N=256, clients=4, dim=300, k=2, rule="krum", select="0", secure=0,
                         lazy=1, mode="row_sums", reduce=1),
    "tiny_rowsums_kgc": dict(N=512, clients=5, dim=700, k=1, rule="krum", select="3", secure=0,
                             lazy=1, mode="row_sums", reduce=0),
    "tiny_perpair_kgc": dict(N=512, clients=5, dim=700, k=1, rule="multi_krum", select="0,3",
                             secure=0, lazy=1, mode="per_pair", reduce=0),
    # BASELINE configs[2] exactly as benchmarked: 20 clients x 11,173,962
    # params (342 chunks: the pair kernel's 256-chunk passes re-enter), N =
    # 2^16, lazy relin, hoisted rotations at the bench plan's k = 3
    "cfg3_hoist": dict(N=65536, clients=20, dim=11173962, k=3, rule="krum", select="0",
                       secure=1, lazy=1),
    "n13_rowsums": dict(N=8192, clients=5, dim=10000, k=3, rule="krum", select="1", secure=1,
                        lazy=1, mode="row_sums", reduce=1),
}


def sha(path):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for blk in iter(lambda: f.read(1 << 20), b""):
            h.update(blk)
    return h.hexdigest()


def generate(name, opts):
    with tempfile.TemporaryDirectory() as d:
        args = [DRIVER, "gen"]
        for k, v in opts.items():
            args += [f"--{k}", str(v)]
        args += ["--inter", "1" if opts["N"] <= 8192 else "0", "--out", d]
        subprocess.run(args, check=True)
        with open(os.path.join(d, "meta.json")) as f:
            meta = json.load(f)
        digests = {os.path.basename(p)[:-4]: sha(p) for p in sorted(glob.glob(os.path.join(d, "*.bin")))}
    meta["options"] = opts
    meta["sha256"] = digests
    meta["generator"] = "tests/golden/make_golden.py via oracle/_ref/ref_driver (reference core, -O3 -DNDEBUG)"
    out = os.path.join(HERE, f"{name}.json")
    with open(out, "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", out)


def main():
    if not os.path.exists(DRIVER):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    names = sys.argv[1:] or list(CONFIGS)
    for n in names:
        generate(n, CONFIGS[n])


if __name__ == "__main__":
    main()
