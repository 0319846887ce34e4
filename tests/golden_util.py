"""Shared helpers: regenerate a golden configuration with the oracle port and
digest its artifacts exactly the way tests/golden/make_golden.py digests the
reference's dumps."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from oracle.oracle import Oracle, slot_reduce_steps

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as f:
        return json.load(f)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


def width_for(dim, N):
    need = min(dim, N // 2)
    return 1 << (need - 1).bit_length()


class Rig:
    """Keys, client ciphertexts and mask of one golden configuration."""

    def __init__(self, name, threads=None):
        self.meta = load(name)
        o = self.meta["options"]
        self.name = name
        self.N = o["N"]
        self.n = o["clients"]
        self.dim = o["dim"]
        self.k = o["k"]
        self.lazy = bool(o["lazy"])
        self.rule = o["rule"]
        self.selected = [int(x) for x in str(o["select"]).split(",")]
        self.average = self.rule == "multi_krum" and len(self.selected) > 1
        self.mode = o.get("mode", "per_pair")
        self.reduce = bool(o.get("reduce", 1))
        self.oracle = Oracle(self.N, secure=bool(o["secure"]), threads=threads)
        self.width = width_for(self.dim, self.N)
        # make_system: no rotation keys when the KGC sums the slots
        self.steps = slot_reduce_steps(self.width, self.k) if self.reduce else []
        self.oracle.keygen(1, self.steps)
        self.clients = self.oracle.make_clients(1, self.n, self.dim)
        self.selectors = self.oracle.build_mask(1, self.selected, self.n)
        self.C = self.clients.shape[1]

    def dist_keys(self):
        """Matrix entry keys in the reference's std::map order."""
        if self.mode == "row_sums":
            return [(i, i) for i in range(self.n)]
        return [(i, j) for i in range(self.n) for j in range(i + 1, self.n)]

    def plain_entries(self):
        """Plaintext slot totals per matrix entry (row sums add the pairs)."""
        pd = self.meta["plain_dist"]
        if self.mode != "row_sums":
            return pd
        pairs = [(i, j) for i in range(self.n) for j in range(i + 1, self.n)]
        return [sum(v for (a, b), v in zip(pairs, pd) if i in (a, b)) for i in range(self.n)]
