"""The C++ mirror header (include/lancelot_b200.hpp), linked by a reference-style
caller (tests/cpp/server_round.cpp), reproduces the reference's cfg1 server
round bit for bit (golden digests from the unmodified reference)."""
import json
import os
import subprocess

import numpy as np
import pytest

from tests.golden_util import Rig, sha

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "paper_2408_06197_b200", "_lib", "server_round")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg1", "tiny_hoist_multikrum"])
def test_cpp_mirror_server_round(tmp_path, name):
    rig = Rig(name, threads=8)
    if rig.meta["options"]["secure"]:
        pass  # the driver builds an unsecured context; primes are identical
    d = str(tmp_path)
    rig.oracle.relin_key().tofile(os.path.join(d, "relin.bin"))
    for s in rig.meta["rot_keys"]:
        rig.oracle.rotation_key(s).tofile(os.path.join(d, f"rot_{s}.bin"))
    rig.clients.tofile(os.path.join(d, "clients.bin"))
    rig.selectors.tofile(os.path.join(d, "selectors.bin"))
    rule = 1 if rig.rule == "multi_krum" else 0
    out = subprocess.run([DRIVER, d, str(rig.N), str(rig.n), str(rig.C), str(rig.dim),
                          str(rig.width), str(rig.k), str(rule), str(len(rig.selected)),
                          repr(rig.oracle.scale)], capture_output=True, text=True, check=True)
    info = json.loads(out.stdout.strip().splitlines()[0])
    dist = np.fromfile(os.path.join(d, "out_dist.bin"), dtype=np.uint64)
    agg = np.fromfile(os.path.join(d, "out_agg.bin"), dtype=np.uint64)
    per = dist.size // (rig.n * (rig.n - 1) // 2)
    p = 0
    for i in range(rig.n):
        for j in range(i + 1, rig.n):
            assert sha(dist[p * per:(p + 1) * per]) == rig.meta["sha256"][f"dist_{i}_{j}"]
            p += 1
    assert sha(agg) == rig.meta["sha256"]["agg"]
    assert info["dist_scale"] == rig.meta["dist"][0]["scale"]
    assert info["agg_scale"] == rig.meta["agg_scale"]
    assert info["rotations"] == rig.meta["dist_ops"]["rotations"]
