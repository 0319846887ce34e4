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
@pytest.mark.parametrize("name", ["cfg1", "tiny_hoist_multikrum", "tiny_rowsums",
                                  "tiny_perpair_kgc"])
def test_cpp_mirror_server_round(tmp_path, name):
    rig = Rig(name, threads=8)
    if rig.meta["options"]["secure"]:
        pass  # the driver builds an unsecured context; primes are identical
    d = str(tmp_path)
    rig.oracle.relin_key().tofile(os.path.join(d, "relin.bin"))
    mode = 1 if rig.mode == "row_sums" else 0
    for s in rig.meta["rot_keys"]:
        rig.oracle.rotation_key(s).tofile(os.path.join(d, f"rot_{s}.bin"))
    rig.clients.tofile(os.path.join(d, "clients.bin"))
    rig.selectors.tofile(os.path.join(d, "selectors.bin"))
    rule = 1 if rig.rule == "multi_krum" else 0
    out = subprocess.run([DRIVER, d, str(rig.N), str(rig.n), str(rig.C), str(rig.dim),
                          str(rig.width), str(rig.k), str(rule), str(len(rig.selected)),
                          repr(rig.oracle.scale), str(mode), str(int(rig.reduce))],
                         capture_output=True, text=True, check=True)
    info = json.loads(out.stdout.strip().splitlines()[0])
    dist = np.fromfile(os.path.join(d, "out_dist.bin"), dtype=np.uint64)
    agg = np.fromfile(os.path.join(d, "out_agg.bin"), dtype=np.uint64)
    keys = rig.dist_keys()
    assert info["entries"] == len(keys) and info["reduced"] == int(rig.reduce)
    per = dist.size // len(keys)
    for p, (i, j) in enumerate(keys):
        assert sha(dist[p * per:(p + 1) * per]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)
    assert sha(agg) == rig.meta["sha256"]["agg"]
    assert info["dist_scale"] == rig.meta["dist"][0]["scale"]
    assert info["agg_scale"] == rig.meta["agg_scale"]
    for k in ("additions", "multiplications", "relinearizations", "rescales", "rotations",
              "mod_ups"):
        assert info[k] == rig.meta["dist_ops"][k] + rig.meta["agg_ops"][k], k
    assert info["threads_identical"] == 1


def test_cpp_mirror_signatures_compile():
    """The reference's run_round call expressions and the exact parameter
    lists of build_distance_matrix / masked_aggregate (static_asserts in
    tests/cpp/server_round.cpp) compile against include/lancelot_b200.hpp."""
    src = os.path.join(ROOT, "tests", "cpp", "server_round.cpp")
    out = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                          src], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr[-3000:]
