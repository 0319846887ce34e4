"""The oracle port is pinned to the UNMODIFIED reference: every artifact it
regenerates (keys, client ciphertexts, selector ciphertexts, distance
ciphertexts, aggregate chunks, op counters) must hash to the digest the
reference produced (tests/golden/*.json, made by tests/golden/make_golden.py)."""
import os

import numpy as np
import pytest

from tests.golden_util import Rig, sha

SMALL = ["tiny_krum", "tiny_hoist_multikrum", "tiny_eager", "tiny_fullhoist", "cfg1",
         "n16_multikrum", "n17_hoist", "tiny_rowsums", "tiny_rowsums_kgc", "tiny_perpair_kgc",
         "n13_rowsums"]


@pytest.fixture(scope="module", params=SMALL)
def rig(request):
    return Rig(request.param, threads=os.cpu_count())


def test_basis_matches_reference(rig):
    m = rig.meta
    assert rig.oracle.primes == m["primes"]
    assert rig.oracle.special == m["special"]
    assert rig.oracle.psi == m["psi"]
    assert rig.width == m["width"]
    assert rig.steps == m["steps"]
    assert m.get("mode", "per_pair") == rig.mode and m.get("reduced", True) == rig.reduce
    assert rig.C == m["chunks"]


def test_keys_and_inputs_match_reference(rig):
    d = rig.meta["sha256"]
    o = rig.oracle
    assert sha(o.secret_key()) == d["sk"]
    assert sha(o.relin_key()) == d["relin"]
    for s in rig.meta["rot_keys"]:
        assert sha(o.rotation_key(s)) == d[f"rot_{s}"], s
    for i in range(rig.n):
        assert sha(rig.clients[i]) == d[f"client_{i}"], i
        assert sha(rig.selectors[i]) == d[f"sel_{i}"], i


def test_distance_matrix_matches_reference(rig):
    o = rig.oracle
    o.reset_counts()
    f = o.distance_rows if rig.mode == "row_sums" else o.distance_matrix
    dm = f(rig.clients, rig.width, rig.k, lazy=rig.lazy, reduce=rig.reduce)
    assert o.counts() == rig.meta["dist_ops"]
    for p, (i, j) in enumerate(rig.dist_keys()):
        assert sha(dm[p]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)


def test_aggregate_matches_reference(rig):
    o = rig.oracle
    o.reset_counts()
    ag = o.masked_aggregate(rig.clients, rig.selectors, l=len(rig.selected), average=rig.average)
    assert o.counts() == rig.meta["agg_ops"]
    assert sha(ag) == rig.meta["sha256"]["agg"]


def test_intermediates_match_reference(rig):
    d = rig.meta["sha256"]
    if "p01_acc" not in d:
        pytest.skip("no intermediates recorded")
    o = rig.oracle
    a, b = rig.clients[0], rig.clients[1]
    acc = o.hsquare(o.hsub(a[0], b[0]))
    for c in range(1, rig.C):
        o.lazy_accumulate(acc, o.hsquare(o.hsub(a[c], b[c])))
    assert sha(acc) == d["p01_acc"]
    rl = o.relinearize(acc)
    assert sha(rl) == d["p01_relin"]
    rs = o.rescale(rl)
    assert sha(rs) == d["p01_rescale"]
    for s in rig.meta["rot_keys"]:
        assert sha(o.rotate(rs, s)) == d[f"p01_rot_{s}"], s
    t = o.hmult_triple(rig.clients[0][0], rig.selectors[0])
    for i in range(1, rig.n):
        o.lazy_accumulate(t, o.hmult_triple(rig.clients[i][0], rig.selectors[i]))
    assert sha(t) == d["agg0_acc"]


def test_decrypted_distances_track_plaintext(rig):
    """Reference tolerance: decrypted distances within rel 1e-3 of plaintext
    (test_distance.cpp:361-385)."""
    m = rig.meta
    if not rig.reduce:
        pytest.skip("unreduced: slot 0 holds one coordinate, not the total")
    for e, plain in zip(m["dist"], rig.plain_entries()):
        assert abs(e["slot0"] - plain) <= 1e-3 * max(1.0, abs(plain))


def test_cfg2_inputs_match_reference():
    """BASELINE configs[1] (10 clients, P=272,474, N=2^15): keys and all 170
    client ciphertexts regenerate bit-identically."""
    rig = Rig("cfg2")
    d = rig.meta["sha256"]
    assert rig.oracle.primes == rig.meta["primes"]
    assert sha(rig.oracle.relin_key()) == d["relin"]
    for i in range(rig.n):
        assert sha(rig.clients[i]) == d[f"client_{i}"], i
        assert sha(rig.selectors[i]) == d[f"sel_{i}"], i
