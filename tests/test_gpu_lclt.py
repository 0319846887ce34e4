"""LCLT ingest: the reference's ciphertext wire format
(CkksContext::serialize / deserialize, ckks.cpp:614-678) on the device, and
the server round fed with the blobs the server receives (run_round step 3,
protocol.cpp:419-432). Pinned to the reference's own serialized bytes
(tests/golden/*: lclt_client_0_0, lclt_dist_first) and its error messages."""
import ctypes as C
import hashlib

import numpy as np
import pytest

from tests.golden_util import Rig

pytestmark = pytest.mark.gpu


def _L():
    import paper_2408_06197_b200.lancelot as L
    return L


def bsha(b):
    return hashlib.sha256(bytes(b)).hexdigest()


def lclt(words, N, level, scale_bits=40, count=None):
    """serialize (ckks.cpp:614-638) restated for building test inputs."""
    count = level + 1 if count is None else count
    hdr = (b"LCLT" + (1).to_bytes(2, "little") + int(N).to_bytes(4, "little")
           + bytes([level, scale_bits, count]))
    return hdr + np.ascontiguousarray(words, np.uint64).tobytes()


_CTX = {}


def ctx_for(N, secure):
    L = _L()
    if (N, secure) not in _CTX:
        _CTX[(N, secure)] = L.CkksContext(L.CkksParams(
            ring_degree=N, security=L.SecurityLevel.bits128 if secure else L.SecurityLevel.none))
    return _CTX[(N, secure)]


@pytest.mark.parametrize("name", ["tiny_krum", "cfg1"])
def test_serialize_and_deserialize_match_reference_bytes(name):
    L = _L()
    rig = Rig(name, threads=8)
    d = rig.meta["sha256"]
    ctx = ctx_for(rig.N, bool(rig.meta["options"]["secure"]))
    ct = L.Ciphertext(L.to_device(rig.clients[0, 0]), rig.oracle.scale)
    blob = ctx.serialize(ct)
    assert len(blob) == ctx.blob_bytes()
    assert bsha(blob) == d["lclt_client_0_0"]
    assert blob == lclt(rig.clients[0, 0], rig.N, ctx.full - 1)
    back = ctx.deserialize(blob)
    assert np.array_equal(L.to_host(back.data), rig.clients[0, 0])
    assert back.scale == 2.0 ** 40
    # a matrix entry (level 2, scale s^2 / q_3 -> 40 scale bits in the header)
    dm = L.build_distance_matrix(
        ctx, [L.PackedWeights(L.to_device(rig.clients[i]), rig.dim, 1.0, rig.oracle.scale)
              for i in range(rig.n)],
        L.RelinKey(rig.oracle.relin_key()), L.HoistPlan(k=rig.k, n=rig.width),
        L.DistanceMode.per_pair,
        L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]}),
        L.DistanceOptions())
    first = ctx.serialize(L.Ciphertext(dm.batch[0], dm.scale))
    assert bsha(first) == d["lclt_dist_first"]
    # batch with padding between blobs: verbatim bytes, padding untouched
    stride = ctx.blob_bytes() + 19
    bb = ctx.serialize_batch(L.to_device(rig.clients[1]), rig.oracle.scale, stride)
    for c in range(rig.C):
        assert bb[c, :ctx.blob_bytes()].tobytes() == lclt(rig.clients[1, c], rig.N, ctx.full - 1)
    got, sc = ctx.deserialize_batch(bb, ctx.blob_bytes())
    assert np.array_equal(L.to_host(got), rig.clients[1]) and sc == 2.0 ** 40


def test_deserialize_errors_match_reference():
    """ckks.cpp:640-670: every DataError branch with the reference's message;
    batch rules: one level (ShapeError) and one scale (AlignmentError)."""
    L = _L()
    N = 1024
    ctx = ctx_for(N, False)
    m = ctx.full
    rng = np.random.default_rng(5)
    qs = ctx.primes
    w = np.stack([np.stack([rng.integers(0, qs[r], N, dtype=np.uint64) for r in range(m)])
                  for _ in range(2)])
    good = lclt(w, N, m - 1)
    ct = ctx.deserialize(good)
    assert np.array_equal(L.to_host(ct.data), w)

    def bad(b, msg):
        with pytest.raises(L.DataError, match=msg):
            ctx.deserialize(b)

    bad(good[:12], "not a ciphertext blob")
    bad(b"LCLX" + good[4:], "not a ciphertext blob")
    bad(good[:4] + (2).to_bytes(2, "little") + good[6:], "unsupported ciphertext format version")
    bad(good[:6] + (2 * N).to_bytes(4, "little") + good[10:], "ring degree does not match")
    bad(good[:10] + bytes([m, 40, m + 1]) + good[13:], "level inconsistent")
    bad(good[:10] + bytes([m - 1, 40, m - 1]) + good[13:], "level inconsistent")
    bad(good + b"\0" * 8, "blob length mismatch")
    bad(good[:-8], "blob length mismatch")
    for row, val in ((0, qs[0]), (m - 1, qs[m - 1]), (m + 1, qs[1]), (1, (1 << 64) - 1)):
        w2 = w.copy().reshape(2 * m, N)
        w2[row, 7] = np.uint64(val)
        bad(lclt(w2, N, m - 1), "residue outside its modulus")
    # lower level blobs deserialize at their own limb count
    low = lclt(w[:, :2], N, 1, scale_bits=33)
    ct2 = ctx.deserialize(low)
    assert ct2.data.shape[1] == 2 and ct2.scale == 2.0 ** 33
    mixed = np.frombuffer(good + good[:10] + bytes([m - 1, 41, m]) + good[13:], np.uint8)
    with pytest.raises(L.AlignmentError):
        ctx.deserialize_batch(mixed.reshape(2, -1))
    with pytest.raises(L.ParameterError):
        ctx.serialize(L.Ciphertext(ct.data, 0.5))


@pytest.mark.parametrize("name,pad", [("cfg1", 0), ("tiny_hoist_multikrum", 3), ("cfg2", 51)])
def test_server_round_from_lclt_blobs(name, pad):
    """lcl_server_round_lclt: the clients' and selectors' blobs (unaligned
    13-byte headers; strides with and without padding) go through the
    overlapped H2D pipeline and the device unpack; the distance matrix, the
    aggregate and the counters are the reference's. A single residue >= q in
    one chunk fails the round with DataError."""
    L = _L()
    rig = Rig(name, threads=8)
    ctx = ctx_for(rig.N, bool(rig.meta["options"]["secure"]))
    ctx.use_relin_key(L.RelinKey(rig.oracle.relin_key()))
    keys = L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]})
    ctx.use_rotation_keys(keys, rig.steps)
    m, N, n = ctx.full, rig.N, rig.n
    bb = ctx.blob_bytes()
    stride = bb + pad
    cb = np.zeros((n * rig.C, stride), np.uint8)
    for i in range(n):
        for c in range(rig.C):
            cb[i * rig.C + c, :bb] = np.frombuffer(lclt(rig.clients[i, c], N, m - 1), np.uint8)
    sb = np.zeros((n, stride), np.uint8)
    for i in range(n):
        sb[i, :bb] = np.frombuffer(lclt(rig.selectors[i], N, m - 1), np.uint8)
    P = n * (n - 1) // 2
    mo = m - 2 if rig.average else m - 1
    h_dist = np.zeros((P, 2, m - 1, N), np.uint64)
    h_agg = np.zeros((rig.C, 2, mo, N), np.uint64)
    dsc, asc = C.c_double(), C.c_double()

    def run(blobs):
        L._check(L.lib().lcl_server_round_lclt(
            ctx.h, blobs.ctypes.data, sb.ctypes.data, bb, stride, n, rig.C, rig.width, rig.k,
            len(rig.selected), 1 if rig.average else 0, h_dist.ctypes.data, h_agg.ctypes.data,
            C.byref(dsc), C.byref(asc)))

    ctx.reset_counters()
    run(cb)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    for p, (i, j) in enumerate(pairs):
        assert hashlib.sha256(h_dist[p].tobytes()).hexdigest() == rig.meta["sha256"][f"dist_{i}_{j}"]
    assert hashlib.sha256(h_agg.tobytes()).hexdigest() == rig.meta["sha256"]["agg"]
    want = {k: rig.meta["dist_ops"][k] + rig.meta["agg_ops"][k] for k in rig.meta["dist_ops"]}
    assert ctx.counters() == want
    assert dsc.value == rig.meta["dist"][0]["scale"] and asc.value == rig.meta["agg_scale"]
    bad = cb.copy()
    row = (n // 2) * rig.C + rig.C - 1
    bad[row, 13 + 8 * (N + 5): 13 + 8 * (N + 6)] = np.frombuffer(
        np.uint64(ctx.primes[1]).tobytes(), np.uint8)
    with pytest.raises(L.DataError, match="residue outside its modulus"):
        run(bad)
    bad = cb.copy()
    bad[3, 0] = ord("X")
    with pytest.raises(L.DataError, match="not a ciphertext blob"):
        run(bad)
