"""GPU parity: every sm_100a kernel path, called through the C-ABI, against
the oracle port (which is itself pinned to the reference by
tests/test_oracle_golden.py) and against the reference's golden digests."""
import numpy as np
import pytest

from oracle.oracle import Oracle, slot_reduce_steps
from tests.golden_util import Rig, sha

pytestmark = pytest.mark.gpu


def _L():
    import paper_2408_06197_b200.lancelot as L
    return L


_CTX = {}


def gpu_ctx(N, secure=False):
    L = _L()
    key = (N, secure)
    if key not in _CTX:
        _CTX[key] = L.CkksContext(L.CkksParams(
            ring_degree=N, security=L.SecurityLevel.bits128 if secure else L.SecurityLevel.none))
    return _CTX[key]


@pytest.mark.parametrize("N", [256, 1024, 4096, 8192, 16384, 32768, 65536, 131072])
def test_ntt_matches_oracle(N):
    L = _L()
    import torch
    orc = Oracle(N, secure=False, threads=1)
    ctx = gpu_ctx(N)
    assert ctx.primes == orc.primes and ctx.special == orc.special
    rng = np.random.default_rng(N)
    P = orc.full + 1
    items = 3
    rows = np.zeros((items, P, N), np.uint64)
    qs = orc.primes + [orc.special]
    for r in range(P):
        rows[:, r] = rng.integers(0, qs[r], size=(items, N), dtype=np.uint64)
    rows[0, 0, :] = 0
    rows[0, 1, :] = np.uint64(qs[1] - 1)
    want_f = np.stack([[orc.ntt_forward(rows[i, r], r) for r in range(P)] for i in range(items)])
    d = L.to_device(rows)
    L._check(L.lib().lcl_ntt_forward(ctx.h, L._ptr(d), items, orc.full, 1))
    torch.cuda.synchronize()
    got_f = L.to_host(d)
    assert np.array_equal(got_f, want_f)
    L._check(L.lib().lcl_ntt_inverse(ctx.h, L._ptr(d), items, orc.full, 1))
    torch.cuda.synchronize()
    assert np.array_equal(L.to_host(d), rows)
    want_i = np.stack([[orc.ntt_inverse(rows[i, r], r) for r in range(P)] for i in range(items)])
    d = L.to_device(rows)
    L._check(L.lib().lcl_ntt_inverse(ctx.h, L._ptr(d), items, orc.full, 1))
    torch.cuda.synchronize()
    assert np.array_equal(L.to_host(d), want_i)


@pytest.fixture(scope="module", params=[1024, 8192])
def evalrig(request):
    N = request.param
    orc = Oracle(N, secure=False, threads=4)
    steps = [1, 2, 3, 4, 7, 8, 16, 32, 64]
    orc.keygen(1, steps)
    clients = orc.make_clients(1, 3, N)  # two chunks each
    return N, orc, steps, clients


def test_evaluator_matches_oracle(evalrig):
    L = _L()
    N, orc, steps, clients = evalrig
    ctx = gpu_ctx(N)
    rk = L.RelinKey(orc.relin_key())
    keys = L.RotationKeySet({s: orc.rotation_key(s) for s in steps})
    s = orc.scale
    a = L.Ciphertext(L.to_device(clients[0, 0]), s)
    b = L.Ciphertext(L.to_device(clients[1, 0]), s)
    assert np.array_equal(L.to_host(ctx.hsub(a, b).data), orc.hsub(clients[0, 0], clients[1, 0]))
    assert np.array_equal(L.to_host(ctx.hadd(a, b).data), orc.hadd(clients[0, 0], clients[1, 0]))
    t = orc.hsquare(orc.hsub(clients[0, 0], clients[1, 0]))
    sq = ctx.hsquare(ctx.hsub(a, b))
    assert np.array_equal(L.to_host(sq.data), t) and sq.scale == s * s
    hm = ctx.hmult_triple(a, b)
    assert np.array_equal(L.to_host(hm.data), orc.hmult_triple(clients[0, 0], clients[1, 0]))
    tern = L.TernaryCiphertext(L.to_device(t), s * s)
    rl = ctx.relinearize(tern, rk)
    want_rl = orc.relinearize(t)
    assert np.array_equal(L.to_host(rl.data), want_rl)
    rs = ctx.rescale(rl)
    want_rs = orc.rescale(want_rl)
    assert np.array_equal(L.to_host(rs.data), want_rs)
    assert rs.scale == (s * s) / float(orc.primes[3])
    for st in steps:
        got = ctx.rotate(rs, st, keys)
        assert np.array_equal(L.to_host(got.data), orc.rotate(want_rs, st)), st
    hs = [1, 2, 3, 0, 7]
    got = ctx.hoisted_rotations(rs, hs, keys)
    want = orc.hoisted_rotations(want_rs, hs)
    for i in range(len(hs)):
        assert np.array_equal(L.to_host(got[i].data), want[i]), hs[i]
    for width, k in [(128, 1), (128, 3), (8, 3), (64, 2), (1, 1)]:
        got = L.slot_reduce(ctx, rs, L.HoistPlan(k=k, n=width), keys)
        assert np.array_equal(L.to_host(got.data), orc.slot_reduce(want_rs, width, k)), (width, k)
    # fresh-level (m = 4) rotation and rescale chain down to level 0
    top = L.Ciphertext(L.to_device(clients[2, 1]), s)
    assert np.array_equal(L.to_host(ctx.rotate(top, 3, keys).data), orc.rotate(clients[2, 1], 3))
    x, xw = top, clients[2, 1]
    for _ in range(3):
        x, xw = ctx.rescale(x), orc.rescale(xw)
        assert np.array_equal(L.to_host(x.data), xw)
    with pytest.raises(L.DepthExhaustedError):
        ctx.rescale(x)
    with pytest.raises(L.KeyError):
        ctx.rotate(rs, 5, keys)


@pytest.mark.parametrize("N", [8192, 16384])
def test_fused_hoisted_key_switch_matches_oracle(N):
    """modup_ip_hoist (one ModUp block pass shared by up to 8 steps; 15
    steps = two launches): hoisted_rotations on a batch of 2 fresh (m = 4)
    and rescaled (m = 3) ciphertexts, zero / repeated / beyond-slots steps,
    and slot_reduce with k = 5 (15 hoisted steps), word for word."""
    L = _L()
    import ctypes as C
    import torch
    orc = Oracle(N, secure=False, threads=8)
    width = 4096
    steps = slot_reduce_steps(width, 5)
    orc.keygen(3, steps)
    cl = orc.make_clients(3, 2, N)  # 2 clients x 2 chunks
    ctx = gpu_ctx(N)
    keys = L.RotationKeySet({s_: orc.rotation_key(s_) for s_ in steps})
    ctx.use_rotation_keys(keys, steps)
    hs = [1, 2, 3, 0, 7, 9, 15, 4, 5, 6, 11, 3, N // 2 + 1]
    cts = [cl[0, 0], cl[1, 1]]
    for m in (4, 3):
        if m == 3:
            cts = [orc.rescale(x) for x in cts]
        d = L.to_device(np.stack(cts))
        outs = torch.empty((len(hs), 2, 2, m, N), dtype=torch.int64, device="cuda")
        arr = (C.c_size_t * len(hs))(*hs)
        L._check(L.lib().lcl_hoisted_rotations(ctx.h, L._ptr(d), 2, m, arr, len(hs), L._ptr(outs)))
        got = L.to_host(outs)
        for b in range(2):
            want = orc.hoisted_rotations(cts[b], hs)
            for i, st in enumerate(hs):
                assert np.array_equal(got[i, b], want[i]), (m, b, st)
    rs = L.Ciphertext(L.to_device(cts[0]), orc.scale)
    for k in (5, 4):
        got = L.slot_reduce(ctx, rs, L.HoistPlan(k=k, n=width), keys)
        assert np.array_equal(L.to_host(got.data), orc.slot_reduce(cts[0], width, k)), k
    with pytest.raises(L.KeyError):
        ctx.hoisted_rotations(rs, [1, 2, 17], keys)


def test_mult_plain_matches_oracle(evalrig):
    L = _L()
    N, orc, steps, clients = evalrig
    ctx = gpu_ctx(N)
    ct = orc.rescale(clients[0, 0])
    for l in (2, 3, 7, 25):
        got = ctx.mult_plain_const(L.Ciphertext(L.to_device(ct), 1.0), 1.0 / l, orc.scale)
        want = orc.mult_plain_inv_l(ct, l)  # includes the rescale
        assert np.array_equal(L.to_host(ctx.rescale(got).data), want), l


GOLDEN = ["tiny_krum", "tiny_hoist_multikrum", "tiny_eager", "tiny_fullhoist", "cfg1", "cfg2",
          "n16_multikrum", "n17_hoist"]


@pytest.fixture(scope="module", params=GOLDEN)
def golden(request):
    return Rig(request.param, threads=8)


def _packed(L, rig):
    dev = L.to_device(rig.clients)
    return [L.PackedWeights(dev[i], rig.dim, 1.0, rig.oracle.scale) for i in range(rig.n)]


def test_distance_matrix_bit_exact_vs_reference(golden):
    L = _L()
    rig = golden
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    rk = L.RelinKey(rig.oracle.relin_key())
    keys = L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]})
    pw = _packed(L, rig)
    ctx.reset_counters()
    dm = L.build_distance_matrix(ctx, pw, rk, L.HoistPlan(k=rig.k, n=rig.width),
                                 L.DistanceMode.per_pair, keys,
                                 L.DistanceOptions(lazy_relin=rig.lazy))
    got = L.to_host(dm.batch)
    counts = ctx.counters()
    for p, (i, j) in enumerate(dm.keys):
        assert sha(got[p]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)
    assert counts == rig.meta["dist_ops"]
    e0 = rig.meta["dist"][0]
    assert dm.scale == e0["scale"]
    assert dm.value_scale == 1.0


MODE_GOLDEN = ["tiny_rowsums", "tiny_rowsums_kgc", "tiny_perpair_kgc", "n13_rowsums"]


@pytest.mark.parametrize("name", MODE_GOLDEN)
def test_distance_modes_bit_exact_vs_reference(name):
    """build_distance_matrix's other branches through lcl_build_distance_matrix:
    DistanceMode::row_sums (one device row-sum launch, then slot_reduce per
    row) and reduce_on_server = false (slot sums left to the KGC), against
    the reference's digests, op counters, scale and `reduced` flag."""
    L = _L()
    rig = Rig(name, threads=8)
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    rk = L.RelinKey(rig.oracle.relin_key())
    keys = L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]})
    mode = L.DistanceMode.row_sums if rig.mode == "row_sums" else L.DistanceMode.per_pair
    ctx.reset_counters()
    dm = L.build_distance_matrix(ctx, _packed(L, rig), rk, L.HoistPlan(k=rig.k, n=rig.width),
                                 mode, keys, L.DistanceOptions(lazy_relin=rig.lazy,
                                                               reduce_on_server=rig.reduce))
    got = L.to_host(dm.batch)
    assert list(dm.keys) == rig.dist_keys()
    for p, (i, j) in enumerate(dm.keys):
        assert sha(got[p]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)
    assert ctx.counters() == rig.meta["dist_ops"]
    assert dm.reduced == rig.meta["reduced"]
    assert dm.scale == rig.meta["dist"][0]["scale"]
    if rig.reduce:  # slot 0 holds the total: the reference's decryption
        sk = L.SecretKey(rig.oracle.secret_key())
        vals = ctx.decrypt_values_batch(dm.batch, dm.scale, sk).cpu().numpy()
        for p, e in enumerate(rig.meta["dist"]):
            assert vals[p][0] == e["slot0"], p


@pytest.mark.parametrize("name", ["tiny_krum", "cfg1", "tiny_perpair_kgc", "tiny_rowsums",
                                  "tiny_rowsums_kgc", "n13_rowsums"])
def test_kgc_distance_table_and_totals(name):
    """table_from_matrix / totals_from_matrix (aggregation.cpp:242-277) on
    the device: reduced entries give the reference's decrypted slot 0 (golden)
    / value_scale clamped at 0; unreduced ones the left-to-right sum of the
    oracle-decrypted slots; totals are the rows' left-to-right sums."""
    L = _L()
    rig = Rig(name, threads=8)
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    mode = L.DistanceMode.row_sums if rig.mode == "row_sums" else L.DistanceMode.per_pair
    dm = L.build_distance_matrix(ctx, _packed(L, rig), L.RelinKey(rig.oracle.relin_key()),
                                 L.HoistPlan(k=rig.k, n=rig.width), mode,
                                 L.RotationKeySet({s: rig.oracle.rotation_key(s)
                                                   for s in rig.meta["rot_keys"]}),
                                 L.DistanceOptions(reduce_on_server=rig.reduce))
    sk = L.SecretKey(rig.oracle.secret_key())
    words = L.to_host(dm.batch)
    want = []
    for p in range(len(dm.keys)):
        if rig.reduce:
            v = rig.meta["dist"][p]["slot0"]
        else:
            v = np.add.accumulate(rig.oracle.decrypt_values(words[p], dm.scale))[-1]
        want.append(max(0.0, v / dm.value_scale))
    totals = L.totals_from_matrix(ctx, dm, sk)
    if mode == L.DistanceMode.per_pair:
        t = L.table_from_matrix(ctx, dm, sk)
        for p, (i, j) in enumerate(dm.keys):
            assert t.d[i][j] == want[p] and t.d[j][i] == want[p]
        assert all(t.d[i][i] == 0.0 for i in range(rig.n))
        for i in range(rig.n):
            acc = 0.0
            for j in range(rig.n):
                acc += t.d[i][j]
            assert totals[i] == acc
    else:
        with pytest.raises(L.UsageError):
            L.table_from_matrix(ctx, dm, sk)
        assert list(totals) == want


@pytest.mark.parametrize("name,lazy", [("tiny_krum", True), ("cfg1", True), ("tiny_eager", False)])
def test_pairwise_distance_entry(name, lazy):
    """lcl_pairwise_distance (encrypted_pairwise_distance, distance.cpp:107-142)
    for clients 0 and 1: the lazy result is the reference's p01_rescale
    intermediate; the eager one equals the oracle's."""
    L = _L()
    rig = Rig(name, threads=8)
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    pw = _packed(L, rig)
    ctx.reset_counters()
    ct = L.encrypted_pairwise_distance(ctx, pw[0], pw[1], L.RelinKey(rig.oracle.relin_key()),
                                       lazy=lazy)
    got = L.to_host(ct.data)
    if lazy:
        assert sha(got) == rig.meta["sha256"]["p01_rescale"]
    else:
        assert np.array_equal(got, rig.oracle.pairwise_distance(rig.clients[0], rig.clients[1],
                                                                lazy=False))
    c = ctx.counters()
    assert c["multiplications"] == rig.C
    assert c["relinearizations"] == (1 if lazy else rig.C)
    assert ct.scale == rig.meta["dist"][0]["scale"]


def test_masked_aggregate_bit_exact_vs_reference(golden):
    L = _L()
    rig = golden
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    rk = L.RelinKey(rig.oracle.relin_key())
    pw = _packed(L, rig)
    mask = L.SelectionMask(rig.n, len(rig.selected), L.to_device(rig.selectors), rig.oracle.scale)
    rule = {"krum": L.SelectionRule.krum, "multi_krum": L.SelectionRule.multi_krum,
            "median": L.SelectionRule.median}[rig.rule]
    ctx.reset_counters()
    agg = L.masked_aggregate(ctx, pw, mask, rule, rk)
    assert sha(L.to_host(agg.chunks)) == rig.meta["sha256"]["agg"]
    assert ctx.counters() == rig.meta["agg_ops"]
    assert agg.scale == rig.meta["agg_scale"]


@pytest.mark.parametrize("mode", ["1", "0", "3", "8", "8:unsliced", "8:singles", "8:singles+slicepairs"])
def test_host_round_overlapped_bit_exact_vs_reference(golden, mode, monkeypatch):
    """lcl_server_round_host (host buffers in and out; H2D overlapped with
    the computation: 1 = two client groups on two lanes, 0 = chunk slices,
    3 / 8 = three / eight client groups, 8 the default: the last group's
    aggregate in chunk slices; unsliced = one piece; singles = the last two
    clients as single-client groups on high-priority lanes; slicepairs = the
    last group's pairs accumulated per slice on a low-priority stream)
    against the reference digests and op counters."""
    L = _L()
    import ctypes as C
    groups, _, form = mode.partition(":")
    monkeypatch.setenv("LCL_HOST_ROUND", groups)
    if form == "unsliced":
        monkeypatch.setenv("LCL_LAST_SLICES", "1")
    if form.startswith("singles"):
        monkeypatch.setenv("LCL_TAIL_SINGLES", "2")
        monkeypatch.setenv("LCL_LANE_PRIO", "1")
    if form.endswith("slicepairs"):
        monkeypatch.setenv("LCL_LAST_PAIRS", "1")
    rig = golden
    if not rig.lazy:
        pytest.skip("the host round entry is the lazy, reduced per-pair round")
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    ctx.use_relin_key(L.RelinKey(rig.oracle.relin_key()))
    keys = L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]})
    ctx.use_rotation_keys(keys, rig.steps)
    m, N, n = rig.oracle.full, rig.N, rig.n
    h_clients = np.ascontiguousarray(rig.clients)
    h_sel = np.ascontiguousarray(rig.selectors)
    npairs = n * (n - 1) // 2
    h_dist = np.zeros((npairs, 2, m - 1, N), np.uint64)
    mo = m - 2 if rig.average else m - 1
    h_agg = np.zeros((rig.C, 2, mo, N), np.uint64)
    ctx.reset_counters()
    L._check(L.lib().lcl_server_round_host(
        ctx.h, C.c_void_p(h_clients.ctypes.data), C.c_void_p(h_sel.ctypes.data), n, rig.C,
        rig.oracle.scale, rig.width, rig.k, len(rig.selected), 1 if rig.average else 0,
        C.c_void_p(h_dist.ctypes.data), C.c_void_p(h_agg.ctypes.data)))
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    for p, (i, j) in enumerate(pairs):
        assert sha(h_dist[p]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)
    assert sha(h_agg) == rig.meta["sha256"]["agg"]
    want = {k: rig.meta["dist_ops"][k] + rig.meta["agg_ops"][k] for k in rig.meta["dist_ops"]}
    assert ctx.counters() == want


def test_decrypted_results_within_ckks_tolerance(golden):
    """Decrypt the GPU outputs with the oracle: distances within rel 1e-5 of
    the reference's decryption (same words => identical), and within the
    reference's own 1e-3 of the plaintext distances."""
    L = _L()
    rig = golden
    if rig.N > 8192:
        pytest.skip("decryption check on small rings only")
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    rk = L.RelinKey(rig.oracle.relin_key())
    keys = L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]})
    dm = L.build_distance_matrix(ctx, _packed(L, rig), rk, L.HoistPlan(k=rig.k, n=rig.width),
                                 L.DistanceMode.per_pair, keys,
                                 L.DistanceOptions(lazy_relin=rig.lazy))
    got = L.to_host(dm.batch)
    for p, e in enumerate(rig.meta["dist"]):
        v = rig.oracle.decrypt_values(got[p], dm.scale)[0]
        assert abs(v - e["slot0"]) <= 1e-5 * max(1.0, abs(e["slot0"]))
        plain = rig.meta["plain_dist"][p]
        assert abs(v - plain) <= 1e-3 * max(1.0, abs(plain))


def test_server_round_concurrent_bit_exact(golden):
    """lcl_server_round (distance matrix + aggregate, the aggregate on its own
    stream concurrently) reproduces the reference digests and counters."""
    L = _L()
    import torch
    rig = golden
    if not rig.lazy:
        pytest.skip("the combined entry is the lazy, reduced per-pair round")
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    ctx.use_relin_key(L.RelinKey(rig.oracle.relin_key()))
    keys = L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]})
    ctx.use_rotation_keys(keys, rig.steps)
    m, N, n = rig.oracle.full, rig.N, rig.n
    P = n * (n - 1) // 2
    mo = m - 2 if rig.average else m - 1
    cl = L.to_device(rig.clients)
    sel = L.to_device(rig.selectors)
    dd = torch.empty((P, 2, m - 1, N), dtype=torch.int64, device="cuda")
    da = torch.empty((rig.C, 2, mo, N), dtype=torch.int64, device="cuda")
    ctx.reset_counters()
    L._check(L.lib().lcl_server_round(ctx.h, L._ptr(cl), L._ptr(sel), n, rig.C, rig.width, rig.k,
                                      len(rig.selected), 1 if rig.average else 0, L._ptr(dd),
                                      L._ptr(da)))
    torch.cuda.synchronize()
    got = L.to_host(dd)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    for p, (i, j) in enumerate(pairs):
        assert sha(got[p]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)
    assert sha(L.to_host(da)) == rig.meta["sha256"]["agg"]
    want = {k: rig.meta["dist_ops"][k] + rig.meta["agg_ops"][k] for k in rig.meta["dist_ops"]}
    assert ctx.counters() == want


def test_kgc_decrypt_decode_bit_exact(golden):
    """Batched decrypt_values on the device (KGC side): every
    slot of every distance ciphertext and aggregate chunk equals the oracle's
    decode of the same words bit for bit, and slot 0 of each distance equals
    the reference's own decrypted value from the golden run."""
    L = _L()
    rig = golden
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    rk = L.RelinKey(rig.oracle.relin_key())
    keys = L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]})
    sk = L.SecretKey(rig.oracle.secret_key())
    dm = L.build_distance_matrix(ctx, _packed(L, rig), rk, L.HoistPlan(k=rig.k, n=rig.width),
                                 L.DistanceMode.per_pair, keys,
                                 L.DistanceOptions(lazy_relin=rig.lazy))
    got = ctx.decrypt_values_batch(dm.batch, dm.scale, sk).cpu().numpy()
    words = L.to_host(dm.batch)
    for p, e in enumerate(rig.meta["dist"]):
        if p < 6:
            assert np.array_equal(got[p], rig.oracle.decrypt_values(words[p], dm.scale)), p
        assert got[p][0] == e["slot0"], p
    mask = L.SelectionMask(rig.n, len(rig.selected), L.to_device(rig.selectors), rig.oracle.scale)
    rule = {"krum": L.SelectionRule.krum, "multi_krum": L.SelectionRule.multi_krum,
            "median": L.SelectionRule.median}[rig.rule]
    agg = L.masked_aggregate(ctx, _packed(L, rig), mask, rule, rk)
    got = ctx.decrypt_values_batch(agg.chunks, agg.scale, sk).cpu().numpy()
    aw = L.to_host(agg.chunks)
    for c in range(min(3, aw.shape[0])):
        assert np.array_equal(got[c], rig.oracle.decrypt_values(aw[c], agg.scale)), c


@pytest.mark.parametrize("name,shards", [("cfg2", 3), ("tiny_hoist_multikrum", 2)])
def test_chunk_sharded_partials_bit_exact(name, shards):
    """The chunk-sharded distance path (lcl_pair_partials per chunk slice,
    integer sum of the partial ternaries, lcl_pair_combine, lcl_pair_finish)
    run shard by shard on one GPU reproduces the reference digests and op
    counters; the multi-rank orchestration is tests/test_sharded.py."""
    L = _L()
    import torch
    from paper_2408_06197_b200.sharded import shard_range
    rig = Rig(name, threads=8)
    if not rig.lazy:
        pytest.skip("lazy accumulation only")
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    ctx.use_relin_key(L.RelinKey(rig.oracle.relin_key()))
    keys = L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]})
    ctx.use_rotation_keys(keys, rig.steps)
    lib = L.lib()
    m, N, n = rig.oracle.full, rig.N, rig.n
    P = n * (n - 1) // 2
    ctx.reset_counters()
    total = None
    for g in range(shards):
        c0, c1 = shard_range(rig.C, shards, g)
        local = L.to_device(np.ascontiguousarray(rig.clients[:, c0:c1]))
        t = torch.empty((P, 3, m, N), dtype=torch.int64, device="cuda")
        L._check(lib.lcl_pair_partials(ctx.h, L._ptr(local), n, c1 - c0, L._ptr(t)))
        total = t if total is None else total + t
    L._check(lib.lcl_pair_combine(ctx.h, L._ptr(total), P, shards))
    out = torch.empty((P, 2, m - 1, N), dtype=torch.int64, device="cuda")
    L._check(lib.lcl_pair_finish(ctx.h, L._ptr(total), P, rig.width, rig.k, 1, L._ptr(out)))
    got = L.to_host(out)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    for p, (i, j) in enumerate(pairs):
        assert sha(got[p]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)
    assert ctx.counters() == rig.meta["dist_ops"]


@pytest.mark.parametrize("name", ["cfg1", "tiny_hoist_multikrum", "cfg2"])
def test_pack_and_encrypt_bit_exact(name):
    """Client side: measure_distance_phase's inputs (one
    Sampler(derive_seed(1, 0xAB1A7E)) shared by the clients: dim uniform_real
    draws, then pack_and_encrypt) produced through lcl_pack_and_encrypt equal
    the reference's client ciphertexts (golden digests) word for word."""
    L = _L()
    rig = Rig(name, threads=8)
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    pk = L.PublicKey(rig.oracle.public_key())
    rng = L.Sampler(L.derive_seed(1, 0xAB1A7E))
    ctx.reset_counters()
    got = []
    for i in range(rig.n):
        w = rng.uniform_real(rig.dim) - 0.5
        pw = L.pack_and_encrypt(ctx, w, pk, rng)
        assert pw.chunk_count() == rig.C
        got.append(L.to_host(pw.chunks))
    got = np.stack(got)
    assert np.array_equal(got, rig.clients)
    assert ctx.counters()["encryptions"] == rig.n * rig.C


@pytest.mark.parametrize("name", ["cfg1", "tiny_hoist_multikrum"])
def test_build_mask_bit_exact(name):
    """build_mask through lcl_build_mask with the protocol's mask sampler
    (derive_seed(1, 0x3000000000000000)): the client selectors equal the
    reference's (golden digests via the oracle) word for word."""
    L = _L()
    rig = Rig(name, threads=8)
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    pk = L.PublicKey(rig.oracle.public_key())
    rng = L.Sampler(L.derive_seed(1, 0x3000000000000000))
    ctx.reset_counters()
    _, sels = L.build_mask(ctx, rig.selected, rig.n, pk, rng)
    assert np.array_equal(L.to_host(sels), rig.selectors)
    assert ctx.counters()["encryptions"] == 2 * rig.n


def test_client_and_kgc_errors():
    """The new entry points raise the reference's exception types:
    pack_and_encrypt DataError / CapacityError / ShapeError (distance.cpp:68-76,
    ckks.cpp:267-281), build_mask ShapeError / CapacityError
    (aggregation.cpp:158-163), decrypt_values KeyError for a short key."""
    L = _L()
    N = 1024
    orc = Oracle(N, secure=False, threads=2)
    orc.keygen(1, [1])
    ctx = gpu_ctx(N)
    pk = L.PublicKey(orc.public_key())
    rng = L.Sampler(3)
    with pytest.raises(L.DataError):
        L.pack_and_encrypt(ctx, np.array([0.1, np.nan]), pk, rng)
    with pytest.raises(L.CapacityError):
        L.pack_and_encrypt(ctx, np.array([2.0 ** 21]), pk, rng)
    with pytest.raises(L.ShapeError):
        L.pack_and_encrypt(ctx, np.array([]), pk, rng)
    with pytest.raises(L.ShapeError):
        L.build_mask(ctx, [5], 4, pk, rng)
    with pytest.raises(L.CapacityError):
        L.build_mask(ctx, [0], N, pk, rng)
    ct = L.pack_and_encrypt(ctx, np.full(10, 0.25), pk, rng)
    short = L.SecretKey(orc.secret_key()[:2])
    with pytest.raises(L.KeyError):
        ctx.decrypt_values(L.Ciphertext(ct.chunks[0], ct.scale), short)
    vals = ctx.decrypt_values(L.Ciphertext(ct.chunks[0], ct.scale), L.SecretKey(orc.secret_key()))
    assert np.allclose(vals.cpu().numpy()[:10], 0.25, atol=1e-6)


@pytest.mark.parametrize("name", ["cfg1", "tiny_hoist_multikrum"])
def test_generate_keys_bit_exact(name):
    """generate_keys on the device with make_system's key sampler
    (derive_seed(1, 5)): secret, public, relinearization and every rotation
    key equal the reference's (golden-pinned oracle) word for word."""
    L = _L()
    rig = Rig(name, threads=8)
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    rng = L.Sampler(L.derive_seed(1, 5))
    sk, pk, rk, keys = L.generate_keys(ctx, rng, rig.steps)
    o = rig.oracle
    assert np.array_equal(sk.rows, o.secret_key())
    assert np.array_equal(pk.rows, o.public_key())
    assert np.array_equal(np.asarray(rk.key).ravel(), np.asarray(o.relin_key()).ravel())
    want = sorted({s % (rig.N // 2) for s in rig.steps} - {0})
    assert sorted(keys.steps) == want
    for st in want:
        assert np.array_equal(np.asarray(keys.steps[st]).ravel(),
                              np.asarray(o.rotation_key(st)).ravel()), st


def test_shape_and_width_errors():
    L = _L()
    orc = Oracle(256, secure=False, threads=1)
    orc.keygen(1, [1, 2, 4])
    ctx = gpu_ctx(256)
    cl = orc.make_clients(1, 3, 200)
    dev = L.to_device(cl)
    rk = L.RelinKey(orc.relin_key())
    keys = L.RotationKeySet({s: orc.rotation_key(s) for s in (1, 2, 4)})
    pw = [L.PackedWeights(dev[i], 200, 1.0, orc.scale) for i in range(3)]
    with pytest.raises(L.ShapeError):
        L.build_distance_matrix(ctx, pw[:1], rk, L.HoistPlan(k=1, n=128), L.DistanceMode.per_pair,
                                keys)
    with pytest.raises(L.WidthError):
        L.build_distance_matrix(ctx, pw, rk, L.HoistPlan(k=1, n=64), L.DistanceMode.per_pair, keys)
    with pytest.raises(L.KeyError):  # width 128 needs steps up to 64
        L.build_distance_matrix(ctx, pw, rk, L.HoistPlan(k=1, n=128), L.DistanceMode.per_pair,
                                keys)
    bad = L.PackedWeights(dev[2], 199, 1.0, orc.scale)
    with pytest.raises(L.ShapeError):
        L.build_distance_matrix(ctx, pw[:2] + [bad], rk, L.HoistPlan(k=1, n=128),
                                L.DistanceMode.per_pair, keys)
    with pytest.raises(L.ShapeError):
        L.masked_aggregate(ctx, pw, L.SelectionMask(2, 1, L.to_device(cl[:2, 0]), orc.scale),
                           L.SelectionRule.krum, rk)


@pytest.mark.parametrize("name,world", [("cfg1", 3), ("tiny_hoist_multikrum", 4)])
def test_cuda_shards_concatenate_to_reference(name, world):
    """The multi-GPU shard entry points (pair / chunk ranges) concatenate to
    the reference's matrix and aggregate word for word."""
    import torch

    from paper_2408_06197_b200.sharded import cuda_shard_fns, shard_range
    L = _L()
    rig = Rig(name, threads=8)
    ctx = gpu_ctx(rig.N, secure=bool(rig.meta["options"]["secure"]))
    ctx.use_relin_key(L.RelinKey(rig.oracle.relin_key()))
    keys = L.RotationKeySet({s: rig.oracle.rotation_key(s) for s in rig.meta["rot_keys"]})
    ctx.use_rotation_keys(keys, rig.meta["rot_keys"])
    clients = L.to_device(rig.clients)
    sel = L.to_device(rig.selectors)
    average = rig.average
    fp, fc, _, _ = cuda_shard_fns(ctx, clients, sel, rig.n, rig.C, rig.oracle.scale,
                                  rig.oracle.scale, rig.width, rig.k, l=len(rig.selected),
                                  average=average, lazy=rig.lazy)
    npairs = rig.n * (rig.n - 1) // 2
    d = torch.cat([fp(*shard_range(npairs, world, r)) for r in range(world)])
    a = torch.cat([fc(*shard_range(rig.C, world, r)) for r in range(world)])
    got = L.to_host(d)
    p = 0
    for i in range(rig.n):
        for j in range(i + 1, rig.n):
            assert sha(got[p]) == rig.meta["sha256"][f"dist_{i}_{j}"], (i, j)
            p += 1
    assert sha(L.to_host(a)) == rig.meta["sha256"]["agg"]


@pytest.mark.parametrize("pair_f64,n,C,blocked", [("1", 4, 600, "1"), ("0", 4, 600, "1"), ("1", 30, 3, "1"),
                                                   ("1", 7, 5, "1"), ("1", 48, 2, "1"), ("1", 48, 2, "0"),
                                                   ("0", 48, 2, "1")])
def test_pair_accumulation_long_ranges_and_extremes(pair_f64, n, C, blocked, monkeypatch):
    """Lazy pair accumulation over 600 chunks (three 256-chunk passes of the
    FP64-pipe kernel), over 435 pairs (three CTA pair groups, 30 clients) and
    over 1128 pairs (48 clients: more pairs than one key-switch sub-batch, so
    every pair is accumulated in one pass and finished per sub-batch; with
    client-blocked pair groups above 27 clients, LCL_PAIR_BLOCKED=0 the flat
    ones), with boundary residues (all 0 against all q-1), for both arithmetic forms
    (LCL_PAIR_F64=1: FP64 pipe, 0: split-23 integer), odd n included, word
    for word against the oracle's distance matrix."""
    L = _L()
    monkeypatch.setenv("LCL_PAIR_F64", pair_f64)
    monkeypatch.setenv("LCL_PAIR_BLOCKED", blocked)
    N = 256
    orc = Oracle(N, secure=False, threads=8)
    width = 128
    steps = slot_reduce_steps(width, 1)
    orc.keygen(3, steps)
    rng = np.random.default_rng(7)
    m = orc.full
    clients = np.zeros((n, C, 2, m, N), np.uint64)
    for r in range(m):
        q = orc.primes[r]
        clients[1, :, :, r] = np.uint64(q - 1)
        clients[2, :, :, r] = rng.integers(0, q, size=(C, 2, N), dtype=np.uint64)
        clients[3, :, :, r] = rng.integers(q - 4096, q, size=(C, 2, N), dtype=np.uint64)
        for i in range(4, n):
            clients[i, :, :, r] = rng.integers(0, q, size=(C, 2, N), dtype=np.uint64)
    ctx = L.CkksContext(L.CkksParams(ring_degree=N, security=L.SecurityLevel.none))
    rk = L.RelinKey(orc.relin_key())
    keys = L.RotationKeySet({s: orc.rotation_key(s) for s in steps})
    dev = L.to_device(clients)
    pw = [L.PackedWeights(dev[i], C * (N // 2), 1.0, orc.scale) for i in range(n)]
    dm = L.build_distance_matrix(ctx, pw, rk, L.HoistPlan(k=1, n=width),
                                 L.DistanceMode.per_pair, keys, L.DistanceOptions())
    want = orc.distance_matrix(clients, width, 1)
    assert np.array_equal(L.to_host(dm.batch), want)


@pytest.mark.parametrize("n", [60, 190])
def test_pair_ranges_of_many_clients(n):
    """Client-blocked pair groups for ANY pair set: pair
    sub-ranges of 60 and 190 clients (lcl_distance_matrix_pairs, unreduced:
    accumulation + relinearize + rescale) and the whole 190-client matrix's
    lazy partials (lcl_pair_partials) equal the oracle's -- a CTA never stages
    more than 26 clients, so there is no client-count limit (formerly
    'too many clients for one tile' from 178 clients)."""
    L = _L()
    import ctypes as C
    import torch
    N = 256
    orc = Oracle(N, secure=False, threads=8)
    orc.keygen(3, [])
    rng = np.random.default_rng(n)
    m = orc.full
    Cc = 2
    clients = np.zeros((n, Cc, 2, m, N), np.uint64)
    for r in range(m):
        clients[:, :, :, r] = rng.integers(0, orc.primes[r], size=(n, Cc, 2, N), dtype=np.uint64)
    ctx = L.CkksContext(L.CkksParams(ring_degree=N, security=L.SecurityLevel.none))
    ctx.use_relin_key(L.RelinKey(orc.relin_key()))
    dev = L.to_device(clients)
    P = n * (n - 1) // 2
    osc = C.c_double()
    for a, b in ((0, 37), (P // 3, P // 3 + 500), (P - 70, P)):
        out = torch.empty((b - a, 2, m - 1, N), dtype=torch.int64, device="cuda")
        L._check(L.lib().lcl_distance_matrix_pairs(ctx.h, L._ptr(dev), n, Cc, orc.scale, 1, 1, 1, 0,
                                                   a, b, L._ptr(out), C.byref(osc)))
        got = L.to_host(out)
        pairs = [(i, j) for i in range(n) for j in range(i + 1, n)][a:b]
        for q in range(0, b - a, 23):
            i, j = pairs[q]
            assert np.array_equal(got[q], orc.pairwise_distance(clients[i], clients[j])), (a, q)
    if n == 190:
        t = torch.empty((P, 3, m, N), dtype=torch.int64, device="cuda")
        L._check(L.lib().lcl_pair_partials(ctx.h, L._ptr(dev), n, Cc, L._ptr(t)))
        got = L.to_host(t)
        pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
        for q in range(0, P, 997):
            i, j = pairs[q]
            acc = orc.hsquare(orc.hsub(clients[i, 0], clients[j, 0]))
            orc.lazy_accumulate(acc, orc.hsquare(orc.hsub(clients[i, 1], clients[j, 1])))
            assert np.array_equal(got[q], acc), q


def test_cfg3_benchmark_round_bit_exact_vs_reference():
    """BASELINE configs[2] exactly as bench.py times it: 20 clients x
    11,173,962 params (342 chunks), N = 2^16, lazy relin, hoisted rotations
    at the bench plan's k = 3 (fused modup_ip_hoist), Krum mask. Keys,
    client ciphertexts and the mask are produced on the device from the
    reference's seeds (word-identical: their digests are checked against the
    reference's own dump), then the distance matrix, the aggregate, the op
    counters and every decrypted slot-0 distance are checked against the
    reference run (tests/golden/cfg3_hoist.json)."""
    import hashlib
    import os

    import torch

    L = _L()
    from tests.golden_util import load
    meta = load("cfg3_hoist")
    o = meta["options"]
    N, n, dim, k = o["N"], o["clients"], o["dim"], o["k"]
    d = meta["sha256"]

    def dsha(t):
        h = hashlib.sha256()
        h.update(t.cpu().numpy().tobytes())
        return h.hexdigest()

    ctx = gpu_ctx(N, secure=True)
    width = 1 << (min(dim, N // 2) - 1).bit_length()
    assert L.slot_reduce_steps(width, k) == meta["steps"]
    sk, pk, rk, keys = L.generate_keys(ctx, L.Sampler(L.derive_seed(1, 5)), meta["steps"])
    assert sha(np.asarray(rk.key)) == d["relin"]
    rng = L.Sampler(L.derive_seed(1, 0xAB1A7E))
    C_ = -(-dim // (N // 2))
    assert C_ == meta["chunks"] == 342
    big = torch.empty((n, C_, 2, ctx.full, N), dtype=torch.int64, device="cuda")
    for i in range(n):
        w = rng.uniform_real(dim) - 0.5
        pw = L.pack_and_encrypt(ctx, w, pk, rng)
        big[i].copy_(pw.chunks)
        del pw
        assert dsha(big[i]) == d[f"client_{i}"], i
    _, sels = L.build_mask(ctx, [0], n, pk, L.Sampler(L.derive_seed(1, 0x3000000000000000)))
    for i in range(n):
        assert dsha(sels[i]) == d[f"sel_{i}"], i
    pws = [L.PackedWeights(big[i], dim, 1.0, ctx.scale()) for i in range(n)]
    assert L.stack_clients(pws).data_ptr() == big.data_ptr()
    ctx.reset_counters()
    dm = L.build_distance_matrix(ctx, pws, rk, L.HoistPlan(k=k, n=width),
                                 L.DistanceMode.per_pair, keys, L.DistanceOptions())
    torch.cuda.synchronize()
    assert ctx.counters() == meta["dist_ops"]
    for p, (i, j) in enumerate(dm.keys):
        assert dsha(dm.batch[p]) == d[f"dist_{i}_{j}"], (i, j)
    vals = ctx.decrypt_values_batch(dm.batch, dm.scale, sk).cpu().numpy()
    for p, e in enumerate(meta["dist"]):
        assert vals[p][0] == e["slot0"], p
        assert abs(vals[p][0] - meta["plain_dist"][p]) <= 1e-3 * max(1.0, abs(meta["plain_dist"][p]))
    mask = L.SelectionMask(n, 1, sels, ctx.scale())
    ctx.reset_counters()
    agg = L.masked_aggregate(ctx, pws, mask, L.SelectionRule.krum, rk)
    torch.cuda.synchronize()
    assert ctx.counters() == meta["agg_ops"]
    assert dsha(agg.chunks) == d["agg"]
    assert agg.scale == meta["agg_scale"]
    # the same round through the host entry, pinned buffers in and out (the
    # bench's e2e form at its own shape: the last group's aggregate in chunk
    # slices, n / 4 single-client tail groups on high-priority lanes)
    import ctypes as C
    h_clients = torch.empty(big.shape, dtype=torch.int64, pin_memory=True)
    h_clients.copy_(big)
    del big
    torch.cuda.empty_cache()
    h_sel = torch.empty((n,) + tuple(sels[0].shape), dtype=torch.int64, pin_memory=True)
    for i in range(n):
        h_sel[i].copy_(sels[i])
    m = ctx.full
    h_dist = torch.empty((n * (n - 1) // 2, 2, m - 1, N), dtype=torch.int64, pin_memory=True)
    h_agg = torch.empty((C_, 2, m - 1, N), dtype=torch.int64, pin_memory=True)
    ctx.use_relin_key(rk)
    ctx.use_rotation_keys(keys, meta["steps"])
    ctx.reset_counters()
    L._check(L.lib().lcl_server_round_host(
        ctx.h, C.c_void_p(h_clients.data_ptr()), C.c_void_p(h_sel.data_ptr()), n, C_,
        ctx.scale(), width, k, 1, 0, C.c_void_p(h_dist.data_ptr()), C.c_void_p(h_agg.data_ptr())))
    for p, (i, j) in enumerate(dm.keys):
        assert dsha(h_dist[p]) == d[f"dist_{i}_{j}"], (i, j)
    assert dsha(h_agg) == d["agg"]
    want = {key: meta["dist_ops"][key] + meta["agg_ops"][key] for key in meta["dist_ops"]}
    assert ctx.counters() == want
    del h_clients, h_sel, h_dist, h_agg
