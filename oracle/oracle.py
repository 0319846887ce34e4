"""ctypes view of the plain-C oracle (oracle/lancelot_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py as the CHECKER. The product
(paper_2408_06197_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liblancelot_oracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")

_u64p = C.POINTER(C.c_uint64)
_szp = C.POINTER(C.c_size_t)


class Counts(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in (
        "encryptions", "additions", "multiplications", "relinearizations",
        "rescales", "rotations", "mod_ups")]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


def build():
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)


def _lib():
    if not os.path.exists(LIB_PATH):
        build()
    lib = C.CDLL(LIB_PATH)
    lib.lo_ctx_new.restype = C.c_void_p
    lib.lo_ctx_new.argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_int]
    lib.lo_ctx_free.argtypes = [C.c_void_p]
    for f in ("lo_degree", "lo_prime_count", "lo_key_words"):
        getattr(lib, f).restype = C.c_size_t
        getattr(lib, f).argtypes = [C.c_void_p]
    lib.lo_prime.restype = C.c_uint64
    lib.lo_prime.argtypes = [C.c_void_p, C.c_size_t]
    lib.lo_psi.restype = C.c_uint64
    lib.lo_psi.argtypes = [C.c_void_p, C.c_size_t]
    lib.lo_scale.restype = C.c_double
    lib.lo_scale.argtypes = [C.c_void_p]
    lib.lo_get_counts.restype = Counts
    lib.lo_get_counts.argtypes = [C.c_void_p]
    lib.lo_reset_counts.argtypes = [C.c_void_p]
    lib.lo_ntt_forward.argtypes = [C.c_void_p, _u64p, C.c_size_t]
    lib.lo_ntt_inverse.argtypes = [C.c_void_p, _u64p, C.c_size_t]
    lib.lo_ntt_tables.argtypes = [C.c_void_p, C.c_size_t] + [_u64p] * 5
    lib.lo_galois_perm.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_uint32)]
    lib.lo_galois_elt.restype = C.c_uint64
    lib.lo_galois_elt.argtypes = [C.c_size_t, C.c_size_t]
    lib.lo_keygen.argtypes = [C.c_void_p, C.c_uint64, _szp, C.c_size_t]
    for f in ("lo_relin_key", "lo_secret_key", "lo_public_key_p0", "lo_public_key_p1"):
        getattr(lib, f).restype = C.c_void_p
        getattr(lib, f).argtypes = [C.c_void_p]
    lib.lo_rotation_key.restype = C.c_void_p
    lib.lo_rotation_key.argtypes = [C.c_void_p, C.c_size_t]
    lib.lo_make_clients.argtypes = [C.c_void_p, C.c_uint64, C.c_size_t, C.c_size_t,
                                    C.c_double, _u64p]
    lib.lo_chunk_count.restype = C.c_size_t
    lib.lo_chunk_count.argtypes = [C.c_void_p, C.c_size_t]
    lib.lo_build_mask.argtypes = [C.c_void_p, C.c_uint64, _szp, C.c_size_t, C.c_size_t, _u64p]
    lib.lo_hsub.argtypes = [C.c_void_p, C.c_size_t, _u64p, _u64p, _u64p]
    lib.lo_hadd.argtypes = [C.c_void_p, C.c_size_t, _u64p, _u64p, _u64p]
    lib.lo_hsquare.argtypes = [C.c_void_p, C.c_size_t, _u64p, _u64p]
    lib.lo_hmult_triple.argtypes = [C.c_void_p, C.c_size_t, _u64p, _u64p, _u64p]
    lib.lo_lazy_accumulate.argtypes = [C.c_void_p, C.c_size_t, _u64p, _u64p]
    lib.lo_relinearize.argtypes = [C.c_void_p, C.c_size_t, _u64p, _u64p]
    lib.lo_rescale.argtypes = [C.c_void_p, C.c_size_t, _u64p, _u64p]
    lib.lo_rotate.argtypes = [C.c_void_p, C.c_size_t, _u64p, C.c_size_t, _u64p]
    lib.lo_hoisted_rotations.argtypes = [C.c_void_p, C.c_size_t, _u64p, _szp, C.c_size_t, _u64p]
    lib.lo_slot_reduce.argtypes = [C.c_void_p, C.c_size_t, _u64p, C.c_size_t, C.c_size_t, _u64p]
    lib.lo_mult_plain_inv_l.argtypes = [C.c_void_p, C.c_size_t, _u64p, C.c_size_t, _u64p]
    lib.lo_encode.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_size_t, C.c_double,
                              C.c_int, _u64p]
    lib.lo_pairwise_distance.argtypes = [C.c_void_p, C.c_size_t, _u64p, _u64p, C.c_int, _u64p]
    lib.lo_distance_matrix.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, _u64p, C.c_size_t,
                                       C.c_size_t, C.c_int, C.c_int, _u64p]
    lib.lo_distance_rows.argtypes = lib.lo_distance_matrix.argtypes
    lib.lo_masked_aggregate.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, _u64p, _u64p,
                                        C.c_size_t, C.c_int, _u64p]
    lib.lo_decrypt_values.argtypes = [C.c_void_p, C.c_size_t, _u64p, C.c_double,
                                      C.POINTER(C.c_double)]
    lib.lo_derive_seed.restype = C.c_uint64
    lib.lo_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
    return lib


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = _lib()
    return _LIB


def _p(a):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(_u64p)


class OracleError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"oracle {where} failed with code {code}")
        self.code = code


def _chk(rc, where):
    if rc:
        raise OracleError(rc, where)


class Oracle:
    """One oracle CkksContext plus keys, mirroring the reference's CkksContext."""

    def __init__(self, N, depth=3, secure=False, threads=None):
        L = lib()
        threads = threads or os.cpu_count() or 1
        self.h = L.lo_ctx_new(N, depth, int(bool(secure)), threads)
        if not self.h:
            raise OracleError(1, "ctx_new")
        self.N = N
        self.depth = depth
        self.full = L.lo_prime_count(self.h)
        self.primes = [L.lo_prime(self.h, i) for i in range(self.full)]
        self.special = L.lo_prime(self.h, self.full)
        self.psi = [L.lo_psi(self.h, i) for i in range(self.full + 1)]
        self.slots = N // 2
        self.scale = L.lo_scale(self.h)
        self.steps = []

    def __del__(self):
        try:
            lib().lo_ctx_free(self.h)
        except Exception:
            pass

    # --- tables / transforms
    def ntt_forward(self, row, prime_index):
        r = np.ascontiguousarray(row, dtype=np.uint64).copy()
        lib().lo_ntt_forward(self.h, _p(r), prime_index)
        return r

    def ntt_inverse(self, row, prime_index):
        r = np.ascontiguousarray(row, dtype=np.uint64).copy()
        lib().lo_ntt_inverse(self.h, _p(r), prime_index)
        return r

    def ntt_tables(self, i):
        out = [np.zeros(self.N, np.uint64) for _ in range(4)]
        ni = np.zeros(2, np.uint64)
        lib().lo_ntt_tables(self.h, i, *[_p(o) for o in out], _p(ni))
        return out + [ni]

    def galois_perm(self, step):
        p = np.zeros(self.N, np.uint32)
        lib().lo_galois_perm(self.h, step, p.ctypes.data_as(C.POINTER(C.c_uint32)))
        return p

    # --- keys and inputs
    def keygen(self, seed, steps):
        self.steps = list(steps)
        arr = (C.c_size_t * max(1, len(steps)))(*steps)
        _chk(lib().lo_keygen(self.h, seed, arr, len(steps)), "keygen")

    def _key(self, ptr):
        if not ptr:
            return None
        words = lib().lo_key_words(self.h)
        buf = (C.c_uint64 * words).from_address(ptr)
        return np.frombuffer(buf, dtype=np.uint64).reshape(
            self.full, 2, self.full + 1, self.N).copy()

    def relin_key(self):
        return self._key(lib().lo_relin_key(self.h))

    def rotation_key(self, step):
        return self._key(lib().lo_rotation_key(self.h, step))

    def public_key(self):
        """(p0, p1) stacked: [2][full][N], evaluation domain."""
        out = np.empty((2, self.full, self.N), np.uint64)
        for x, f in enumerate((lib().lo_public_key_p0, lib().lo_public_key_p1)):
            buf = (C.c_uint64 * (self.full * self.N)).from_address(f(self.h))
            out[x] = np.frombuffer(buf, dtype=np.uint64).reshape(self.full, self.N)
        return out

    def secret_key(self):
        ptr = lib().lo_secret_key(self.h)
        buf = (C.c_uint64 * ((self.full + 1) * self.N)).from_address(ptr)
        return np.frombuffer(buf, dtype=np.uint64).reshape(self.full + 1, self.N).copy()

    def chunk_count(self, dim):
        return lib().lo_chunk_count(self.h, dim)

    def make_clients(self, seed, clients, dim, prescale=1.0):
        Cc = self.chunk_count(dim)
        out = np.zeros((clients, Cc, 2, self.full, self.N), np.uint64)
        _chk(lib().lo_make_clients(self.h, seed, clients, dim, prescale, _p(out)), "make_clients")
        return out

    def build_mask(self, seed, selected, n):
        out = np.zeros((n, 2, self.full, self.N), np.uint64)
        arr = (C.c_size_t * max(1, len(selected)))(*selected)
        _chk(lib().lo_build_mask(self.h, seed, arr, len(selected), n, _p(out)), "build_mask")
        return out

    # --- counters
    def counts(self):
        return lib().lo_get_counts(self.h).as_dict()

    def reset_counts(self):
        lib().lo_reset_counts(self.h)

    # --- evaluator (count = live q limbs of the input)
    def _ct(self, a):
        return np.ascontiguousarray(a, dtype=np.uint64)

    def hsub(self, a, b):
        a, b = self._ct(a), self._ct(b)
        out = np.empty_like(a)
        lib().lo_hsub(self.h, a.shape[-2], _p(a), _p(b), _p(out))
        return out

    def hadd(self, a, b):
        a, b = self._ct(a), self._ct(b)
        out = np.empty_like(a)
        lib().lo_hadd(self.h, a.shape[-2], _p(a), _p(b), _p(out))
        return out

    def hsquare(self, a):
        a = self._ct(a)
        m = a.shape[-2]
        out = np.empty((3, m, self.N), np.uint64)
        lib().lo_hsquare(self.h, m, _p(a), _p(out))
        return out

    def hmult_triple(self, a, b):
        a, b = self._ct(a), self._ct(b)
        m = a.shape[-2]
        out = np.empty((3, m, self.N), np.uint64)
        lib().lo_hmult_triple(self.h, m, _p(a), _p(b), _p(out))
        return out

    def lazy_accumulate(self, acc, t):
        t = self._ct(t)
        lib().lo_lazy_accumulate(self.h, acc.shape[-2], _p(acc), _p(t))
        return acc

    def relinearize(self, t):
        t = self._ct(t)
        m = t.shape[-2]
        out = np.empty((2, m, self.N), np.uint64)
        _chk(lib().lo_relinearize(self.h, m, _p(t), _p(out)), "relinearize")
        return out

    def rescale(self, ct):
        ct = self._ct(ct)
        m = ct.shape[-2]
        out = np.empty((2, m - 1, self.N), np.uint64)
        _chk(lib().lo_rescale(self.h, m, _p(ct), _p(out)), "rescale")
        return out

    def rotate(self, ct, step):
        ct = self._ct(ct)
        out = np.empty_like(ct)
        _chk(lib().lo_rotate(self.h, ct.shape[-2], _p(ct), step, _p(out)), "rotate")
        return out

    def hoisted_rotations(self, ct, steps):
        ct = self._ct(ct)
        out = np.empty((len(steps),) + ct.shape, np.uint64)
        arr = (C.c_size_t * max(1, len(steps)))(*steps)
        _chk(lib().lo_hoisted_rotations(self.h, ct.shape[-2], _p(ct), arr, len(steps), _p(out)),
             "hoisted_rotations")
        return out

    def slot_reduce(self, ct, width, k):
        ct = self._ct(ct)
        out = np.empty_like(ct)
        _chk(lib().lo_slot_reduce(self.h, ct.shape[-2], _p(ct), width, k, _p(out)), "slot_reduce")
        return out

    def mult_plain_inv_l(self, ct, l):
        ct = self._ct(ct)
        m = ct.shape[-2]
        out = np.empty((2, m - 1, self.N), np.uint64)
        _chk(lib().lo_mult_plain_inv_l(self.h, m, _p(ct), l, _p(out)), "mult_plain_inv_l")
        return out

    def encode(self, values, scale, level):
        v = np.ascontiguousarray(values, dtype=np.float64)
        out = np.zeros((level + 1, self.N), np.uint64)
        _chk(lib().lo_encode(self.h, v.ctypes.data_as(C.POINTER(C.c_double)), len(v), scale,
                             level, _p(out)), "encode")
        return out

    def pairwise_distance(self, a, b, lazy=True):
        a, b = self._ct(a), self._ct(b)
        out = np.empty((2, self.full - 1, self.N), np.uint64)
        _chk(lib().lo_pairwise_distance(self.h, a.shape[0], _p(a), _p(b), int(lazy), _p(out)),
             "pairwise_distance")
        return out

    def distance_matrix(self, clients, width, k, lazy=True, reduce=True):
        clients = self._ct(clients)
        n, Cc = clients.shape[0], clients.shape[1]
        out = np.empty((n * (n - 1) // 2, 2, self.full - 1, self.N), np.uint64)
        _chk(lib().lo_distance_matrix(self.h, n, Cc, _p(clients), width, k, int(lazy),
                                      int(reduce), _p(out)), "distance_matrix")
        return out

    def distance_rows(self, clients, width, k, lazy=True, reduce=True):
        """DistanceMode::row_sums: [n][2][L][N]."""
        clients = self._ct(clients)
        n, Cc = clients.shape[0], clients.shape[1]
        out = np.empty((n, 2, self.full - 1, self.N), np.uint64)
        _chk(lib().lo_distance_rows(self.h, n, Cc, _p(clients), width, k, int(lazy),
                                    int(reduce), _p(out)), "distance_rows")
        return out

    def masked_aggregate(self, clients, selectors, l=1, average=False):
        clients, selectors = self._ct(clients), self._ct(selectors)
        n, Cc = clients.shape[0], clients.shape[1]
        m_out = self.full - (2 if average else 1)
        out = np.empty((Cc, 2, m_out, self.N), np.uint64)
        _chk(lib().lo_masked_aggregate(self.h, n, Cc, _p(clients), _p(selectors), l,
                                       int(average), _p(out)), "masked_aggregate")
        return out

    def decrypt_values(self, ct, scale):
        ct = self._ct(ct)
        out = np.empty(self.slots, np.float64)
        lib().lo_decrypt_values(self.h, ct.shape[-2], _p(ct), scale,
                                out.ctypes.data_as(C.POINTER(C.c_double)))
        return out


def derive_seed(root, tag):
    return lib().lo_derive_seed(root, tag)


def slot_reduce_steps(width, k):
    """slot_reduce_steps (distance.cpp:199-212)."""
    levels = width.bit_length() - 1
    unf = min(k - 1, levels)
    return list(range(1, 1 << unf)) + [1 << j for j in range(unf, levels)]
