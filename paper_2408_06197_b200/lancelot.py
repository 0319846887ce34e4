"""Host-side mirror of the reference's server API, backed by the sm_100a library.

Names, argument meaning and error behaviour follow the reference C++ API of
Lancelot's server path (/root/reference/proj/core):

    CkksParams / CkksContext          ckks.hpp:39-55, 146-222
    Ciphertext / TernaryCiphertext    ckks.hpp:99-114
    RelinKey / RotationKeySet         ckks.hpp:73-83
    PackedWeights, chunk_count_for, distance_prescale       distance.hpp:31-49
    encrypted_pairwise_distance       distance.hpp:57-65
    HoistPlan, plan_unfold, fixed_plan, slot_reduce_steps, slot_reduce
                                      distance.hpp:67-99
    DistanceMode, EncryptedDistanceMatrix, DistanceOptions, build_distance_matrix
                                      distance.hpp:101-126
    SelectionRule, SelectionMask, masked_aggregate          aggregation.hpp:38-93
    exception hierarchy               errors.hpp:27-104

Ciphertext words live in HBM as torch int64 tensors (raw u64 bit patterns,
limb-major [2][count][N]). Every computation goes through the C-ABI in
include/lancelot_b200.h; there is no CPU fallback: without the built library
or a CUDA device the calls raise.
"""
from __future__ import annotations

import builtins
import ctypes as C
import math
import os
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# LCL_LIB_PATH: an alternative in-tree build for A/B experiments (tools/)
LIB_PATH = os.environ.get("LCL_LIB_PATH") or os.path.join(HERE, "_lib", "liblancelot_b200.so")


# --------------------------------------------------------------- errors
class Error(RuntimeError):
    """Base of every failure the library raises (errors.hpp:27-31)."""


class ParameterError(Error):
    pass


class BasisMismatchError(Error):
    pass


class DomainError(Error):
    pass


class AlignmentError(Error):
    pass


class KeyError(Error):  # noqa: A001 - mirrors lancelot::KeyError
    pass


class DepthExhaustedError(Error):
    pass


class CapacityError(Error):
    pass


class ShapeError(Error):
    pass


class WidthError(Error):
    pass


class InfeasibleError(Error):
    pass


class DataError(Error):
    pass


class UsageError(Error):
    pass


class DeviceError(Error):
    """CUDA failure (no reference counterpart)."""


_CODES = {1: ParameterError, 2: BasisMismatchError, 3: DomainError, 4: AlignmentError,
          5: KeyError, 6: DepthExhaustedError, 7: CapacityError, 8: ShapeError, 9: WidthError,
          10: InfeasibleError, 11: DataError, 12: UsageError, 100: DeviceError}


class Counts(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in (
        "encryptions", "additions", "multiplications", "relinearizations", "rescales",
        "rotations", "mod_ups")]

    def as_dict(self):
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


# --------------------------------------------------------------- library
_LIB = None
_P = C.c_void_p
_SZ = C.c_size_t


def lib():
    """Load the in-tree CUDA library; raise loudly when it is missing."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    sig = {
        "lcl_context_create": [_SZ, C.c_int, C.c_int, C.c_int, C.POINTER(_P)],
        "lcl_context_destroy": [_P],
        "lcl_context_primes": [_P, C.POINTER(C.c_uint64), C.POINTER(_SZ)],
        "lcl_set_stream": [_P, _P],
        "lcl_synchronize": [_P],
        "lcl_get_counts": [_P, C.POINTER(Counts)],
        "lcl_reset_counts": [_P],
        "lcl_upload_relin_key": [_P, _P, _SZ],
        "lcl_upload_rotation_key": [_P, _SZ, _P, _SZ],
        "lcl_has_rotation_key": [_P, _SZ],
        "lcl_ntt_forward": [_P, _P, _SZ, _SZ, C.c_int],
        "lcl_ntt_inverse": [_P, _P, _SZ, _SZ, C.c_int],
        "lcl_hadd": [_P, _P, _P, _SZ, _SZ, _P],
        "lcl_hsub": [_P, _P, _P, _SZ, _SZ, _P],
        "lcl_sampler_create": [C.c_uint64, C.POINTER(C.c_void_p)],
        "lcl_sampler_destroy": [_P],
        "lcl_sampler_uniform_real": [_P, _SZ, _P],
        "lcl_pack_and_encrypt": [_P, _P, _P, _SZ, C.c_double, _P, _P],
        "lcl_build_mask": [_P, _P, _SZ, _P, _SZ, _P, _P, _P],
        "lcl_generate_keys": [_P, _P, _P, _SZ, _P, _P, _P, _P, _P, _P],
        "lcl_server_round": [_P, _P, _P, _SZ, _SZ, _SZ, _SZ, _SZ, C.c_int, _P, _P],
        "lcl_pair_partials": [_P, _P, _SZ, _SZ, _P],
        "lcl_pair_combine": [_P, _P, _SZ, _SZ],
        "lcl_pair_finish": [_P, _P, _SZ, _SZ, _SZ, C.c_int, _P],
        "lcl_decrypt": [_P, _P, _SZ, _SZ, _P, _P],
        "lcl_decode": [_P, _P, _SZ, _SZ, C.c_double, _P],
        "lcl_decrypt_values": [_P, _P, _SZ, _SZ, C.c_double, _P, _P],
        "lcl_hmult": [_P, _P, _P, _SZ, _SZ, _P],
        "lcl_hsquare": [_P, _P, _SZ, _SZ, _P],
        "lcl_relinearize": [_P, _P, _SZ, _SZ, _P],
        "lcl_rescale": [_P, _P, _SZ, _SZ, _P],
        "lcl_rotate": [_P, _P, _SZ, _SZ, _SZ, _P],
        "lcl_hoisted_rotations": [_P, _P, _SZ, _SZ, C.POINTER(_SZ), _SZ, _P],
        "lcl_slot_reduce": [_P, _P, _SZ, _SZ, _SZ, _SZ, _P],
        "lcl_mult_plain_const": [_P, _P, _SZ, _SZ, C.c_double, C.c_double, _P],
        "lcl_pairwise_distance": [_P, _P, _P, _SZ, C.c_int, _P],
        "lcl_distance_matrix": [_P, _P, _SZ, _SZ, C.c_double, _SZ, _SZ, C.c_int, C.c_int, _P,
                                C.POINTER(C.c_double)],
        "lcl_deserialize": [_P, _P, _SZ, _SZ, _SZ, _P, C.POINTER(C.c_double)],
        "lcl_serialize": [_P, _P, _SZ, _SZ, C.c_double, _P, _SZ],
        "lcl_server_round_lclt": [_P, _P, _P, _SZ, _SZ, _SZ, _SZ, _SZ, _SZ, _SZ, C.c_int, _P, _P,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)],
        "lcl_table_from_matrix": [_P, _P, _SZ, _SZ, C.c_double, C.c_int, C.c_double, _P, _P],
        "lcl_totals_from_matrix": [_P, _P, _SZ, C.c_int, _SZ, C.c_double, C.c_int, C.c_double, _P,
                                   _P],
        "lcl_calibrate": [_P, _P, _SZ, C.POINTER(C.c_double), C.POINTER(C.c_double),
                          C.POINTER(C.c_double)],
        "lcl_build_distance_matrix": [_P, _P, _SZ, _SZ, C.c_double, _SZ, _SZ, C.c_int, C.c_int,
                                      C.c_int, _P, C.POINTER(C.c_double)],
        "lcl_masked_aggregate": [_P, _P, _P, _SZ, _SZ, C.c_double, C.c_double, _SZ, C.c_int, _P,
                                 C.POINTER(C.c_double)],
        "lcl_server_round_host": [_P, _P, _P, _SZ, _SZ, C.c_double, _SZ, _SZ, _SZ, C.c_int, _P,
                                  _P],
        "lcl_distance_matrix_pairs": [_P, _P, _SZ, _SZ, C.c_double, _SZ, _SZ, C.c_int, C.c_int,
                                      _SZ, _SZ, _P, C.POINTER(C.c_double)],
        "lcl_masked_aggregate_chunks": [_P, _P, _P, _SZ, _SZ, C.c_double, C.c_double, _SZ, C.c_int,
                                        _SZ, _SZ, _P, C.POINTER(C.c_double)],
        "lcl_profile_begin": [_P],
        "lcl_profile_end": [_P, C.c_char_p, _SZ],
        "lcl_peak_butterflies": [_P, C.POINTER(C.c_double)],
        "lcl_peak_butterflies_f64": [_P, C.POINTER(C.c_double)],
        "lcl_device_alloc": [_P, _SZ, C.POINTER(_P)],
        "lcl_device_free": [_P, _P],
        "lcl_copy_h2d": [_P, _P, _P, _SZ],
        "lcl_copy_d2h": [_P, _P, _P, _SZ],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.lcl_last_error.restype = C.c_char_p
    L.lcl_last_error.argtypes = []
    L.lcl_launch_count.restype = C.c_uint64
    L.lcl_launch_count.argtypes = [_P]
    _LIB = L
    return L


def exported_symbols():
    """Names every C-ABI entry point declared in include/lancelot_b200.h."""
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "lancelot_b200.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(lcl_[a-z0-9_]+)\s*\(", text)))


def _check(rc):
    if rc != 0:
        msg = lib().lcl_last_error().decode(errors="replace")
        raise _CODES.get(rc, Error)(msg)


def _torch():
    import torch
    return torch


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def to_device(arr, device="cuda"):
    """numpy uint64 array -> torch int64 tensor on the device (bit pattern kept)."""
    torch = _torch()
    a = np.ascontiguousarray(arr, dtype=np.uint64)
    return torch.from_numpy(a.view(np.int64)).to(device)


def to_host(t):
    """torch int64 device tensor -> numpy uint64 array."""
    return t.detach().cpu().contiguous().numpy().view(np.uint64)


# --------------------------------------------------------------- parameters
class SecurityLevel(Enum):
    none = 0
    bits128 = 1


@dataclass
class CkksParams:
    """CkksParams (ckks.hpp:39-55). Only the defaults of the prime sizes are
    supported by the device basis (q0 44, scale 40, special 54 bits)."""
    ring_degree: int = 8192
    depth: int = 3
    scale_bits: int = 40
    first_prime_bits: int = 44
    special_prime_bits: int = 54
    security: SecurityLevel = SecurityLevel.bits128
    key_hamming_weight: int = 64
    error_eta: int = 21
    message_bound: float = float(1 << 20)

    def scale(self):
        return math.pow(2.0, self.scale_bits)

    def validate(self):
        n = self.ring_degree
        if n < 8 or n & (n - 1):
            raise ParameterError("ring degree must be a power of two >= 8")
        if self.depth < 0 or self.depth > 40:
            raise ParameterError("depth outside supported range")
        if (self.scale_bits, self.first_prime_bits, self.special_prime_bits) != (40, 44, 54):
            raise ParameterError("device basis supports the default 44/40/54-bit chain")


# --------------------------------------------------------------- data types
@dataclass
class Ciphertext:
    """(c0, c1) in evaluation domain: data = [2][count][N] int64 on the device."""
    data: object
    scale: float

    def level(self):
        return int(self.data.shape[-2]) - 1

    def size_bytes(self):
        return int(self.data.numel()) * 8


@dataclass
class TernaryCiphertext:
    data: object  # [3][count][N]
    scale: float
    accumulated: int = 1

    def level(self):
        return int(self.data.shape[-2]) - 1


@dataclass
class RelinKey:
    key: np.ndarray  # [full][2][full+1][N] host words


@dataclass
class RotationKeySet:
    steps: dict = field(default_factory=dict)  # step -> [full][2][full+1][N]

    def has_step(self, step):
        return step in self.steps


@dataclass
class PackedWeights:
    """Chunked encrypted weight vector (distance.hpp:31-38); chunks = [C][2][full][N]."""
    chunks: object
    dimension: int
    prescale: float = 1.0
    scale: float = 0.0

    def chunk_count(self):
        return int(self.chunks.shape[0])


def derive_seed(root: int, tag: int) -> int:
    """derive_seed (sampling.cpp:24-30)."""
    lib().lcl_derive_seed.restype = C.c_uint64
    lib().lcl_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
    return int(lib().lcl_derive_seed(root, tag))


class Sampler:
    """Sampler(seed) (sampling.hpp:32-65): the reference's mt19937_64 stream."""

    def __init__(self, seed: int):
        h = C.c_void_p()
        _check(lib().lcl_sampler_create(C.c_uint64(seed), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().lcl_sampler_destroy(self.h)
            self.h = None

    def uniform_real(self, count: int):
        out = np.empty(count, np.float64)
        _check(lib().lcl_sampler_uniform_real(self.h, count, out.ctypes.data))
        return out


class PublicKey:
    """PublicKey (ckks.hpp:62-66): (p0, p1) rows over the full chain,
    evaluation domain, as one [2][full][N] array."""

    def __init__(self, rows):
        self.rows = np.ascontiguousarray(rows, dtype=np.uint64)
        self._dev = None

    def device(self):
        if self._dev is None:
            self._dev = to_device(self.rows)
        return self._dev


def pack_and_encrypt(ctx: "CkksContext", weights, pk: PublicKey, rng: Sampler,
                     prescale: float = 1.0) -> "PackedWeights":
    """distance.cpp:64-91 on the device: the weights chunked into slots,
    encoded and encrypted, consuming rng's draws as the reference does."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if w.size == 0:
        raise ShapeError("empty weight vector")
    N = ctx.params().ring_degree
    chunks = -(-w.size // (N // 2))
    out = ctx._empty(chunks, 2, ctx.full, N)
    _check(lib().lcl_pack_and_encrypt(ctx.h, rng.h, w.ctypes.data, w.size, prescale,
                                      _ptr(pk.device()), _ptr(out)))
    return PackedWeights(out, int(w.size), prescale, ctx.scale())


def generate_keys(ctx: "CkksContext", rng: Sampler, steps):
    """generate_keys (ckks.cpp:225-261) on the device from the KGC's Sampler:
    (SecretKey, PublicKey, RelinKey, RotationKeySet) with host copies of the
    words (word-identical to the reference for the same Sampler state)."""
    import torch
    N = ctx.params().ring_degree
    full = ctx.full
    kw = (full, 2, full + 1, N)
    steps = list(steps)
    sk = ctx._empty(full + 1, N)
    pk = ctx._empty(2, full, N)
    rl = ctx._empty(*kw)
    rot = ctx._empty(max(1, len(steps)), *kw)
    arr = (C.c_size_t * max(1, len(steps)))(*steps)
    got = (C.c_size_t * max(1, len(steps)))()
    nk = C.c_size_t()
    _check(lib().lcl_generate_keys(ctx.h, rng.h, arr, len(steps), _ptr(sk), _ptr(pk), _ptr(rl),
                                   _ptr(rot), got, C.byref(nk)))
    torch.cuda.synchronize()
    rot_h = to_host(rot)
    keys = RotationKeySet({int(got[i]): rot_h[i] for i in range(nk.value)})
    return SecretKey(to_host(sk)), PublicKey(to_host(pk)), RelinKey(to_host(rl)), keys


def build_mask(ctx: "CkksContext", selected, n: int, pk: PublicKey, rng: Sampler):
    """aggregation.cpp:156-186 on the device -> (rank_rows, client selectors),
    each [n][2][full][N]."""
    N = ctx.params().ring_degree
    sel = (C.c_size_t * max(1, len(selected)))(*selected)
    rows = ctx._empty(n, 2, ctx.full, N)
    sels = ctx._empty(n, 2, ctx.full, N)
    _check(lib().lcl_build_mask(ctx.h, rng.h, n, sel, len(selected), _ptr(pk.device()),
                                _ptr(rows), _ptr(sels)))
    return rows, sels


class SecretKey:
    """SecretKey (ckks.hpp:57-60): the evaluation-domain rows of s over the
    full chain (+ special row); the KGC's key, used by decrypt_values."""

    def __init__(self, rows):
        self.rows = np.ascontiguousarray(rows, dtype=np.uint64)
        self._dev = {}

    def device_rows(self, count):
        if count not in self._dev:
            self._dev[count] = to_device(self.rows[:count])
        return self._dev[count]


class SelectionRule(Enum):
    krum = 0
    multi_krum = 1
    median = 2


@dataclass
class SelectionMask:
    """aggregation.hpp:77-82: client_selectors = [n][2][full][N]; rank_rows are
    never read by the server (aggregation.cpp:171-176 vs :211-217)."""
    n: int
    l: int
    client_selectors: object
    scale: float
    rank_rows: object = None


class DistanceMode(Enum):
    per_pair = 0
    row_sums = 1


class HoistMode(Enum):
    off = 0
    full = 1
    dynamic_lp = 2


@dataclass
class HoistPlan:
    k: int = 1
    t_hoist: float = 0.0
    t_decompose: float = 0.0
    m_cipher: float = 0.0
    m_budget: float = 0.0
    n: int = 1
    cost: float = 0.0


@dataclass
class DistanceOptions:
    lazy_relin: bool = True
    reduce_on_server: bool = True


@dataclass
class EncryptedDistanceMatrix:
    """distance.hpp:108-114. `batch` holds the entries as one device tensor in
    the order of `keys` ((i, j) i<j for per_pair, (i, i) for row_sums)."""
    mode: DistanceMode
    n: int
    reduced: bool
    value_scale: float
    batch: object
    keys: list
    scale: float

    @property
    def entries(self):
        return {k: Ciphertext(self.batch[p], self.scale) for p, k in enumerate(self.keys)}


# --------------------------------------------------------------- context
class CkksContext:
    """Server-side CkksContext: device basis, resident keys, evaluator."""

    def __init__(self, params: CkksParams | None = None, device: int = 0):
        params = params or CkksParams()
        params.validate()
        self._params = params
        L = lib()
        h = C.c_void_p()
        _check(L.lcl_context_create(params.ring_degree, params.depth,
                                    1 if params.security == SecurityLevel.bits128 else 0,
                                    device, C.byref(h)))
        self.h = h
        self.device = device
        full = C.c_size_t()
        buf = (C.c_uint64 * (params.depth + 2))()
        _check(L.lcl_context_primes(self.h, buf, C.byref(full)))
        self.full = full.value
        self.primes = [int(buf[i]) for i in range(self.full)]
        self.special = int(buf[self.full])
        self._relin_id = None
        self._rot_ids = {}

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().lcl_context_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # --- accessors (ckks.hpp:153-163)
    def params(self):
        return self._params

    def slot_count(self):
        return self._params.ring_degree // 2

    def top_level(self):
        return self._params.depth

    def scale(self):
        return self._params.scale()

    def counters(self):
        c = Counts()
        _check(lib().lcl_get_counts(self.h, C.byref(c)))
        return c.as_dict()

    def reset_counters(self):
        _check(lib().lcl_reset_counts(self.h))

    def launch_count(self):
        return int(lib().lcl_launch_count(self.h))

    def set_stream(self, stream):
        """Bind a torch.cuda.Stream (or raw handle) as the context's stream."""
        handle = getattr(stream, "cuda_stream", stream)
        _check(lib().lcl_set_stream(self.h, C.c_void_p(handle)))

    def synchronize(self):
        _check(lib().lcl_synchronize(self.h))

    # --- keys (resident in HBM; uploaded once per key object)
    def _key_words(self):
        return self.full * 2 * (self.full + 1) * self._params.ring_degree

    def use_relin_key(self, rk: RelinKey):
        if rk is None:
            raise KeyError("no relinearization key")
        # the uploaded object is held, so identity cannot be recycled by the GC
        if self._relin_id is not rk.key:
            k = np.ascontiguousarray(rk.key, dtype=np.uint64)
            _check(lib().lcl_upload_relin_key(self.h, k.ctypes.data, k.size))
            self._relin_id = rk.key

    def use_rotation_keys(self, keys: RotationKeySet, steps):
        slots = self.slot_count()
        for raw in steps:
            st = raw % slots
            if st == 0:
                continue
            if st not in keys.steps:
                raise KeyError("no rotation key for the requested step")
            if self._rot_ids.get(st) is not keys.steps[st]:
                k = np.ascontiguousarray(keys.steps[st], dtype=np.uint64)
                _check(lib().lcl_upload_rotation_key(self.h, st, k.ctypes.data, k.size))
                self._rot_ids[st] = keys.steps[st]

    # --- helpers
    def _empty(self, *shape):
        return _torch().empty(shape, dtype=_torch().int64, device=f"cuda:{self.device}")

    def ciphertext(self, words, scale):
        return Ciphertext(to_device(words, f"cuda:{self.device}"), scale)

    # --- evaluator (ckks.cpp:395-612)
    def _same(self, a, b):
        if a.level() != b.level():
            raise AlignmentError("operand levels diverge")
        ref = max(abs(a.scale), abs(b.scale))
        if abs(a.scale - b.scale) > 1e-9 * ref:
            raise AlignmentError("operand scales diverge")

    def hadd(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        self._same(a, b)
        out = self._empty(*a.data.shape)
        _check(lib().lcl_hadd(self.h, _ptr(a.data), _ptr(b.data), 1, a.level() + 1, _ptr(out)))
        return Ciphertext(out, a.scale)

    def hsub(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        self._same(a, b)
        out = self._empty(*a.data.shape)
        _check(lib().lcl_hsub(self.h, _ptr(a.data), _ptr(b.data), 1, a.level() + 1, _ptr(out)))
        return Ciphertext(out, a.scale)

    def decrypt_values(self, ct: Ciphertext, sk: "SecretKey"):
        """decrypt_values (ckks.cpp:390-393) on the device: float64 slots [N/2]."""
        return self.decrypt_values_batch(ct.data.reshape(1, *ct.data.shape), ct.scale, sk)[0]

    def decrypt_values_batch(self, cts, scale: float, sk: "SecretKey"):
        """KGC decode of a batch [B][2][m][N] at one scale -> float64 [B][N/2]
        (the distance matrix or the aggregate chunks in one call)."""
        import torch
        B, _, m, N = (int(x) for x in cts.shape)
        if m > sk.rows.shape[0]:
            raise KeyError("secret key narrower than the ciphertext")
        dsk = sk.device_rows(m)
        out = torch.empty((B, N // 2), dtype=torch.float64, device=dsk.device)
        _check(lib().lcl_decrypt_values(self.h, _ptr(cts.contiguous()), B, m, scale, _ptr(dsk),
                                        _ptr(out)))
        return out

    # ---- LCLT wire format (ckks.cpp:614-678)
    def blob_bytes(self, limbs=None) -> int:
        m = self.full if limbs is None else limbs
        return 13 + 16 * m * self._params.ring_degree

    def serialize_batch(self, cts, scale: float, stride=None):
        """CkksContext::serialize for a batch [B][2][m][N] -> uint8 [B][stride]."""
        B, _, m, N = (int(x) for x in cts.shape)
        stride = stride or self.blob_bytes(m)
        out = np.zeros((B, stride), np.uint8)
        _check(lib().lcl_serialize(self.h, _ptr(cts.contiguous()), B, m, scale,
                                   out.ctypes.data, stride))
        return out

    def serialize(self, ct: Ciphertext) -> bytes:
        return self.serialize_batch(ct.data.reshape(1, *ct.data.shape), ct.scale)[0].tobytes()

    def deserialize_batch(self, blobs, blob_bytes=None):
        """CkksContext::deserialize for blobs uint8 [B][stride] -> (device
        [B][2][m][N], scale); DataError exactly as the reference."""
        blobs = np.ascontiguousarray(blobs, dtype=np.uint8)
        B, stride = blobs.shape
        blob_bytes = stride if blob_bytes is None else blob_bytes
        m = int(blobs[0, 12]) if B and stride >= 13 else self.full
        m = max(1, min(m, self.full))
        out = self._empty(B, 2, m, self._params.ring_degree)
        sc = C.c_double()
        _check(lib().lcl_deserialize(self.h, blobs.ctypes.data, blob_bytes, stride, B, _ptr(out),
                                     C.byref(sc)))
        return out, sc.value

    def deserialize(self, data: bytes) -> Ciphertext:
        arr = np.frombuffer(bytes(data), np.uint8).reshape(1, -1)
        out, sc = self.deserialize_batch(arr)
        return Ciphertext(out[0], sc)

    def hmult_triple(self, a: Ciphertext, b: Ciphertext) -> TernaryCiphertext:
        """ckks.cpp:417-439 (Karatsuba; scale = product)."""
        if a.level() != b.level():
            raise AlignmentError("operands at different levels")
        m = a.level() + 1
        out = self._empty(3, m, self._params.ring_degree)
        _check(lib().lcl_hmult(self.h, _ptr(a.data.contiguous()), _ptr(b.data.contiguous()), 1, m,
                               _ptr(out)))
        return TernaryCiphertext(out, a.scale * b.scale)

    def hsquare(self, a: Ciphertext) -> TernaryCiphertext:
        """ckks.cpp:441-451 (scale = square)."""
        m = a.level() + 1
        out = self._empty(3, m, self._params.ring_degree)
        _check(lib().lcl_hsquare(self.h, _ptr(a.data.contiguous()), 1, m, _ptr(out)))
        return TernaryCiphertext(out, a.scale * a.scale)

    def relinearize(self, t: TernaryCiphertext, rk: RelinKey) -> Ciphertext:
        self.use_relin_key(rk)
        m = t.level() + 1
        out = self._empty(2, m, self._params.ring_degree)
        _check(lib().lcl_relinearize(self.h, _ptr(t.data.contiguous()), 1, m, _ptr(out)))
        return Ciphertext(out, t.scale)

    def rescale(self, ct: Ciphertext) -> Ciphertext:
        if ct.level() == 0:
            raise DepthExhaustedError("no prime left to rescale by")
        m = ct.level() + 1
        out = self._empty(2, m - 1, self._params.ring_degree)
        _check(lib().lcl_rescale(self.h, _ptr(ct.data.contiguous()), 1, m, _ptr(out)))
        return Ciphertext(out, ct.scale / float(self.primes[ct.level()]))

    def rotate(self, ct: Ciphertext, step: int, keys: RotationKeySet) -> Ciphertext:
        step %= self.slot_count()
        if step == 0:
            return ct
        self.use_rotation_keys(keys, [step])
        out = self._empty(*ct.data.shape)
        _check(lib().lcl_rotate(self.h, _ptr(ct.data.contiguous()), 1, ct.level() + 1, step,
                                _ptr(out)))
        return Ciphertext(out, ct.scale)

    def hoisted_rotations(self, ct: Ciphertext, steps, keys: RotationKeySet):
        self.use_rotation_keys(keys, steps)
        outs = self._empty(len(steps), *ct.data.shape)
        arr = (C.c_size_t * max(1, len(steps)))(*steps)
        _check(lib().lcl_hoisted_rotations(self.h, _ptr(ct.data.contiguous()), 1, ct.level() + 1,
                                           arr, len(steps), _ptr(outs)))
        return [Ciphertext(outs[i], ct.scale) for i in range(len(steps))]

    def mult_plain_const(self, ct: Ciphertext, value: float, pt_scale: float) -> Ciphertext:
        out = self._empty(*ct.data.shape)
        _check(lib().lcl_mult_plain_const(self.h, _ptr(ct.data.contiguous()), 1, ct.level() + 1,
                                          value, pt_scale, _ptr(out)))
        return Ciphertext(out, ct.scale * pt_scale)


# --------------------------------------------------------------- distance.hpp
def chunk_count_for(dimension: int, slot_count: int) -> int:
    if dimension == 0 or slot_count == 0:
        raise ShapeError("empty weight vector or slotless context")
    return (dimension + slot_count - 1) // slot_count


def distance_prescale(dimension: int, message_bound: float) -> float:
    if float(dimension) * message_bound > math.ldexp(1.0, 42):
        return 1.0 / math.sqrt(float(dimension))
    return 1.0


def _pow2(n):
    return n != 0 and (n & (n - 1)) == 0


def _require_width(n):
    if not _pow2(n):
        raise WidthError("reduction width must be a power of two")


def plan_unfold(t_hoist, t_decompose, m_cipher, m_budget, n) -> HoistPlan:
    """distance.cpp:144-179: exhaustive minimisation, ties to the smallest k."""
    if not (t_hoist > 0 and t_decompose > 0 and m_cipher > 0 and m_budget > 0):
        raise ParameterError("plan inputs must all be positive")
    _require_width(n)
    if m_cipher > m_budget:
        raise InfeasibleError("one ciphertext already exceeds the memory budget")
    levels = n.bit_length() - 1
    mem_cap = math.floor(m_budget / m_cipher)
    k_max = levels + 1
    if mem_cap < float(k_max):
        k_max = int(mem_cap)
    plan = HoistPlan(k=1, t_hoist=t_hoist, t_decompose=t_decompose, m_cipher=m_cipher,
                     m_budget=m_budget, n=n, cost=float(levels) * t_hoist)
    for k in range(2, k_max + 1):
        cost = float(levels - k + 1) * t_hoist + float(k - 1) * t_decompose
        if cost < plan.cost:
            plan.cost = cost
            plan.k = k
    return plan


@dataclass
class Calibration:
    """protocol.hpp:256-260 (the reference's field naming)."""
    t_hoist: float = 0.0      # seconds: decompose + first rotation (t1)
    t_decompose: float = 0.0  # seconds: one more hoisted rotation (t2 - t1)
    m_cipher: float = 0.0     # bytes per ciphertext


def calibrate(ctx: CkksContext, keys: RotationKeySet, ct: Ciphertext) -> Calibration:
    """calibrate (protocol.cpp:224-253) timed on the device: median of 11
    hoisted_rotations(ct, {1}) and ({1, 2}) calls (lcl_calibrate). `ct` is a
    fresh ciphertext (the reference encrypts 0.5 in every slot; every kernel
    is data-oblivious, so any fresh ciphertext times the same)."""
    if not (keys.has_step(1) and keys.has_step(2)):
        raise KeyError("calibration needs rotation keys for steps 1 and 2")
    ctx.use_rotation_keys(keys, [1, 2])
    th, td, mc = C.c_double(), C.c_double(), C.c_double()
    _check(lib().lcl_calibrate(ctx.h, _ptr(ct.data.contiguous()), ct.level() + 1, C.byref(th),
                               C.byref(td), C.byref(mc)))
    return Calibration(th.value, td.value, mc.value)


def fixed_plan(mode: HoistMode, n: int) -> HoistPlan:
    _require_width(n)
    levels = n.bit_length() - 1
    if mode == HoistMode.off:
        return HoistPlan(k=1, n=n)
    if mode == HoistMode.full:
        return HoistPlan(k=levels + 1, n=n)
    raise UsageError("dynamic plans come from plan_unfold with calibration")


def slot_reduce_steps(n: int, k: int):
    _require_width(n)
    if k == 0:
        raise ParameterError("unfold factor starts at 1")
    levels = n.bit_length() - 1
    unf = min(k - 1, levels)
    return list(range(1, 1 << unf)) + [1 << j for j in range(unf, levels)]


def slot_reduce(ctx: CkksContext, a: Ciphertext, plan: HoistPlan, keys: RotationKeySet):
    _require_width(plan.n)
    if plan.n > ctx.slot_count():
        raise WidthError("reduction width exceeds the slot count")
    if plan.k == 0:
        raise ParameterError("unfold factor starts at 1")
    if plan.n == 1:
        return a
    ctx.use_rotation_keys(keys, slot_reduce_steps(plan.n, plan.k))
    out = ctx._empty(*a.data.shape)
    _check(lib().lcl_slot_reduce(ctx.h, _ptr(a.data.contiguous()), 1, a.level() + 1, plan.n,
                                 plan.k, _ptr(out)))
    return Ciphertext(out, a.scale)


def _require_same_shape(a: PackedWeights, b: PackedWeights):
    if (a.dimension != b.dimension or a.chunk_count() != b.chunk_count()
            or a.prescale != b.prescale):
        raise ShapeError("packed weights disagree in length, chunking or prescale")


def encrypted_pairwise_distance(ctx, a: PackedWeights, b: PackedWeights, rk: RelinKey,
                                lazy=True) -> Ciphertext:
    _require_same_shape(a, b)
    ctx.use_relin_key(rk)
    m = ctx.full
    out = ctx._empty(2, m - 1, ctx.params().ring_degree)
    _check(lib().lcl_pairwise_distance(ctx.h, _ptr(a.chunks.contiguous()),
                                       _ptr(b.chunks.contiguous()), a.chunk_count(),
                                       1 if lazy else 0, _ptr(out)))
    return Ciphertext(out, (a.scale * a.scale) / float(ctx.primes[m - 1]))


def stack_clients(all_weights):
    """[n][C][2][full][N] device tensor for a list of PackedWeights (no copy
    when the chunks are consecutive views of one batch tensor)."""
    torch = _torch()
    base = all_weights[0].chunks
    try:
        parent = base._base
        # zero-copy only when the parent IS the [n][C][2][full][N] batch: a
        # view of a prefix slice (big[:, :C']) or of fewer limbs has the
        # same data pointers but strides clients by the parent's shape
        if (parent is not None and parent.dim() == 5 and parent.shape[0] == len(all_weights)
                and parent.is_contiguous() and parent.dtype == base.dtype
                and tuple(parent.shape[1:]) == tuple(base.shape)
                and all(w.chunks.data_ptr() == parent[i].data_ptr()
                        and tuple(w.chunks.shape) == tuple(base.shape)
                        for i, w in enumerate(all_weights))):
            return parent
    except AttributeError:
        pass
    return torch.stack([w.chunks for w in all_weights]).contiguous()


def build_distance_matrix(ctx: CkksContext, all_weights, rk: RelinKey, plan: HoistPlan,
                          mode: DistanceMode, keys: RotationKeySet,
                          options: DistanceOptions = DistanceOptions()):
    """distance.cpp:242-300 on the device."""
    n = len(all_weights)
    if n < 2:
        raise ShapeError("pairwise distances need at least two clients")
    for pw in all_weights:
        _require_same_shape(all_weights[0], pw)
    for pw in all_weights:
        ref = max(abs(pw.scale), abs(all_weights[0].scale))
        if abs(pw.scale - all_weights[0].scale) > 1e-9 * ref:
            raise AlignmentError("operand scales diverge")
    if options.reduce_on_server:
        needed = min(all_weights[0].dimension, ctx.slot_count())
        if plan.n < (1 << (needed - 1).bit_length()):
            raise WidthError("plan width misses populated slots")
    ctx.use_relin_key(rk)
    if options.reduce_on_server:
        _require_width(plan.n)
        if plan.n > ctx.slot_count():
            raise WidthError("reduction width exceeds the slot count")
        if plan.k == 0:
            raise ParameterError("unfold factor starts at 1")
        ctx.use_rotation_keys(keys, slot_reduce_steps(plan.n, plan.k) if plan.n > 1 else [])
    clients = stack_clients(all_weights)
    C_ = all_weights[0].chunk_count()
    m = ctx.full
    N = ctx.params().ring_degree
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    per_pair = mode == DistanceMode.per_pair
    out = ctx._empty(len(pairs) if per_pair else n, 2, m - 1, N)
    osc = C.c_double()
    _check(lib().lcl_build_distance_matrix(
        ctx.h, _ptr(clients), n, C_, all_weights[0].scale, plan.n, plan.k,
        0 if per_pair else 1, 1 if options.lazy_relin else 0,
        1 if options.reduce_on_server else 0, _ptr(out), C.byref(osc)))
    value_scale = all_weights[0].prescale * all_weights[0].prescale
    keys_ = pairs if per_pair else [(i, i) for i in range(n)]
    return EncryptedDistanceMatrix(mode, n, options.reduce_on_server, value_scale, out, keys_,
                                   osc.value)


@dataclass
class DistanceTable:
    """aggregation.hpp:30-35: the KGC's plaintext distance table."""
    n: int
    d: np.ndarray  # [n][n] float64


def table_from_matrix(ctx: CkksContext, m: "EncryptedDistanceMatrix", sk: "SecretKey"):
    """aggregation.cpp:242-258 on the device (decrypt_values of every entry)."""
    if m.mode != DistanceMode.per_pair:
        raise UsageError("pair entries required to rebuild the full table")
    count = int(m.batch.shape[2])
    out = np.zeros((m.n, m.n), np.float64)
    _check(lib().lcl_table_from_matrix(ctx.h, _ptr(m.batch.contiguous()), m.n, count, m.scale,
                                       1 if m.reduced else 0, m.value_scale,
                                       _ptr(sk.device_rows(count)), out.ctypes.data))
    return DistanceTable(m.n, out)


def totals_from_matrix(ctx: CkksContext, m: "EncryptedDistanceMatrix", sk: "SecretKey"):
    """aggregation.cpp:260-277: per-row totals from either matrix mode."""
    count = int(m.batch.shape[2])
    out = np.zeros(m.n, np.float64)
    _check(lib().lcl_totals_from_matrix(ctx.h, _ptr(m.batch.contiguous()), m.n,
                                        0 if m.mode == DistanceMode.per_pair else 1, count,
                                        m.scale, 1 if m.reduced else 0, m.value_scale,
                                        _ptr(sk.device_rows(count)), out.ctypes.data))
    return out


def masked_aggregate(ctx: CkksContext, weights, mask: SelectionMask, rule: SelectionRule,
                     rk: RelinKey) -> PackedWeights:
    """aggregation.cpp:188-229 on the device."""
    if len(weights) == 0:
        raise ShapeError("no client weights to aggregate")
    if len(weights) != mask.n or int(mask.client_selectors.shape[0]) != mask.n:
        raise ShapeError("mask rows do not match the client count")
    for pw in weights:
        if (pw.dimension != weights[0].dimension or pw.chunk_count() != weights[0].chunk_count()
                or pw.prescale != weights[0].prescale):
            raise ShapeError("client weights disagree in shape")
    ctx.use_relin_key(rk)
    average = rule == SelectionRule.multi_krum and mask.l > 1
    clients = stack_clients(weights)
    C_ = weights[0].chunk_count()
    m = ctx.full
    mo = m - 2 if average else m - 1
    out = ctx._empty(C_, 2, mo, ctx.params().ring_degree)
    osc = C.c_double()
    _check(lib().lcl_masked_aggregate(ctx.h, _ptr(clients), _ptr(mask.client_selectors.contiguous()),
                                      len(weights), C_, weights[0].scale, mask.scale, mask.l,
                                      1 if average else 0, _ptr(out), C.byref(osc)))
    return PackedWeights(out, weights[0].dimension, weights[0].prescale, osc.value)


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("builtins",)]
