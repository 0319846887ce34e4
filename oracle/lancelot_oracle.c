/*
 * lancelot_oracle.c — TEST INFRASTRUCTURE ONLY (see lancelot_oracle.h).
 *
 * Plain-C restatement of the reference algorithm for the server hot path.
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/core). Compiled with -ffp-contract=off so the only
 * floating-point code on the path (the canonical-embedding FFT inside encode)
 * reproduces the reference's non-FMA x86-64 Release build.
 */
#define _GNU_SOURCE
#include "lancelot_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

#define MAXP 48

/* ------------------------------------------------------------------ L0 */
/* Modulus: value < 2^62, ratio = floor((2^128-1)/q) (modmath.cpp:24-33). */
typedef struct {
  u64 v, rlo, rhi;
} mod_t;

static mod_t mod_make(u64 q) {
  mod_t m;
  u128 r = ~(u128)0 / q;
  m.v = q;
  m.rlo = (u64)r;
  m.rhi = (u64)(r >> 64);
  return m;
}

static inline u64 addm(u64 a, u64 b, const mod_t* m) {
  u64 s = a + b;
  return s >= m->v ? s - m->v : s;
}
static inline u64 subm(u64 a, u64 b, const mod_t* m) {
  return a >= b ? a - b : a + m->v - b;
}
static inline u64 negm(u64 a, const mod_t* m) { return a ? m->v - a : 0; }

/* barrett_reduce_128 (modmath.hpp:62-73): exact for every 128-bit input. */
static inline u64 red128(u128 x, const mod_t* m) {
  u64 x0 = (u64)x, x1 = (u64)(x >> 64);
  u128 c0 = (u128)x0 * m->rlo;
  u128 c1 = (u128)x0 * m->rhi + (u64)(c0 >> 64);
  u128 c2 = (u128)x1 * m->rlo + (u64)c1;
  u64 qh = x1 * m->rhi + (u64)(c1 >> 64) + (u64)(c2 >> 64);
  u64 r = x0 - qh * m->v;
  return r >= m->v ? r - m->v : r;
}
static inline u64 redm(u64 a, const mod_t* m) { return red128((u128)a, m); }
static inline u64 mulm(u64 a, u64 b, const mod_t* m) { return red128((u128)a * b, m); }
/* Shoup (modmath.hpp:84-95). */
static inline u64 shoup(u64 w, const mod_t* m) { return (u64)(((u128)w << 64) / m->v); }
static inline u64 mulsh(u64 a, u64 w, u64 ws, const mod_t* m) {
  u64 hi = (u64)(((u128)a * ws) >> 64);
  u64 r = a * w - hi * m->v;
  return r >= m->v ? r - m->v : r;
}

static u64 powm(u64 b, u64 e, const mod_t* m) {
  u64 r = 1;
  b = redm(b, m);
  while (e) {
    if (e & 1) r = mulm(r, b, m);
    b = mulm(b, b, m);
    e >>= 1;
  }
  return r;
}
static u64 invm(u64 a, const mod_t* m) { return powm(redm(a, m), m->v - 2, m); }

/* Deterministic Miller-Rabin with the first twelve primes (modmath.cpp:54-86). */
static int is_prime(u64 n) {
  static const u64 sp[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i) {
    if (n == sp[i]) return 1;
    if (n % sp[i] == 0) return 0;
  }
  u64 d = n - 1;
  int r = 0;
  while (!(d & 1)) {
    d >>= 1;
    ++r;
  }
  mod_t m = mod_make(n);
  for (int i = 0; i < 12; ++i) {
    u64 x = powm(sp[i], d, &m);
    if (x == 1 || x == n - 1) continue;
    int ok = 0;
    for (int t = 1; t < r; ++t) {
      x = mulm(x, x, &m);
      if (x == n - 1) {
        ok = 1;
        break;
      }
    }
    if (!ok) return 0;
  }
  return 1;
}

/* generate_ntt_primes (modmath.cpp:88-115): scan down from 2^bits - 2N + 1. */
static int gen_primes(int bits, size_t n, size_t count, const u64* avoid,
                      size_t navoid, u64* out) {
  u64 step = 2 * (u64)n, lo = (u64)1 << (bits - 1);
  u64 cand = ((u64)1 << bits) - step + 1;
  size_t got = 0;
  while (got < count && cand > lo) {
    int skip = !is_prime(cand);
    for (size_t i = 0; !skip && i < navoid; ++i) skip = avoid[i] == cand;
    for (size_t i = 0; !skip && i < got; ++i) skip = out[i] == cand;
    if (!skip) out[got++] = cand;
    cand -= step;
  }
  return got == count ? LO_OK : LO_PARAMETER_ERROR;
}

/* primitive_root_2n (modmath.cpp:117-132): smallest g >= 2 whose image has order 2n. */
static u64 root_2n(size_t n, const mod_t* q) {
  u64 quot = (q->v - 1) / (2 * (u64)n);
  for (u64 g = 2; g < q->v; ++g) {
    u64 r = powm(g, quot, q);
    if (powm(r, n, q) == q->v - 1) return r;
  }
  return 0;
}

static size_t brv(size_t x, int bits) {
  size_t r = 0;
  for (int i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1);
  return r;
}

/* ------------------------------------------------------------------ L1 */
typedef struct {
  u64 psi;
  u64 *rp, *rps, *irp, *irps;
  u64 ninv, ninvs;
} tables_t;

struct lo_ctx {
  size_t n;
  int logn;
  size_t full;         /* q primes */
  mod_t mod[MAXP + 1]; /* index full = special */
  tables_t tab[MAXP + 1];
  u64 inv[(MAXP + 1) * (MAXP + 1)]; /* inv[i*(full+1)+j] = p_i^-1 mod p_j */
  double scale;
  size_t hamming;
  int eta;
  double message_bound;
  int threads;
  lo_counts cnt;
  /* keys */
  u64* sk;           /* (full+1) rows eval */
  u64 *pk0, *pk1;    /* full rows eval */
  u64* relin;        /* switch key */
  size_t nrot;
  size_t rot_step[256];
  u64* rot_key[256];
  /* galois cache: perm per step */
  size_t ngal;
  size_t gal_step[256];
  uint32_t* gal_perm[256];
  pthread_mutex_t gal_mu;
};

static __thread int g_err = 0;
int lo_last_error(void) { return g_err; }

#define CNT(c, f, v) __atomic_fetch_add(&(c)->cnt.f, (v), __ATOMIC_RELAXED)

/* build_tables (rns.cpp:115-138). */
static void build_tables(lo_ctx* c, size_t i) {
  const mod_t* q = &c->mod[i];
  tables_t* t = &c->tab[i];
  size_t n = c->n;
  t->psi = root_2n(n, q);
  u64 psi_inv = invm(t->psi, q);
  t->rp = malloc(n * 8);
  t->rps = malloc(n * 8);
  t->irp = malloc(n * 8);
  t->irps = malloc(n * 8);
  u64 f = 1, g = 1;
  for (size_t k = 0; k < n; ++k) {
    size_t r = brv(k, c->logn);
    t->rp[r] = f;
    t->irp[r] = g;
    f = mulm(f, t->psi, q);
    g = mulm(g, psi_inv, q);
  }
  for (size_t k = 0; k < n; ++k) {
    t->rps[k] = shoup(t->rp[k], q);
    t->irps[k] = shoup(t->irp[k], q);
  }
  t->ninv = invm(n, q);
  t->ninvs = shoup(t->ninv, q);
}

/* forward_ntt_impl (rns.cpp:140-158): CT butterflies, psi^brv twiddles. */
static void ntt_fwd(const lo_ctx* c, u64* a, size_t pi) {
  const mod_t* q = &c->mod[pi];
  const tables_t* t = &c->tab[pi];
  size_t n = c->n, half = n;
  for (size_t m = 1; m < n; m <<= 1) {
    half >>= 1;
    for (size_t i = 0; i < m; ++i) {
      u64 w = t->rp[m + i], ws = t->rps[m + i];
      u64 *x = a + 2 * i * half, *y = x + half;
      for (size_t j = 0; j < half; ++j) {
        u64 u = x[j], v = mulsh(y[j], w, ws, q);
        x[j] = addm(u, v, q);
        y[j] = subm(u, v, q);
      }
    }
  }
}

/* inverse_ntt_impl (rns.cpp:160-181): GS butterflies then x N^-1. */
static void ntt_inv(const lo_ctx* c, u64* a, size_t pi) {
  const mod_t* q = &c->mod[pi];
  const tables_t* t = &c->tab[pi];
  size_t n = c->n, half = 1;
  for (size_t m = n >> 1; m >= 1; m >>= 1) {
    for (size_t i = 0; i < m; ++i) {
      u64 w = t->irp[m + i], ws = t->irps[m + i];
      u64 *x = a + 2 * i * half, *y = x + half;
      for (size_t j = 0; j < half; ++j) {
        u64 u = x[j], v = y[j];
        x[j] = addm(u, v, q);
        y[j] = mulsh(subm(u, v, q), w, ws, q);
      }
    }
    half <<= 1;
  }
  for (size_t j = 0; j < n; ++j) a[j] = mulsh(a[j], t->ninv, t->ninvs, q);
}

/* Row r of a poly with `count` q rows (+special last) -> basis index. */
static inline size_t row_pi(const lo_ctx* c, size_t count, size_t r) {
  return r < count ? r : c->full;
}

static void poly_ntt_fwd(const lo_ctx* c, u64* p, size_t count, int sp) {
  for (size_t r = 0; r < count + (size_t)sp; ++r) ntt_fwd(c, p + r * c->n, row_pi(c, count, r));
}
static void poly_ntt_inv(const lo_ctx* c, u64* p, size_t count, int sp) {
  for (size_t r = 0; r < count + (size_t)sp; ++r) ntt_inv(c, p + r * c->n, row_pi(c, count, r));
}

/* PolyRns elementwise ops (rns.cpp:224-280); rows = count (+special). */
static void poly_add(const lo_ctx* c, u64* a, const u64* b, size_t count, int sp) {
  for (size_t r = 0; r < count + (size_t)sp; ++r) {
    const mod_t* q = &c->mod[row_pi(c, count, r)];
    for (size_t j = 0; j < c->n; ++j) a[r * c->n + j] = addm(a[r * c->n + j], b[r * c->n + j], q);
  }
}
static void poly_sub(const lo_ctx* c, u64* a, const u64* b, size_t count, int sp) {
  for (size_t r = 0; r < count + (size_t)sp; ++r) {
    const mod_t* q = &c->mod[row_pi(c, count, r)];
    for (size_t j = 0; j < c->n; ++j) a[r * c->n + j] = subm(a[r * c->n + j], b[r * c->n + j], q);
  }
}
static void poly_neg(const lo_ctx* c, u64* a, size_t count, int sp) {
  for (size_t r = 0; r < count + (size_t)sp; ++r) {
    const mod_t* q = &c->mod[row_pi(c, count, r)];
    for (size_t j = 0; j < c->n; ++j) a[r * c->n + j] = negm(a[r * c->n + j], q);
  }
}
static void poly_mul(const lo_ctx* c, u64* a, const u64* b, size_t count, int sp) {
  for (size_t r = 0; r < count + (size_t)sp; ++r) {
    const mod_t* q = &c->mod[row_pi(c, count, r)];
    for (size_t j = 0; j < c->n; ++j) a[r * c->n + j] = mulm(a[r * c->n + j], b[r * c->n + j], q);
  }
}

/* divide_and_round_by_last (rns.cpp:463-506). x has `count` q rows and
 * optionally the special row; eval domain. out gets the remaining rows. */
static void divide_round_last(const lo_ctx* c, const u64* x, size_t count, int sp, u64* out) {
  size_t n = c->n;
  size_t out_count = sp ? count : count - 1;
  size_t div_pi = sp ? c->full : out_count;
  const mod_t* p = &c->mod[div_pi];
  u64* last = malloc(n * 8);
  u64* lift = malloc(n * 8);
  memcpy(last, x + (count + (size_t)sp - 1) * n, n * 8);
  ntt_inv(c, last, div_pi);
  u64 half = p->v >> 1;
  for (size_t i = 0; i < out_count; ++i) {
    const mod_t* q = &c->mod[i];
    u64 pq = redm(p->v, q);
    for (size_t j = 0; j < n; ++j) {
      u64 r = redm(last[j], q);
      if (last[j] > half) r = subm(r, pq, q);
      lift[j] = r;
    }
    ntt_fwd(c, lift, i);
    u64 pinv = c->inv[div_pi * (c->full + 1) + i];
    u64 pinvs = shoup(pinv, q);
    for (size_t j = 0; j < n; ++j)
      out[i * n + j] = mulsh(subm(x[i * n + j], lift[j], q), pinv, pinvs, q);
  }
  free(last);
  free(lift);
}

/* galois_elt_for_rotation / make_galois_tables (rns.cpp:508-532). */
uint64_t lo_galois_elt(size_t degree, size_t step) {
  u64 m = 2 * (u64)degree, e = 1;
  for (size_t i = 0; i < step % (degree / 2); ++i) e = (e * 5) % m;
  return e;
}

static void make_perm(const lo_ctx* c, u64 elt, uint32_t* perm) {
  size_t n = c->n;
  for (size_t i = 0; i < n; ++i) {
    u64 e = 2 * (u64)brv(i, c->logn) + 1;
    u64 t = (e * elt) % (2 * (u64)n);
    perm[i] = (uint32_t)brv((size_t)((t - 1) / 2), c->logn);
  }
}

static const uint32_t* gal(lo_ctx* c, size_t step) {
  pthread_mutex_lock(&c->gal_mu);
  for (size_t i = 0; i < c->ngal; ++i)
    if (c->gal_step[i] == step) {
      pthread_mutex_unlock(&c->gal_mu);
      return c->gal_perm[i];
    }
  uint32_t* p = malloc(c->n * 4);
  make_perm(c, lo_galois_elt(c->n, step), p);
  c->gal_step[c->ngal] = step;
  c->gal_perm[c->ngal++] = p;
  pthread_mutex_unlock(&c->gal_mu);
  return p;
}

void lo_galois_perm(const lo_ctx* c, size_t step, uint32_t* perm) {
  make_perm(c, lo_galois_elt(c->n, step), perm);
}

/* apply_galois (rns.cpp:534-547): o[j] = in[perm[j]] per row. */
static void apply_perm(const lo_ctx* c, const u64* in, size_t rows, const uint32_t* perm, u64* out) {
  for (size_t r = 0; r < rows; ++r)
    for (size_t j = 0; j < c->n; ++j) out[r * c->n + j] = in[r * c->n + perm[j]];
}

/* ------------------------------------------------------------ sampling */
/* std::mt19937_64 (the engine behind Sampler, sampling.hpp:34-65). */
typedef struct {
  u64 mt[312];
  int idx;
} mt64;

static void mt_seed(mt64* s, u64 seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (u64)i;
  s->idx = 312;
}

static u64 mt_next(mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      u64 y = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      u64 v = s->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = v;
    }
    s->idx = 0;
  }
  u64 x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* derive_seed: splitmix64 finalizer (sampling.cpp:25-31). */
uint64_t lo_derive_seed(uint64_t root, uint64_t tag) {
  u64 z = root + 0x9e3779b97f4a7c15ULL * (tag + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* Sampler::uniform_below (sampling.cpp:33-40): rejection, then modulo. */
static u64 below(mt64* s, u64 bound) {
  if ((bound & (bound - 1)) == 0) return mt_next(s) & (bound - 1);
  u64 lim = ~(u64)0 - (~(u64)0 % bound) - 1;
  u64 x = mt_next(s);
  while (x > lim) x = mt_next(s);
  return x % bound;
}
static double ureal(mt64* s) { return (double)(mt_next(s) >> 11) * 0x1.0p-53; }

/* uniform_poly (sampling.cpp:51-59). */
static void s_uniform(const lo_ctx* c, mt64* s, u64* p, size_t count, int sp) {
  for (size_t r = 0; r < count + (size_t)sp; ++r) {
    u64 q = c->mod[row_pi(c, count, r)].v;
    for (size_t j = 0; j < c->n; ++j) p[r * c->n + j] = below(s, q);
  }
}
/* set_coeff (sampling.cpp:61-67). */
static void s_set(const lo_ctx* c, u64* p, size_t count, int sp, size_t j, long v) {
  for (size_t r = 0; r < count + (size_t)sp; ++r) {
    u64 q = c->mod[row_pi(c, count, r)].v;
    p[r * c->n + j] = v >= 0 ? (u64)v : q - (u64)(-v);
  }
}
/* sparse_ternary_poly (sampling.cpp:79-97) / ternary_poly (:69-77). */
static void s_secret(const lo_ctx* c, mt64* s, u64* p, size_t count, int sp) {
  size_t n = c->n;
  if (c->hamming == 0) {
    for (size_t j = 0; j < n; ++j) s_set(c, p, count, sp, j, (long)below(s, 3) - 1);
    return;
  }
  memset(p, 0, (count + (size_t)sp) * n * 8);
  size_t* idx = malloc(n * sizeof(size_t));
  for (size_t i = 0; i < n; ++i) idx[i] = i;
  for (size_t i = 0; i < c->hamming; ++i) {
    size_t k = i + (size_t)below(s, n - i);
    size_t t = idx[i];
    idx[i] = idx[k];
    idx[k] = t;
    long sign = below(s, 2) == 0 ? 1 : -1;
    s_set(c, p, count, sp, idx[i], sign);
  }
  free(idx);
}
/* cbd_poly (sampling.cpp:99-112). */
static void s_cbd(const lo_ctx* c, mt64* s, u64* p, size_t count, int sp) {
  int eta = c->eta;
  u64 mask = eta == 32 ? (~(u64)0 >> 32) : (((u64)1 << eta) - 1);
  for (size_t j = 0; j < c->n; ++j) {
    u64 b = mt_next(s);
    int x = __builtin_popcountll(b & mask), y = __builtin_popcountll((b >> eta) & mask);
    s_set(c, p, count, sp, j, (long)(x - y));
  }
}

/* ------------------------------------------------------------ context */
/* CkksContext(params) -> make_basis (ckks.cpp:77-93) -> RnsBasis (rns.cpp:61-113).
 * CkksParams defaults (ckks.hpp:39-55): scale 2^40, q0 44 bits, P 54 bits,
 * hamming weight 64, eta 21, message bound 2^20. */
lo_ctx* lo_ctx_new(size_t degree, int depth, int secure, int threads) {
  g_err = LO_OK;
  if (degree < 8 || (degree & (degree - 1)) || depth < 0 || depth + 1 > MAXP) {
    g_err = LO_PARAMETER_ERROR;
    return NULL;
  }
  lo_ctx* c = calloc(1, sizeof(lo_ctx));
  c->n = degree;
  c->logn = __builtin_ctzll(degree);
  c->full = (size_t)depth + 1;
  c->scale = ldexp(1.0, 40);
  c->hamming = 64;
  c->eta = 21;
  c->message_bound = (double)(1 << 20);
  c->threads = threads < 1 ? 1 : threads;
  pthread_mutex_init(&c->gal_mu, NULL);
  u64 chain[MAXP + 1] = {0}, avoid[MAXP + 1] = {0};
  size_t na = 0;
  if (gen_primes(44, degree, 1, avoid, 0, chain) != LO_OK) goto fail;
  avoid[na++] = chain[0];
  if (depth > 0) {
    if (gen_primes(40, degree, (size_t)depth, avoid, na, chain + 1) != LO_OK) goto fail;
    for (int i = 0; i < depth; ++i) avoid[na++] = chain[1 + i];
  }
  u64 sp;
  if (gen_primes(54, degree, 1, avoid, na, &sp) != LO_OK) goto fail;
  double total = 0;
  for (size_t i = 0; i < c->full; ++i) {
    c->mod[i] = mod_make(chain[i]);
    total += log2((double)chain[i]);
  }
  c->mod[c->full] = mod_make(sp);
  total += log2((double)sp);
  if (secure) {
    /* security_budget_bits128 (rns.cpp:35-57). */
    double budget;
    switch (degree) {
      case 1024: budget = 27; break;
      case 2048: budget = 54; break;
      case 4096: budget = 109; break;
      case 8192: budget = 218; break;
      case 16384: budget = 438; break;
      case 32768: budget = 881; break;
      case 65536: budget = 1770; break;
      case 131072: budget = 3540; break;
      default: goto fail;
    }
    if (total > budget) goto fail;
  }
  for (size_t i = 0; i <= c->full; ++i) build_tables(c, i);
  size_t k = c->full + 1;
  for (size_t i = 0; i < k; ++i)
    for (size_t j = 0; j < k; ++j)
      c->inv[i * k + j] = i == j ? 0 : invm(c->mod[i].v, &c->mod[j]);
  return c;
fail:
  g_err = LO_PARAMETER_ERROR;
  free(c);
  return NULL;
}

void lo_ctx_free(lo_ctx* c) {
  if (!c) return;
  for (size_t i = 0; i <= c->full; ++i) {
    free(c->tab[i].rp);
    free(c->tab[i].rps);
    free(c->tab[i].irp);
    free(c->tab[i].irps);
  }
  free(c->sk);
  free(c->pk0);
  free(c->pk1);
  free(c->relin);
  for (size_t i = 0; i < c->nrot; ++i) free(c->rot_key[i]);
  for (size_t i = 0; i < c->ngal; ++i) free(c->gal_perm[i]);
  free(c);
}

size_t lo_degree(const lo_ctx* c) { return c->n; }
size_t lo_prime_count(const lo_ctx* c) { return c->full; }
uint64_t lo_prime(const lo_ctx* c, size_t i) { return c->mod[i].v; }
uint64_t lo_psi(const lo_ctx* c, size_t i) { return c->tab[i].psi; }
double lo_scale(const lo_ctx* c) { return c->scale; }
lo_counts lo_get_counts(const lo_ctx* c) { return c->cnt; }
void lo_reset_counts(lo_ctx* c) { memset(&c->cnt, 0, sizeof c->cnt); }
void lo_ntt_forward(const lo_ctx* c, uint64_t* row, size_t i) { ntt_fwd(c, row, i); }
void lo_ntt_inverse(const lo_ctx* c, uint64_t* row, size_t i) { ntt_inv(c, row, i); }
void lo_ntt_tables(const lo_ctx* c, size_t i, uint64_t* root, uint64_t* root_shoup,
                   uint64_t* iroot, uint64_t* iroot_shoup, uint64_t* n_inv2) {
  const tables_t* t = &c->tab[i];
  memcpy(root, t->rp, c->n * 8);
  memcpy(root_shoup, t->rps, c->n * 8);
  memcpy(iroot, t->irp, c->n * 8);
  memcpy(iroot_shoup, t->irps, c->n * 8);
  n_inv2[0] = t->ninv;
  n_inv2[1] = t->ninvs;
}

/* ------------------------------------------------------------ keys */
size_t lo_key_words(const lo_ctx* c) { return c->full * 2 * (c->full + 1) * c->n; }
const uint64_t* lo_relin_key(const lo_ctx* c) { return c->relin; }
const uint64_t* lo_secret_key(const lo_ctx* c) { return c->sk; }
/* PublicKey (p0, p1), full rows each, evaluation domain (ckks.cpp:208-219) */
const uint64_t* lo_public_key_p0(const lo_ctx* c) { return c->pk0; }
const uint64_t* lo_public_key_p1(const lo_ctx* c) { return c->pk1; }
const uint64_t* lo_rotation_key(const lo_ctx* c, size_t step) {
  for (size_t i = 0; i < c->nrot; ++i)
    if (c->rot_step[i] == step) return c->rot_key[i];
  return NULL;
}

/* make_switch_key (ckks.cpp:196-226). */
static u64* make_switch_key(lo_ctx* c, mt64* s, const u64* target) {
  size_t n = c->n, full = c->full, rows = full + 1, pw = rows * n;
  u64* key = malloc(lo_key_words(c) * 8);
  u64* e = malloc(pw * 8);
  for (size_t j = 0; j < full; ++j) {
    u64* k0 = key + (2 * j) * pw;
    u64* a = key + (2 * j + 1) * pw;
    s_uniform(c, s, a, full, 1);
    s_cbd(c, s, e, full, 1);
    poly_ntt_fwd(c, e, full, 1);
    memcpy(k0, a, pw * 8);
    poly_mul(c, k0, c->sk, full, 1);
    poly_neg(c, k0, full, 1);
    poly_add(c, k0, e, full, 1);
    const mod_t* qj = &c->mod[j];
    u64 th = redm(c->mod[full].v, qj), ths = shoup(th, qj);
    for (size_t i = 0; i < n; ++i)
      k0[j * n + i] = addm(k0[j * n + i], mulsh(target[j * n + i], th, ths, qj), qj);
  }
  free(e);
  return key;
}

/* generate_keys (ckks.cpp:228-261). */
int lo_keygen(lo_ctx* c, uint64_t seed, const size_t* steps, size_t nsteps) {
  size_t n = c->n, full = c->full, pw = (full + 1) * n;
  mt64 s;
  mt_seed(&s, lo_derive_seed(seed, 5));
  c->sk = malloc(pw * 8);
  s_secret(c, &s, c->sk, full, 1);
  poly_ntt_fwd(c, c->sk, full, 1);
  c->pk1 = malloc(full * n * 8);
  c->pk0 = malloc(full * n * 8);
  u64* e = malloc(full * n * 8);
  s_uniform(c, &s, c->pk1, full, 0);
  s_cbd(c, &s, e, full, 0);
  poly_ntt_fwd(c, e, full, 0);
  memcpy(c->pk0, c->pk1, full * n * 8);
  poly_mul(c, c->pk0, c->sk, full, 0);
  poly_neg(c, c->pk0, full, 0);
  poly_add(c, c->pk0, e, full, 0);
  free(e);
  u64* s2 = malloc(pw * 8);
  memcpy(s2, c->sk, pw * 8);
  poly_mul(c, s2, c->sk, full, 1);
  c->relin = make_switch_key(c, &s, s2);
  size_t slots = n / 2;
  for (size_t i = 0; i < nsteps; ++i) {
    size_t st = steps[i] % slots;
    if (st == 0 || lo_rotation_key(c, st)) continue;
    apply_perm(c, c->sk, full + 1, gal(c, st), s2);
    c->rot_step[c->nrot] = st;
    c->rot_key[c->nrot++] = make_switch_key(c, &s, s2);
  }
  free(s2);
  return LO_OK;
}

/* ------------------------------------------------------------ encoding */
typedef struct {
  double re, im;
} cpx;

/* Canonical embedding (encoding.cpp:37-134). Complex products are spelled out
 * as (ac - bd, ad + bc), the expansion GCC uses for finite operands. */
static void emb_fft(const lo_ctx* c, cpx* a, int inverse) {
  size_t h = c->n / 2;
  int logh = c->logn - 1;
  for (size_t i = 0; i < h; ++i) {
    size_t r = brv(i, logh);
    if (i < r) {
      cpx t = a[i];
      a[i] = a[r];
      a[r] = t;
    }
  }
  for (size_t len = 2; len <= h; len <<= 1) {
    size_t stride = h / len;
    for (size_t st = 0; st < h; st += len) {
      for (size_t k = 0; k < len / 2; ++k) {
        double ang = 2.0 * M_PI * (double)(k * stride) / (double)h;
        cpx w = {cos(ang), sin(ang)};
        if (inverse) w.im = -w.im;
        cpx u = a[st + k], x = a[st + k + len / 2];
        cpx v = {x.re * w.re - x.im * w.im, x.re * w.im + x.im * w.re};
        a[st + k].re = u.re + v.re;
        a[st + k].im = u.im + v.im;
        a[st + k + len / 2].re = u.re - v.re;
        a[st + k + len / 2].im = u.im - v.im;
      }
    }
  }
  if (inverse) {
    double s = 1.0 / (double)h;
    for (size_t i = 0; i < h; ++i) {
      a[i].re *= s;
      a[i].im *= s;
    }
  }
}

static size_t slot_bucket(const lo_ctx* c, size_t j) {
  u64 g = 1, two_n = 2 * (u64)c->n;
  for (size_t t = 0; t < j; ++t) g = (g * 5) % two_n;
  return (size_t)((g - 1) / 4);
}

/* CkksContext::encode (ckks.cpp:263-307) -> eval-domain rows [level+1][N]. */
int lo_encode(lo_ctx* c, const double* values, size_t nv, double scale, int level, uint64_t* out) {
  size_t n = c->n, h = n / 2;
  if (level < 0 || (size_t)level >= c->full) return LO_PARAMETER_ERROR;
  if (!(scale > 0.0) || !isfinite(scale)) return LO_PARAMETER_ERROR;
  if (nv > h) return LO_CAPACITY_ERROR;
  for (size_t i = 0; i < nv; ++i)
    if (!isfinite(values[i]) || fabs(values[i]) > c->message_bound) return LO_CAPACITY_ERROR;
  cpx* b = calloc(h, sizeof(cpx));
  u64 g = 1, two_n = 2 * (u64)n;
  for (size_t j = 0; j < nv; ++j) {
    b[(g - 1) / 4].re = values[j];
    g = (g * 5) % two_n;
  }
  emb_fft(c, b, 1);
  long long* rounded = malloc(n * sizeof(long long));
  for (size_t i = 0; i < h; ++i) {
    double ang = M_PI * (double)i / (double)n;
    double tr = cos(ang), ti = sin(ang);
    /* buckets[i] * conj(twist[i]) */
    double re = b[i].re * tr - b[i].im * (-ti);
    double im = b[i].re * (-ti) + b[i].im * tr;
    double xs[2] = {re * scale, im * scale};
    for (int t = 0; t < 2; ++t) {
      if (fabs(xs[t]) >= 4.6e18) {
        free(b);
        free(rounded);
        return LO_CAPACITY_ERROR;
      }
      rounded[i + (size_t)t * h] = llround(xs[t]);
    }
  }
  for (size_t r = 0; r <= (size_t)level; ++r) {
    const mod_t* q = &c->mod[r];
    for (size_t i = 0; i < n; ++i) {
      long long v = rounded[i];
      u64 mag = (u64)(v < 0 ? -v : v);
      u64 m = redm(mag, q);
      out[r * n + i] = v < 0 ? (m == 0 ? 0 : q->v - m) : m;
    }
  }
  poly_ntt_fwd(c, out, (size_t)level + 1, 0);
  free(b);
  free(rounded);
  return LO_OK;
}

/* encrypt (ckks.cpp:350-379) at the top level; ct = [2][full][N]. */
static void encrypt_top(lo_ctx* c, mt64* s, const u64* m, u64* ct) {
  size_t n = c->n, cnt = c->full, pw = cnt * n;
  u64* r = malloc(pw * 8);
  u64* e = malloc(pw * 8);
  s_secret(c, s, r, cnt, 0);
  poly_ntt_fwd(c, r, cnt, 0);
  u64* c0 = ct;
  u64* c1 = ct + pw;
  memcpy(c0, c->pk0, pw * 8);
  poly_mul(c, c0, r, cnt, 0);
  s_cbd(c, s, e, cnt, 0);
  poly_ntt_fwd(c, e, cnt, 0);
  poly_add(c, c0, e, cnt, 0);
  poly_add(c, c0, m, cnt, 0);
  memcpy(c1, c->pk1, pw * 8);
  poly_mul(c, c1, r, cnt, 0);
  s_cbd(c, s, e, cnt, 0);
  poly_ntt_fwd(c, e, cnt, 0);
  poly_add(c, c1, e, cnt, 0);
  CNT(c, encryptions, 1);
  free(r);
  free(e);
}

size_t lo_chunk_count(const lo_ctx* c, size_t dim) { return (dim + c->n / 2 - 1) / (c->n / 2); }

/* pack_and_encrypt (distance.cpp:64-91) driven as measure_distance_phase does. */
int lo_make_clients(lo_ctx* c, uint64_t seed, size_t clients, size_t dim, double prescale,
                    uint64_t* out) {
  size_t n = c->n, slots = n / 2, C = lo_chunk_count(c, dim);
  size_t ctw = 2 * c->full * n;
  mt64 s;
  mt_seed(&s, lo_derive_seed(seed, 0xAB1A7EULL));
  double* w = malloc(dim * sizeof(double));
  u64* m = malloc(c->full * n * 8);
  for (size_t i = 0; i < clients; ++i) {
    for (size_t t = 0; t < dim; ++t) w[t] = ureal(&s) - 0.5;
    for (size_t ch = 0; ch < C; ++ch) {
      size_t lo = ch * slots, hi = lo + slots < dim ? lo + slots : dim;
      double* buf = malloc((hi - lo) * sizeof(double));
      for (size_t t = lo; t < hi; ++t) buf[t - lo] = w[t] * prescale;
      int rc = lo_encode(c, buf, hi - lo, c->scale, (int)c->full - 1, m);
      free(buf);
      if (rc) {
        free(w);
        free(m);
        return rc;
      }
      encrypt_top(c, &s, m, out + (i * C + ch) * ctw);
    }
  }
  free(w);
  free(m);
  return LO_OK;
}

/* build_mask (aggregation.cpp:156-186): n rank rows (consumed from the stream,
 * not returned: the server never reads them), then n client selectors. */
int lo_build_mask(lo_ctx* c, uint64_t seed, const size_t* selected, size_t nsel, size_t n,
                  uint64_t* selectors) {
  size_t N = c->n, slots = N / 2, ctw = 2 * c->full * N;
  if (n > slots) return LO_CAPACITY_ERROR;
  for (size_t i = 0; i < nsel; ++i)
    if (selected[i] >= n) return LO_SHAPE_ERROR;
  mt64 s;
  mt_seed(&s, lo_derive_seed(seed, 0x3000000000000000ULL));
  double* v = malloc((n > slots ? n : slots) * sizeof(double));
  u64* m = malloc(c->full * N * 8);
  u64* scratch = malloc(ctw * 8);
  for (size_t r = 0; r < n; ++r) {
    for (size_t i = 0; i < n; ++i) v[i] = 0.0;
    if (r < nsel) v[selected[r]] = 1.0;
    lo_encode(c, v, n, c->scale, (int)c->full - 1, m);
    encrypt_top(c, &s, m, scratch);
  }
  for (size_t i = 0; i < n; ++i) {
    int chosen = 0;
    for (size_t t = 0; t < nsel; ++t) chosen |= selected[t] == i;
    for (size_t t = 0; t < slots; ++t) v[t] = chosen ? 1.0 : 0.0;
    lo_encode(c, v, slots, c->scale, (int)c->full - 1, m);
    encrypt_top(c, &s, m, selectors + i * ctw);
  }
  free(v);
  free(m);
  free(scratch);
  return LO_OK;
}

/* ------------------------------------------------------------ evaluator */
int lo_hsub(lo_ctx* c, size_t count, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  size_t pw = count * c->n;
  if (out != a) memcpy(out, a, 2 * pw * 8);
  poly_sub(c, out, b, count, 0);
  poly_sub(c, out + pw, b + pw, count, 0);
  CNT(c, additions, 1);
  return LO_OK;
}
int lo_hadd(lo_ctx* c, size_t count, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  size_t pw = count * c->n;
  if (out != a) memcpy(out, a, 2 * pw * 8);
  poly_add(c, out, b, count, 0);
  poly_add(c, out + pw, b + pw, count, 0);
  CNT(c, additions, 1);
  return LO_OK;
}
/* hsquare (ckks.cpp:441-451): d0 = c0^2, d2 = c1^2, d1 = 2 c0 c1. */
int lo_hsquare(lo_ctx* c, size_t count, const uint64_t* a, uint64_t* t) {
  size_t pw = count * c->n;
  memcpy(t, a, pw * 8);
  poly_mul(c, t, a, count, 0);
  memcpy(t + 2 * pw, a + pw, pw * 8);
  poly_mul(c, t + 2 * pw, a + pw, count, 0);
  memcpy(t + pw, a, pw * 8);
  poly_mul(c, t + pw, a + pw, count, 0);
  poly_add(c, t + pw, t + pw, count, 0);
  CNT(c, multiplications, 1);
  return LO_OK;
}
/* hmult_triple, Karatsuba form (ckks.cpp:417-439). */
int lo_hmult_triple(lo_ctx* c, size_t count, const uint64_t* a, const uint64_t* b, uint64_t* t) {
  size_t pw = count * c->n;
  u64* sb = malloc(pw * 8);
  memcpy(t, a, pw * 8);
  poly_mul(c, t, b, count, 0);
  memcpy(t + 2 * pw, a + pw, pw * 8);
  poly_mul(c, t + 2 * pw, b + pw, count, 0);
  memcpy(t + pw, a, pw * 8);
  poly_add(c, t + pw, a + pw, count, 0);
  memcpy(sb, b, pw * 8);
  poly_add(c, sb, b + pw, count, 0);
  poly_mul(c, t + pw, sb, count, 0);
  poly_sub(c, t + pw, t, count, 0);
  poly_sub(c, t + pw, t + 2 * pw, count, 0);
  free(sb);
  CNT(c, multiplications, 1);
  return LO_OK;
}
int lo_lazy_accumulate(lo_ctx* c, size_t count, uint64_t* acc, const uint64_t* t) {
  size_t pw = count * c->n;
  for (int i = 0; i < 3; ++i) poly_add(c, acc + i * pw, t + i * pw, count, 0);
  CNT(c, additions, 1);
  return LO_OK;
}

/* decompose_for_keyswitch (ckks.cpp:464-481) with the single-prime mod_up
 * branch (rns.cpp:367-383). digits = [count][count+1][N], eval domain. */
static u64* decompose(lo_ctx* c, const u64* d, size_t count) {
  size_t n = c->n, dw = (count + 1) * n;
  u64* coef = malloc(count * n * 8);
  memcpy(coef, d, count * n * 8);
  poly_ntt_inv(c, coef, count, 0);
  u64* dig = malloc(count * dw * 8);
  for (size_t j = 0; j < count; ++j) {
    const mod_t* src = &c->mod[j];
    u64 half = src->v >> 1;
    const u64* v = coef + j * n;
    for (size_t t = 0; t <= count; ++t) {
      const mod_t* dst = &c->mod[row_pi(c, count, t)];
      u64 sd = redm(src->v, dst);
      u64* o = dig + j * dw + t * n;
      for (size_t i = 0; i < n; ++i) {
        u64 r = redm(v[i], dst);
        if (v[i] > half) r = subm(r, sd, dst);
        o[i] = r;
      }
    }
    poly_ntt_fwd(c, dig + j * dw, count, 1);
  }
  free(coef);
  CNT(c, mod_ups, 1);
  return dig;
}

/* inner_product_moddown (ckks.cpp:483-520): out = (b, a), each [count][N]. */
static void ip_moddown(lo_ctx* c, const u64* dig, size_t count, const u64* key,
                       const uint32_t* perm, u64* b, u64* a) {
  size_t n = c->n, rows = count + 1, dw = rows * n, kpw = (c->full + 1) * n;
  u64* acc0 = calloc(dw, 8);
  u64* acc1 = calloc(dw, 8);
  u64* pd = perm ? malloc(dw * 8) : NULL;
  for (size_t j = 0; j < count; ++j) {
    const u64* dj = dig + j * dw;
    if (perm) {
      apply_perm(c, dj, rows, perm, pd);
      dj = pd;
    }
    const u64* k0 = key + (2 * j) * kpw;
    const u64* k1 = key + (2 * j + 1) * kpw;
    for (size_t r = 0; r < rows; ++r) {
      size_t kr = r == count ? c->full : r;
      const mod_t* q = &c->mod[row_pi(c, count, r)];
      for (size_t i = 0; i < n; ++i) {
        acc0[r * n + i] = addm(acc0[r * n + i], mulm(dj[r * n + i], k0[kr * n + i], q), q);
        acc1[r * n + i] = addm(acc1[r * n + i], mulm(dj[r * n + i], k1[kr * n + i], q), q);
      }
    }
  }
  divide_round_last(c, acc0, count, 1, b);
  divide_round_last(c, acc1, count, 1, a);
  free(acc0);
  free(acc1);
  free(pd);
}

/* relinearize (ckks.cpp:522-534). */
int lo_relinearize(lo_ctx* c, size_t count, const uint64_t* t, uint64_t* out) {
  if (!c->relin) return LO_KEY_ERROR;
  size_t pw = count * c->n;
  u64* dig = decompose(c, t + 2 * pw, count);
  ip_moddown(c, dig, count, c->relin, NULL, out, out + pw);
  poly_add(c, out, t, count, 0);
  poly_add(c, out + pw, t + pw, count, 0);
  free(dig);
  CNT(c, relinearizations, 1);
  return LO_OK;
}

/* rescale (ckks.cpp:536-547); out = [2][count-1][N]. */
int lo_rescale(lo_ctx* c, size_t count, const uint64_t* ct, uint64_t* out) {
  if (count < 2) return LO_DEPTH_EXHAUSTED;
  size_t pw = count * c->n, ow = (count - 1) * c->n;
  divide_round_last(c, ct, count, 0, out);
  divide_round_last(c, ct + pw, count, 0, out + ow);
  CNT(c, rescales, 1);
  return LO_OK;
}

/* rotate (ckks.cpp:560-580). */
int lo_rotate(lo_ctx* c, size_t count, const uint64_t* ct, size_t step, uint64_t* out) {
  size_t n = c->n, pw = count * n;
  step %= n / 2;
  if (step == 0) {
    memmove(out, ct, 2 * pw * 8);
    return LO_OK;
  }
  const u64* key = lo_rotation_key(c, step);
  if (!key) return LO_KEY_ERROR;
  const uint32_t* perm = gal(c, step);
  u64* dig = decompose(c, ct + pw, count);
  u64* b = malloc(pw * 8);
  ip_moddown(c, dig, count, key, perm, b, out + pw);
  apply_perm(c, ct, count, perm, out);
  poly_add(c, out, b, count, 0);
  free(b);
  free(dig);
  CNT(c, rotations, 1);
  return LO_OK;
}

/* hoisted_rotations (ckks.cpp:582-612): one decomposition for the batch. */
int lo_hoisted_rotations(lo_ctx* c, size_t count, const uint64_t* ct, const size_t* steps,
                         size_t nsteps, uint64_t* outs) {
  size_t n = c->n, pw = count * n, slots = n / 2;
  u64* dig = NULL;
  u64* b = malloc(pw * 8);
  for (size_t s = 0; s < nsteps; ++s) {
    size_t st = steps[s] % slots;
    u64* o = outs + s * 2 * pw;
    if (st == 0) {
      memcpy(o, ct, 2 * pw * 8);
      continue;
    }
    const u64* key = lo_rotation_key(c, st);
    if (!key) {
      free(dig);
      free(b);
      return LO_KEY_ERROR;
    }
    if (!dig) dig = decompose(c, ct + pw, count);
    const uint32_t* perm = gal(c, st);
    ip_moddown(c, dig, count, key, perm, b, o + pw);
    apply_perm(c, ct, count, perm, o);
    poly_add(c, o, b, count, 0);
    CNT(c, rotations, 1);
  }
  free(dig);
  free(b);
  return LO_OK;
}

/* slot_reduce (distance.cpp:214-240). */
int lo_slot_reduce(lo_ctx* c, size_t count, const uint64_t* ct, size_t width, size_t k,
                   uint64_t* out) {
  size_t n = c->n, pw = count * n;
  if (width == 0 || (width & (width - 1))) return LO_WIDTH_ERROR;
  if (width > n / 2) return LO_WIDTH_ERROR;
  if (k == 0) return LO_PARAMETER_ERROR;
  memmove(out, ct, 2 * pw * 8);
  if (width == 1) return LO_OK;
  size_t levels = (size_t)__builtin_ctzll(width);
  size_t unf = k - 1 < levels ? k - 1 : levels;
  int rc;
  if (unf >= 1) {
    size_t nb = ((size_t)1 << unf) - 1;
    size_t* batch = malloc(nb * sizeof(size_t));
    for (size_t u = 1; u <= nb; ++u) batch[u - 1] = u;
    u64* rot = malloc(nb * 2 * pw * 8);
    u64* base = malloc(2 * pw * 8);
    memcpy(base, ct, 2 * pw * 8);
    rc = lo_hoisted_rotations(c, count, base, batch, nb, rot);
    if (rc == LO_OK)
      for (size_t u = 0; u < nb; ++u) lo_hadd(c, count, out, rot + u * 2 * pw, out);
    free(batch);
    free(rot);
    free(base);
    if (rc) return rc;
  }
  u64* r = malloc(2 * pw * 8);
  for (size_t j = unf; j < levels; ++j) {
    rc = lo_rotate(c, count, out, (size_t)1 << j, r);
    if (rc) {
      free(r);
      return rc;
    }
    lo_hadd(c, count, out, r, out);
  }
  free(r);
  return LO_OK;
}

/* encrypted_pairwise_distance (distance.cpp:107-142); out = [2][full-1][N]. */
int lo_pairwise_distance(lo_ctx* c, size_t chunks, const uint64_t* a, const uint64_t* b,
                         int lazy, uint64_t* out) {
  size_t n = c->n, m = c->full, pw = m * n, ctw = 2 * pw;
  u64* diff = malloc(ctw * 8);
  u64* t = malloc(3 * pw * 8);
  int rc = LO_OK;
  if (lazy) {
    u64* acc = malloc(3 * pw * 8);
    u64* rl = malloc(ctw * 8);
    for (size_t ch = 0; ch < chunks; ++ch) {
      lo_hsub(c, m, a + ch * ctw, b + ch * ctw, diff);
      lo_hsquare(c, m, diff, ch == 0 ? acc : t);
      if (ch) lo_lazy_accumulate(c, m, acc, t);
    }
    rc = lo_relinearize(c, m, acc, rl);
    if (!rc) rc = lo_rescale(c, m, rl, out);
    free(acc);
    free(rl);
  } else {
    u64* rl = malloc(ctw * 8);
    u64* part = malloc(2 * (m - 1) * n * 8);
    for (size_t ch = 0; ch < chunks && !rc; ++ch) {
      lo_hsub(c, m, a + ch * ctw, b + ch * ctw, diff);
      lo_hsquare(c, m, diff, t);
      rc = lo_relinearize(c, m, t, rl);
      if (!rc) rc = lo_rescale(c, m, rl, ch == 0 ? out : part);
      if (!rc && ch) lo_hadd(c, m - 1, out, part, out);
    }
    free(rl);
    free(part);
  }
  free(diff);
  free(t);
  return rc;
}

/* Static block split over worker threads, first error wins (threading.cpp:44-70). */
typedef struct {
  size_t lo, hi;
  int (*fn)(void*, size_t);
  void* arg;
  int rc;
} job_t;

static void* run_job(void* p) {
  job_t* j = p;
  for (size_t i = j->lo; i < j->hi && !j->rc; ++i) j->rc = j->fn(j->arg, i);
  return NULL;
}

static int par_for(int threads, size_t count, int (*fn)(void*, size_t), void* arg) {
  size_t w = (size_t)threads < count ? (size_t)threads : count;
  if (w <= 1) {
    for (size_t i = 0; i < count; ++i) {
      int rc = fn(arg, i);
      if (rc) return rc;
    }
    return LO_OK;
  }
  job_t* jobs = calloc(w, sizeof(job_t));
  pthread_t* th = calloc(w, sizeof(pthread_t));
  for (size_t t = 0; t < w; ++t) {
    jobs[t] = (job_t){count * t / w, count * (t + 1) / w, fn, arg, 0};
    if (t) pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  run_job(&jobs[0]);
  int rc = jobs[0].rc;
  for (size_t t = 1; t < w; ++t) {
    pthread_join(th[t], NULL);
    if (!rc) rc = jobs[t].rc;
  }
  free(jobs);
  free(th);
  return rc;
}

typedef struct {
  lo_ctx* c;
  size_t n, chunks, width, k;
  int lazy, reduce;
  const u64* clients;
  u64* out;
  size_t (*pairs)[2];
} dm_arg;

static int dm_one(void* p, size_t idx) {
  dm_arg* d = p;
  lo_ctx* c = d->c;
  size_t m = c->full, ctw = 2 * m * c->n, ow = 2 * (m - 1) * c->n;
  const u64* a = d->clients + d->pairs[idx][0] * d->chunks * ctw;
  const u64* b = d->clients + d->pairs[idx][1] * d->chunks * ctw;
  u64* o = d->out + idx * ow;
  int rc = lo_pairwise_distance(c, d->chunks, a, b, d->lazy, o);
  if (!rc && d->reduce) rc = lo_slot_reduce(c, m - 1, o, d->width, d->k, o);
  return rc;
}

/* build_distance_matrix, per_pair mode (distance.cpp:242-300). */
int lo_distance_matrix(lo_ctx* c, size_t n, size_t chunks, const uint64_t* clients,
                       size_t width, size_t k, int lazy, int reduce, uint64_t* out) {
  if (n < 2) return LO_SHAPE_ERROR;
  size_t np = n * (n - 1) / 2;
  size_t(*pairs)[2] = malloc(np * sizeof *pairs);
  size_t p = 0;
  for (size_t i = 0; i < n; ++i)
    for (size_t j = i + 1; j < n; ++j) {
      pairs[p][0] = i;
      pairs[p++][1] = j;
    }
  dm_arg a = {c, n, chunks, width, k, lazy, reduce, clients, out, pairs};
  int rc = par_for(c->threads, np, dm_one, &a);
  free(pairs);
  return rc;
}

/* build_distance_matrix, row_sums mode (distance.cpp:257-298): unreduced
 * pair distances, row i = hadd chain over the pairs containing i in pair
 * order, then slot_reduce per row when reduce. out = [n][2][L][N]. */
int lo_distance_rows(lo_ctx* c, size_t n, size_t chunks, const uint64_t* clients,
                     size_t width, size_t k, int lazy, int reduce, uint64_t* out) {
  if (n < 2) return LO_SHAPE_ERROR;
  size_t m = c->full, ow = 2 * (m - 1) * c->n, np = n * (n - 1) / 2;
  u64* pd = malloc(np * ow * 8);
  int rc = lo_distance_matrix(c, n, chunks, clients, width, k, lazy, 0, pd);
  for (size_t i = 0; !rc && i < n; ++i) {
    u64* row = out + i * ow;
    int first = 1;
    size_t p = 0;
    for (size_t a = 0; a < n; ++a)
      for (size_t b = a + 1; b < n; ++b, ++p) {
        if (a != i && b != i) continue;
        if (first) memcpy(row, pd + p * ow, ow * 8);
        else rc = rc ? rc : lo_hadd(c, m - 1, row, pd + p * ow, row);
        first = 0;
      }
    if (!rc && reduce) rc = lo_slot_reduce(c, m - 1, row, width, k, row);
  }
  free(pd);
  return rc;
}

typedef struct {
  lo_ctx* c;
  size_t n, chunks, l;
  int average;
  const u64 *clients, *sel;
  u64* out;
} ag_arg;

/* mult_plain by encode(1/l) at the ct level, then rescale (aggregation.cpp:220-225). */
int lo_mult_plain_inv_l(lo_ctx* c, size_t count, const uint64_t* ct, size_t l, uint64_t* out) {
  size_t n = c->n, slots = n / 2, pw = count * n;
  double* v = malloc(slots * sizeof(double));
  for (size_t i = 0; i < slots; ++i) v[i] = 1.0 / (double)l;
  u64* pt = malloc(pw * 8);
  int rc = lo_encode(c, v, slots, c->scale, (int)count - 1, pt);
  free(v);
  if (rc) {
    free(pt);
    return rc;
  }
  u64* prod = malloc(2 * pw * 8);
  memcpy(prod, ct, 2 * pw * 8);
  poly_mul(c, prod, pt, count, 0);
  poly_mul(c, prod + pw, pt, count, 0);
  CNT(c, multiplications, 1);
  rc = lo_rescale(c, count, prod, out);
  free(prod);
  free(pt);
  return rc;
}

static int ag_one(void* p, size_t ch) {
  ag_arg* g = p;
  lo_ctx* c = g->c;
  size_t m = c->full, pw = m * c->n, ctw = 2 * pw;
  u64* acc = malloc(3 * pw * 8);
  u64* t = malloc(3 * pw * 8);
  u64* rl = malloc(ctw * 8);
  for (size_t i = 0; i < g->n; ++i) {
    const u64* w = g->clients + (i * g->chunks + ch) * ctw;
    lo_hmult_triple(c, m, w, g->sel + i * ctw, i == 0 ? acc : t);
    if (i) lo_lazy_accumulate(c, m, acc, t);
  }
  int rc = lo_relinearize(c, m, acc, rl);
  size_t ow = g->average ? 2 * (m - 2) * c->n : 2 * (m - 1) * c->n;
  u64* o = g->out + ch * ow;
  if (!rc) {
    if (g->average) {
      u64* rs = malloc(2 * (m - 1) * c->n * 8);
      rc = lo_rescale(c, m, rl, rs);
      if (!rc) rc = lo_mult_plain_inv_l(c, m - 1, rs, g->l, o);
      free(rs);
    } else {
      rc = lo_rescale(c, m, rl, o);
    }
  }
  free(acc);
  free(t);
  free(rl);
  return rc;
}

/* masked_aggregate (aggregation.cpp:188-229); average = multi_krum && l > 1. */
int lo_masked_aggregate(lo_ctx* c, size_t n, size_t chunks, const uint64_t* clients,
                        const uint64_t* selectors, size_t l, int average, uint64_t* out) {
  if (n == 0) return LO_SHAPE_ERROR;
  ag_arg g = {c, n, chunks, l, average, clients, selectors, out};
  return par_for(c->threads, chunks, ag_one, &g);
}

/* decrypt (ckks.cpp:381-388) + decode (:313-348). */
int lo_decrypt_values(lo_ctx* c, size_t count, const uint64_t* ct, double scale, double* slots) {
  size_t n = c->n, h = n / 2, pw = count * n;
  u64* m = malloc(pw * 8);
  memcpy(m, ct + pw, pw * 8);
  poly_mul(c, m, c->sk, count, 0);
  poly_add(c, m, ct, count, 0);
  poly_ntt_inv(c, m, count, 0);
  double* co = malloc(n * sizeof(double));
  if (count >= 2) {
    const mod_t *q0 = &c->mod[0], *q1 = &c->mod[1];
    u64 inv01 = invm(redm(q0->v, q1), q1), invs = shoup(inv01, q1);
    u128 q01 = (u128)q0->v * q1->v, half = q01 >> 1;
    for (size_t i = 0; i < n; ++i) {
      u64 r0 = m[i];
      u64 d = subm(m[n + i], redm(r0, q1), q1);
      u64 t = mulsh(d, inv01, invs, q1);
      u128 x = (u128)q0->v * t + r0;
      co[i] = x > half ? -(double)(q01 - x) : (double)x;
      co[i] /= scale;
    }
  } else {
    u64 half = c->mod[0].v >> 1;
    for (size_t i = 0; i < n; ++i) {
      u64 r = m[i];
      co[i] = r > half ? -(double)(c->mod[0].v - r) : (double)r;
      co[i] /= scale;
    }
  }
  cpx* b = malloc(h * sizeof(cpx));
  for (size_t i = 0; i < h; ++i) {
    double ang = M_PI * (double)i / (double)n;
    double tr = cos(ang), ti = sin(ang);
    b[i].re = co[i] * tr - co[i + h] * ti;
    b[i].im = co[i] * ti + co[i + h] * tr;
  }
  emb_fft(c, b, 0);
  for (size_t j = 0; j < h; ++j) slots[j] = b[slot_bucket(c, j)].re;
  free(m);
  free(co);
  free(b);
  return LO_OK;
}
