/*
 * lancelot_oracle — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's server-side CKKS path (Lancelot,
 * arXiv 2408.06197; reference at /root/reference/proj/core) used as the
 * CHECKER for the CUDA product in paper_2408_06197_b200/. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Parity pinning: the outputs of this restatement are compared byte for byte
 * against the unmodified reference core built by oracle/Makefile (oracle/_ref)
 * and against the SHA-256 golden digests committed in tests/golden/ (generated
 * by tests/golden/make_golden.py from oracle/_ref/ref_driver).
 *
 * Layouts (all little-endian u64, limb-major, LCLT-compatible):
 *   poly       [rows][N]; rows = count q-limbs (+1 special row last)
 *   ciphertext [2][count][N]                (c0 rows then c1 rows)
 *   ternary    [3][count][N]                (d0, d1, d2)
 *   switch key [full][2][full+1][N]         (digit j: k0 rows, then k1 rows)
 */
#ifndef LANCELOT_ORACLE_H
#define LANCELOT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lo_ctx lo_ctx;

typedef struct {
  uint64_t encryptions, additions, multiplications, relinearizations, rescales,
      rotations, mod_ups;
} lo_counts;

/* Error codes mirror the reference exception types (errors.hpp:27-104). */
enum {
  LO_OK = 0,
  LO_PARAMETER_ERROR = 1,
  LO_BASIS_MISMATCH = 2,
  LO_DOMAIN_ERROR = 3,
  LO_ALIGNMENT_ERROR = 4,
  LO_KEY_ERROR = 5,
  LO_DEPTH_EXHAUSTED = 6,
  LO_CAPACITY_ERROR = 7,
  LO_SHAPE_ERROR = 8,
  LO_WIDTH_ERROR = 9,
  LO_INFEASIBLE_ERROR = 10,
  LO_DATA_ERROR = 11,
  LO_USAGE_ERROR = 12,
};

/* Context: CkksContext(params) -> make_basis -> RnsBasis (ckks.cpp:77-93,164). */
lo_ctx* lo_ctx_new(size_t degree, int depth, int secure, int threads);
void lo_ctx_free(lo_ctx* c);
int lo_last_error(void);
size_t lo_degree(const lo_ctx* c);
size_t lo_prime_count(const lo_ctx* c);      /* q primes (depth+1) */
uint64_t lo_prime(const lo_ctx* c, size_t i); /* i == prime_count -> special */
uint64_t lo_psi(const lo_ctx* c, size_t i);
double lo_scale(const lo_ctx* c);
lo_counts lo_get_counts(const lo_ctx* c);
void lo_reset_counts(lo_ctx* c);

/* NTT of one row modulo prime i (i == prime_count: special). */
void lo_ntt_forward(const lo_ctx* c, uint64_t* row, size_t i);
void lo_ntt_inverse(const lo_ctx* c, uint64_t* row, size_t i);
void lo_ntt_tables(const lo_ctx* c, size_t i, uint64_t* root, uint64_t* root_shoup,
                   uint64_t* iroot, uint64_t* iroot_shoup, uint64_t* n_inv2);
void lo_galois_perm(const lo_ctx* c, size_t step, uint32_t* perm);
uint64_t lo_galois_elt(size_t degree, size_t step);

/* Key generation (ckks.cpp:196-261) from Sampler(derive_seed(seed, 5)). */
int lo_keygen(lo_ctx* c, uint64_t seed, const size_t* steps, size_t nsteps);
size_t lo_key_words(const lo_ctx* c);   /* u64 words in one switch key */
const uint64_t* lo_relin_key(const lo_ctx* c);
const uint64_t* lo_rotation_key(const lo_ctx* c, size_t step); /* NULL: absent */
const uint64_t* lo_secret_key(const lo_ctx* c); /* (full+1) rows, eval domain */
const uint64_t* lo_public_key_p0(const lo_ctx* c); /* full rows, eval domain */
const uint64_t* lo_public_key_p1(const lo_ctx* c);

/* measure_distance_phase inputs (cli.cpp:316-329): one Sampler stream
 * derive_seed(seed, 0xAB1A7E) shared by all clients; out = [clients][C][2][L+1][N]. */
int lo_make_clients(lo_ctx* c, uint64_t seed, size_t clients, size_t dim,
                    double prescale, uint64_t* out);
size_t lo_chunk_count(const lo_ctx* c, size_t dim);
/* build_mask (aggregation.cpp:156-186); selectors out = [n][2][L+1][N]. */
int lo_build_mask(lo_ctx* c, uint64_t seed, const size_t* selected, size_t nsel,
                  size_t n, uint64_t* selectors);

/* Evaluator (ckks.cpp:395-612). count = live q-limbs of the input. */
int lo_hsub(lo_ctx* c, size_t count, const uint64_t* a, const uint64_t* b, uint64_t* out);
int lo_hadd(lo_ctx* c, size_t count, const uint64_t* a, const uint64_t* b, uint64_t* out);
int lo_hsquare(lo_ctx* c, size_t count, const uint64_t* a, uint64_t* tern);
int lo_hmult_triple(lo_ctx* c, size_t count, const uint64_t* a, const uint64_t* b,
                    uint64_t* tern);
int lo_lazy_accumulate(lo_ctx* c, size_t count, uint64_t* acc, const uint64_t* t);
int lo_relinearize(lo_ctx* c, size_t count, const uint64_t* tern, uint64_t* out);
int lo_rescale(lo_ctx* c, size_t count, const uint64_t* ct, uint64_t* out);
int lo_rotate(lo_ctx* c, size_t count, const uint64_t* ct, size_t step, uint64_t* out);
int lo_hoisted_rotations(lo_ctx* c, size_t count, const uint64_t* ct,
                         const size_t* steps, size_t nsteps, uint64_t* outs);
int lo_slot_reduce(lo_ctx* c, size_t count, const uint64_t* ct, size_t width,
                   size_t k, uint64_t* out);
int lo_mult_plain_inv_l(lo_ctx* c, size_t count, const uint64_t* ct, size_t l,
                        uint64_t* out);
int lo_encode(lo_ctx* c, const double* values, size_t nvalues, double scale,
              int level, uint64_t* out);

/* L3 hot path (distance.cpp:107-142, 242-300; aggregation.cpp:188-229).
 * clients = [n][C][2][L+1][N]; out = [pairs][2][L][N] in (i<j) order. */
int lo_pairwise_distance(lo_ctx* c, size_t chunks, const uint64_t* a,
                         const uint64_t* b, int lazy, uint64_t* out);
int lo_distance_matrix(lo_ctx* c, size_t n, size_t chunks, const uint64_t* clients,
                       size_t width, size_t k, int lazy, int reduce, uint64_t* out);
/* row_sums mode (distance.cpp:287-298): out = [n][2][L][N]. */
int lo_distance_rows(lo_ctx* c, size_t n, size_t chunks, const uint64_t* clients,
                     size_t width, size_t k, int lazy, int reduce, uint64_t* out);
int lo_masked_aggregate(lo_ctx* c, size_t n, size_t chunks, const uint64_t* clients,
                        const uint64_t* selectors, size_t l, int average,
                        uint64_t* out);

/* Decrypt + decode (ckks.cpp:313-348, 381-393): slots = N/2 doubles. */
int lo_decrypt_values(lo_ctx* c, size_t count, const uint64_t* ct, double scale,
                      double* slots);

/* Sampler restatement (sampling.cpp:25-116), exposed for golden checks. */
uint64_t lo_derive_seed(uint64_t root, uint64_t tag);

#ifdef __cplusplus
}
#endif

#endif /* LANCELOT_ORACLE_H */
