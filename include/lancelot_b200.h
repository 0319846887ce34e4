/*
 * lancelot_b200.h — C-ABI of the B200-native Lancelot server path.
 *
 * Drop-in boundary for the server half of Lancelot (arXiv 2408.06197): the
 * encrypted pairwise squared-distance matrix and the encrypted masked
 * aggregate, plus the CKKS evaluator primitives they are built from. Every
 * entry point replaces one function of the reference C++ API (paths relative
 * to /root/reference/proj/core) and is bit-exact with it:
 *
 *   lcl_context_create       CkksContext::CkksContext + make_basis     ckks.cpp:77-93, 164-167
 *   lcl_upload_*_key         KeyBundle relin / rotation keys           ckks.hpp:73-97
 *   lcl_ntt_forward/inverse  PolyRns::ntt_forward / ntt_inverse        rns.cpp:282-302
 *   lcl_hadd / lcl_hsub      CkksContext::hadd / hsub                  ckks.cpp:395-415
 *   lcl_hmult / lcl_hsquare  CkksContext::hmult_triple / hsquare       ckks.cpp:417-451
 *   lcl_relinearize          CkksContext::relinearize                  ckks.cpp:522-534
 *   lcl_rescale              CkksContext::rescale                      ckks.cpp:536-547
 *   lcl_rotate               CkksContext::rotate                       ckks.cpp:560-580
 *   lcl_hoisted_rotations    CkksContext::hoisted_rotations            ckks.cpp:582-612
 *   lcl_calibrate            calibrate (make_system, dynamic_lp)       protocol.cpp:224-253
 *   lcl_slot_reduce          slot_reduce                               distance.cpp:214-240
 *   lcl_pairwise_distance    encrypted_pairwise_distance               distance.cpp:107-142
 *   lcl_distance_matrix      build_distance_matrix (per_pair)          distance.cpp:242-300
 *   lcl_build_distance_matrix  build_distance_matrix (both modes)       distance.cpp:242-300
 *   lcl_masked_aggregate     masked_aggregate                          aggregation.cpp:188-229
 *   lcl_*_pairs / _chunks    the same, one shard of pairs / chunks     distance.cpp:257-272,
 *                            (the reference's parallel_for ranges)     aggregation.cpp:211
 *   lcl_get_counts           OpCounters::snapshot                      ckks.cpp:134-156
 *   lcl_deserialize          CkksContext::deserialize (LCLT ingest)    ckks.cpp:640-678
 *   lcl_serialize            CkksContext::serialize                    ckks.cpp:614-638
 *   lcl_server_round_lclt    run_round steps 3 + 8 from received blobs protocol.cpp:419-432
 *   lcl_pack_and_encrypt     pack_and_encrypt (client side)           distance.cpp:64-91
 *   lcl_decrypt / _decode    CkksContext::decrypt / decode (KGC side)  ckks.cpp:313-393,
 *   lcl_decrypt_values       + Embedding::coeffs_to_slots              encoding.cpp:118-134
 *
 * Conventions
 *   - Plain pointers and sizes only. Buffers named d_* are DEVICE pointers on
 *     the context's device; h_* are host pointers.
 *   - Layouts are the reference's (LCLT-compatible): little-endian u64,
 *     limb-major. A ciphertext at `count` live q-limbs is [2][count][N]
 *     (c0 rows then c1 rows); a ternary is [3][count][N]; a switch key is
 *     [full][2][full+1][N] (digit j: k0 rows then k1 rows, special row last).
 *     Client weights are [n][chunks][2][full][N]; selectors [n][2][full][N].
 *   - Every call returns an lcl_status; the codes map 1:1 onto the reference
 *     exception types (errors.hpp:27-104). lcl_last_error() gives the message.
 *   - Work is enqueued on the context's stream (lcl_set_stream; default: the
 *     legacy default stream) and is asynchronous unless stated otherwise.
 *   - Op counters advance exactly as the reference's OpCounters do.
 *   - There is no CPU fallback: without a CUDA device every compute call
 *     fails with LCL_CUDA_ERROR.
 */
#ifndef LANCELOT_B200_H
#define LANCELOT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LCL_OK = 0,
  LCL_PARAMETER_ERROR = 1,  /* ParameterError      */
  LCL_BASIS_MISMATCH = 2,   /* BasisMismatchError  */
  LCL_DOMAIN_ERROR = 3,     /* DomainError         */
  LCL_ALIGNMENT_ERROR = 4,  /* AlignmentError      */
  LCL_KEY_ERROR = 5,        /* KeyError            */
  LCL_DEPTH_EXHAUSTED = 6,  /* DepthExhaustedError */
  LCL_CAPACITY_ERROR = 7,   /* CapacityError       */
  LCL_SHAPE_ERROR = 8,      /* ShapeError          */
  LCL_WIDTH_ERROR = 9,      /* WidthError          */
  LCL_INFEASIBLE_ERROR = 10,/* InfeasibleError     */
  LCL_DATA_ERROR = 11,      /* DataError           */
  LCL_USAGE_ERROR = 12,     /* UsageError          */
  LCL_CUDA_ERROR = 100      /* device failure (no reference counterpart) */
} lcl_status;

typedef struct lcl_context lcl_context;
typedef struct lcl_sampler lcl_sampler;

typedef struct {
  uint64_t encryptions, additions, multiplications, relinearizations, rescales, rotations,
      mod_ups;
} lcl_counts;

/* ------------------------------------------------------------ context */
/* CkksParams{ring_degree = degree, depth, security}: scale 2^40, q0 44 bits,
 * scale primes 40 bits, special prime 54 bits (ckks.hpp:39-55). */
int lcl_context_create(size_t degree, int depth, int secure, int device, lcl_context** out);
int lcl_context_destroy(lcl_context* ctx);
const char* lcl_last_error(void);
/* primes[0..full-1] = q chain, primes[full] = special. */
int lcl_context_primes(const lcl_context* ctx, uint64_t* primes, size_t* full);
int lcl_set_stream(lcl_context* ctx, void* cuda_stream);
int lcl_synchronize(lcl_context* ctx);
int lcl_get_counts(const lcl_context* ctx, lcl_counts* out);
int lcl_reset_counts(lcl_context* ctx);
/* Number of kernel launches issued so far (instrumentation for bench.py). */
uint64_t lcl_launch_count(const lcl_context* ctx);
/* Per-launch CUDA-event timing between begin and end; end writes a JSON list
 * of {name, launches, ms, bytes (algorithmic)} per kernel into json[cap]. */
int lcl_profile_begin(lcl_context* ctx);
/* Integer roofline probe: forward-NTT butterflies/s (Shoup product + lazy
 * add/sub) on register-resident independent chains over the whole device. */
int lcl_peak_butterflies(lcl_context* ctx, double* gbfly_per_s);
/* The same probe for the FP64-pipe butterfly (the q-chain rows' field). */
int lcl_peak_butterflies_f64(lcl_context* ctx, double* gbfly_per_s);
int lcl_profile_end(lcl_context* ctx, char* json, size_t cap);

/* ------------------------------------------------------------ keys */
/* Host key in the reference layout [full][2][full+1][N]; words must equal
 * full * 2 * (full+1) * N. Keys stay resident in HBM. */
int lcl_upload_relin_key(lcl_context* ctx, const uint64_t* h_key, size_t words);
int lcl_upload_rotation_key(lcl_context* ctx, size_t step, const uint64_t* h_key, size_t words);
int lcl_has_rotation_key(const lcl_context* ctx, size_t step);

/* ------------------------------------------------------------ device memory */
int lcl_device_alloc(lcl_context* ctx, size_t bytes, void** d_ptr);
int lcl_device_free(lcl_context* ctx, void* d_ptr);
int lcl_copy_h2d(lcl_context* ctx, void* d_dst, const void* h_src, size_t bytes);
int lcl_copy_d2h(lcl_context* ctx, void* h_dst, const void* d_src, size_t bytes);

/* ------------------------------------------------------------ primitives */
/* Batched negacyclic NTT, in place, over `items` polys of `count` q rows
 * (+ the special row last when with_special). Eval order = reference's. */
int lcl_ntt_forward(lcl_context* ctx, uint64_t* d_polys, size_t items, size_t count,
                    int with_special);
int lcl_ntt_inverse(lcl_context* ctx, uint64_t* d_polys, size_t items, size_t count,
                    int with_special);
/* hadd / hsub (ckks.cpp:395-415) over [batch][2][count][N]; out may alias a. */
int lcl_hadd(lcl_context* ctx, const uint64_t* d_a, const uint64_t* d_b, size_t batch,
             size_t count, uint64_t* d_out);
int lcl_hsub(lcl_context* ctx, const uint64_t* d_a, const uint64_t* d_b, size_t batch,
             size_t count, uint64_t* d_out);
/* batch ternaries [batch][3][count][N] -> ciphertexts [batch][2][count][N]. */
/* CkksContext::hmult_triple (ckks.cpp:417-439, Karatsuba) over `batch` pairs
 * of ciphertexts at `count` limbs: d_tern [batch][3][count][N]. Scales are
 * the caller's (product). multiplications += batch. */
int lcl_hmult(lcl_context* ctx, const uint64_t* d_a, const uint64_t* d_b, size_t batch,
              size_t count, uint64_t* d_tern);
/* CkksContext::hsquare (ckks.cpp:441-451): d0 = c0^2, d1 = 2 c0 c1, d2 = c1^2. */
int lcl_hsquare(lcl_context* ctx, const uint64_t* d_a, size_t batch, size_t count,
                uint64_t* d_tern);
int lcl_relinearize(lcl_context* ctx, const uint64_t* d_tern, size_t batch, size_t count,
                    uint64_t* d_out);
/* [batch][2][count][N] -> [batch][2][count-1][N]; DEPTH_EXHAUSTED at count 1. */
int lcl_rescale(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                uint64_t* d_out);
int lcl_rotate(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count, size_t step,
               uint64_t* d_out);
/* outs: [nsteps][batch][2][count][N]; one decomposition for all steps. */
int lcl_hoisted_rotations(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                          const size_t* h_steps, size_t nsteps, uint64_t* d_outs);
/* calibrate (protocol.cpp:224-253) on the device: the median of 11
 * CUDA-event-timed lcl_hoisted_rotations calls on the fresh ciphertext d_ct
 * ([2][count][N], batch 1) for steps {1} and {1, 2}; *t_hoist = t1,
 * *t_decompose = t2 - t1 (the reference's naming), *m_cipher =
 * Ciphertext::size_bytes. Needs rotation keys 1 and 2 (KeyError otherwise).
 * Synchronises the context stream. Feed the result to plan_unfold
 * (distance.cpp:144-179; mirrored in the C++ / Python hosts). */
int lcl_calibrate(lcl_context* ctx, const uint64_t* d_ct, size_t count, double* t_hoist,
                  double* t_decompose, double* m_cipher);
/* HoistPlan{k, n = width}: first min(k-1, log2 width) levels hoisted. */
int lcl_slot_reduce(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                    size_t width, size_t k, uint64_t* d_out);
/* ct x pt with a plaintext encoded on the host at (value, scale, level). */
int lcl_mult_plain_const(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                         double value, double pt_scale, uint64_t* d_out);

/* Client side.
 * lcl_derive_seed        derive_seed (sampling.cpp:24-30).
 * lcl_sampler_*          Sampler(seed) (sampling.hpp:32-65): the reference's
 *                        mt19937_64 stream; uniform_real draws (sampling.cpp:43-45).
 * lcl_pack_and_encrypt   pack_and_encrypt (distance.cpp:64-91): the client's
 *                        weights (host, dim doubles) chunked, encoded at the
 *                        context scale and encrypted under the public key
 *                        d_pk [2][full][N] (p0 rows then p1 rows, evaluation
 *                        domain) into d_out [chunks][2][full][N]; consumes the
 *                        sampler's draws exactly as the reference does, so the
 *                        words are the reference's. encryptions += chunks. */
uint64_t lcl_derive_seed(uint64_t root, uint64_t tag);
int lcl_sampler_create(uint64_t seed, lcl_sampler** out);
int lcl_sampler_destroy(lcl_sampler* s);
int lcl_sampler_uniform_real(lcl_sampler* s, size_t count, double* out);
int lcl_pack_and_encrypt(lcl_context* ctx, lcl_sampler* rng, const double* h_weights,
                         size_t dim, double prescale, const uint64_t* d_pk, uint64_t* d_out);
/* build_mask (aggregation.cpp:156-186), the KGC's selection mask: n rank rows
 * (d_rank_rows [n][2][full][N]; unused by masked_aggregate, encrypted anyway
 * because they consume the sampler's draws first) and n client selectors
 * (d_selectors [n][2][full][N], all slots 1.0 for a selected client, else 0.0). */
/* generate_keys (ckks.cpp:225-261) from the KGC's Sampler: d_sk [full+1][N]
 * (SecretKey::s, evaluation domain), d_pk [2][full][N] (p0, p1), d_relin
 * [full][2][full+1][N], d_rot [k][full][2][full+1][N] for the k distinct
 * nonzero steps mod slots of steps[0..nsteps) in order (rot_steps[k], *n_rot
 * = k; room for nsteps keys). Word-identical to the reference for the same
 * Sampler state (draws on the host, transforms and products on the device). */
int lcl_generate_keys(lcl_context* ctx, lcl_sampler* rng, const size_t* steps, size_t nsteps,
                      uint64_t* d_sk, uint64_t* d_pk, uint64_t* d_relin, uint64_t* d_rot,
                      size_t* rot_steps, size_t* n_rot);
int lcl_build_mask(lcl_context* ctx, lcl_sampler* rng, size_t n, const size_t* selected,
                   size_t l, const uint64_t* d_pk, uint64_t* d_rank_rows, uint64_t* d_selectors);

/* KGC side, bit-identical to the reference:
 * lcl_decrypt         CkksContext::decrypt (ckks.cpp:381-388): d_pt [batch][count][N] =
 *                     c1 * s + c0 (evaluation domain); d_sk = the first `count` rows of
 *                     SecretKey::s [count][N] (evaluation domain).
 * lcl_decode          CkksContext::decode (ckks.cpp:313-348) + Embedding::coeffs_to_slots
 *                     (encoding.cpp:118-134): d_pt is inverse-transformed in place,
 *                     d_slots [batch][N/2] doubles.
 * lcl_decrypt_values  decrypt_values (ckks.cpp:390-393) = decode(decrypt(ct, sk)). */
int lcl_decrypt(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                const uint64_t* d_sk, uint64_t* d_pt);
int lcl_decode(lcl_context* ctx, uint64_t* d_pt, size_t batch, size_t count, double scale,
               double* d_slots);
int lcl_decrypt_values(lcl_context* ctx, const uint64_t* d_ct, size_t batch, size_t count,
                       double scale, const uint64_t* d_sk, double* d_slots);

/* KGC distance table: table_from_matrix (aggregation.cpp:242-258)
 * and totals_from_matrix (:260-277) over the device matrix entries d_entries
 * [entries][2][count][N] at `scale`: every entry decrypted (lcl_decrypt_values),
 * its value = slot 0 if `reduced` else the left-to-right sum of all slots,
 * max(0, value / value_scale). h_table [n][n] symmetric with a zero diagonal
 * (per_pair entries in (i<j) order); h_totals [n]: row sums of that table
 * (mode LCL_PER_PAIR) or the row_sums entries themselves (LCL_ROW_SUMS).
 * Synchronises. */
int lcl_table_from_matrix(lcl_context* ctx, const uint64_t* d_entries, size_t n, size_t count,
                          double scale, int reduced, double value_scale, const uint64_t* d_sk,
                          double* h_table);
int lcl_totals_from_matrix(lcl_context* ctx, const uint64_t* d_entries, size_t n, int mode,
                           size_t count, double scale, int reduced, double value_scale,
                           const uint64_t* d_sk, double* h_totals);

/* ------------------------------------------------------------ hot path */
/* a, b: [chunks][2][full][N]; out: [2][full-1][N]. lazy != 0 -> one relin. */
int lcl_pairwise_distance(lcl_context* ctx, const uint64_t* d_a, const uint64_t* d_b,
                          size_t chunks, int lazy, uint64_t* d_out);
/* clients [n][chunks][2][full][N] at scale in_scale -> out [pairs][2][full-1][N]
 * in (i<j) row-major order; width/k = HoistPlan n/k; reduce = reduce_on_server.
 * *out_scale receives the output scale (host double bookkeeping). */
int lcl_distance_matrix(lcl_context* ctx, const uint64_t* d_clients, size_t n, size_t chunks,
                        double in_scale, size_t width, size_t k, int lazy, int reduce,
                        uint64_t* d_out, double* out_scale);
/* build_distance_matrix with every DistanceMode and DistanceOptions
 * (distance.cpp:242-300): mode LCL_PER_PAIR -> out [n(n-1)/2][2][full-1][N]
 * in (i<j) order, each pair slot_reduced when reduce_on_server; mode
 * LCL_ROW_SUMS -> out [n][2][full-1][N], row i = sum of the unreduced pair
 * ciphertexts containing client i, slot_reduced once when reduce_on_server
 * (reduce_on_server = !slot_sum_at_kgc, protocol.cpp:555). */
enum { LCL_PER_PAIR = 0, LCL_ROW_SUMS = 1 };
int lcl_build_distance_matrix(lcl_context* ctx, const uint64_t* d_clients, size_t n,
                              size_t chunks, double in_scale, size_t width, size_t k, int mode,
                              int lazy, int reduce_on_server, uint64_t* d_out, double* out_scale);
/* selectors [n][2][full][N]; average = (rule == multi_krum && l > 1);
 * out [chunks][2][full-1 (or full-2 when averaging)][N]. */
int lcl_masked_aggregate(lcl_context* ctx, const uint64_t* d_clients, const uint64_t* d_sel,
                         size_t n, size_t chunks, double w_scale, double sel_scale, size_t l,
                         int average, uint64_t* d_out, double* out_scale);
/* Shards for multi-GPU runs: pairs [pair_begin, pair_end) of the (i<j) order
 * (out [pair_end - pair_begin][2][full-1][N]) and chunks [chunk_begin,
 * chunk_end) of the aggregate. Concatenating the shards in order gives the
 * unsharded result word for word. */
/* run_round steps 3 + 8 on device-resident inputs (protocol.cpp:430-432,
 * 492-493): lcl_distance_matrix (per_pair, lazy, reduced) and
 * lcl_masked_aggregate in one call, the aggregate on its own stream
 * concurrently with the distance matrix; same words and counters. */
int lcl_server_round(lcl_context* ctx, const uint64_t* d_clients, const uint64_t* d_sel,
                     size_t n, size_t chunks, size_t width, size_t k, size_t l, int average,
                     uint64_t* d_dist, uint64_t* d_agg);
int lcl_distance_matrix_pairs(lcl_context* ctx, const uint64_t* d_clients, size_t n,
                              size_t chunks, double in_scale, size_t width, size_t k, int lazy,
                              int reduce, size_t pair_begin, size_t pair_end, uint64_t* d_out,
                              double* out_scale);
/* Chunk-sharded distance matrix (phase A): a rank holding chunks
 * [c0, c1) of every client computes the lazy ternary of EVERY pair over its
 * chunks (lcl_pair_partials, distance.cpp:113-127 restricted to the shard;
 * d_clients [n][c1-c0][2][full][N], d_tern [n(n-1)/2][3][full][N]); the
 * shards' partials are summed as plain integers (NCCL SUM, exact below 2^64)
 * and each rank reduces its pair range mod q (lcl_pair_combine, counting the
 * shards - 1 modular adds that join them) and finishes it: relinearize,
 * rescale, slot_reduce (lcl_pair_finish, distance.cpp:128-141, 296). Summed
 * over ranks, words and counters equal build_distance_matrix's. */
int lcl_pair_partials(lcl_context* ctx, const uint64_t* d_clients, size_t n, size_t chunks,
                      uint64_t* d_tern);
int lcl_pair_combine(lcl_context* ctx, uint64_t* d_tern, size_t pairs, size_t shards);
int lcl_pair_finish(lcl_context* ctx, const uint64_t* d_tern, size_t pairs, size_t width,
                    size_t k, int reduce, uint64_t* d_out);
int lcl_masked_aggregate_chunks(lcl_context* ctx, const uint64_t* d_clients,
                                const uint64_t* d_sel, size_t n, size_t chunks, double w_scale,
                                double sel_scale, size_t l, int average, size_t chunk_begin,
                                size_t chunk_end, uint64_t* d_out, double* out_scale);
/* Host-buffer variant of the server round used by the end-to-end benchmark:
 * H2D of clients + selectors, distance matrix, masked aggregate, D2H of both
 * outputs, synchronised before returning. The transfer is overlapped with
 * the computation (LCLT ingest): the clients arrive in two
 * groups on an internal H2D stream; the pairs the first group completes run
 * their whole chain on one lane while the second group is in flight, the
 * rest on a second lane, and results leave on an internal D2H stream as they
 * are ready (chunk-sliced overlap for n < 4 or integer-pipe q-chains); the
 * words and op counters are those of lcl_distance_matrix +
 * lcl_masked_aggregate. Host buffers should be pinned for full PCIe
 * bandwidth (pageable memory works, slower). */
int lcl_server_round_host(lcl_context* ctx, const uint64_t* h_clients, const uint64_t* h_sel,
                          size_t n, size_t chunks, double in_scale, size_t width, size_t k,
                          size_t l, int average, uint64_t* h_dist, uint64_t* h_agg);

/* ------------------------------------------------------------ LCLT ingest
 * The wire format of CkksContext::serialize / deserialize (ckks.cpp:614-678)
 * and the protocol's .lclt dumps (protocol.cpp:346-360): a 13-byte header
 * ("LCLT", u16 version 1, u32 ring degree, u8 level, u8 scale bits, u8 limb
 * count) followed by the c0 then c1 rows as little-endian u64. A batch of
 * blobs of blob_bytes each sits at a fixed `stride` (>= blob_bytes) in host
 * memory. Header checks run on the host, the residue checks (v < q_i) and
 * the unaligned unpack on the device.
 *
 * lcl_deserialize  CkksContext::deserialize, batched: `count` blobs ->
 *                  d_out [count][2][limbs][N]; *scale = 2^scale_bits. Errors
 *                  (DataError) exactly as the reference: "not a ciphertext
 *                  blob", "unsupported ciphertext format version", "ciphertext
 *                  ring degree does not match the context", "ciphertext level
 *                  inconsistent with the modulus chain", "ciphertext blob
 *                  length mismatch", "residue outside its modulus". Blobs of
 *                  one batch must share level (ShapeError) and scale
 *                  (AlignmentError). Synchronises.
 * lcl_serialize    CkksContext::serialize, batched: d_ct [count][2][limbs][N]
 *                  at `scale` -> blobs at `stride` in h_blobs (ParameterError
 *                  when log2(scale) rounds outside 1..255). Synchronises.
 * lcl_server_round_lclt  lcl_server_round_host fed with the blobs the server
 *                  receives (run_round step 3 deserializes every chunk,
 *                  protocol.cpp:419-429): client i chunk c at h_client_blobs +
 *                  (i * chunks + c) * stride, selector i at h_sel_blobs + i *
 *                  stride, all fresh (top-level). The blob bytes are copied
 *                  verbatim and unpacked on the device inside the overlapped
 *                  H2D pipeline; *dist_scale / *agg_scale receive the output
 *                  scales. Synchronises. */
int lcl_deserialize(lcl_context* ctx, const uint8_t* h_blobs, size_t blob_bytes, size_t stride,
                    size_t count, uint64_t* d_out, double* scale);
int lcl_serialize(lcl_context* ctx, const uint64_t* d_ct, size_t count, size_t limbs,
                  double scale, uint8_t* h_blobs, size_t stride);
int lcl_server_round_lclt(lcl_context* ctx, const uint8_t* h_client_blobs,
                          const uint8_t* h_sel_blobs, size_t blob_bytes, size_t stride, size_t n,
                          size_t chunks, size_t width, size_t k, size_t l, int average,
                          uint64_t* h_dist, uint64_t* h_agg, double* dist_scale,
                          double* agg_scale);

#ifdef __cplusplus
}
#endif

#endif /* LANCELOT_B200_H */
