/*
 * cbrng_b200.h — C ABI of the B200-native counter-based RNG hot path.
 *
 * Drop-in boundary for the reference package `cbrng`
 * (/root/reference/pkg/src/cbrng). The reference has no FFI: its boundary is
 * Python functions over numpy arrays plus three numba-compiled kernels
 * (_kernels.py:22, :54, :89). Each entry point below names the reference
 * interface it replaces (file:line, relative to pkg/src/cbrng/).
 *
 * Conventions (all entry points):
 *  - plain pointers and sizes; no torch types. Buffers marked [dev] are CUDA
 *    device pointers owned by the caller (e.g. torch tensors' data_ptr()),
 *    [host] are host pointers.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Work is
 *    enqueued asynchronously unless the function says it synchronises.
 *  - return 0 on success, <0 on error (CBRNG_E*); cbrng_last_error() gives a
 *    message for the calling thread. Argument errors map to the reference's
 *    ValueError cases (bulk.py:225-226, generators.py:68-73, brownian.py:151-152).
 *  - reentrant: no global mutable state besides per-device launch-geometry
 *    caches (initialised once, thread-safe) and the thread-local error text.
 *  - algorithm ids follow generators.py:59-65 (Algorithm enum tags).
 */
#ifndef CBRNG_B200_H
#define CBRNG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    CBRNG_PHILOX = 0,   /* generators.py:62 */
    CBRNG_THREEFRY = 1, /* generators.py:63 */
    CBRNG_SQUARES = 2,  /* generators.py:64 */
    CBRNG_TYCHE = 3     /* generators.py:65 */
};

enum {
    CBRNG_OK = 0,
    CBRNG_EINVAL = -1, /* bad argument (reference: ValueError) */
    CBRNG_EALG = -2,   /* unknown algorithm (reference: ValueError, generators.py:68-73) */
    CBRNG_ECUDA = -3,  /* CUDA launch/runtime error */
    CBRNG_EALIGN = -4  /* device pointer not aligned for the element type */
};

/* Brownian step-kernel modes. */
enum {
    CBRNG_BROWNIAN_PER_STEP = 0, /* one launch per step (paper Fig. 1 shape) */
    CBRNG_BROWNIAN_FUSED = 1     /* all steps in one launch, particle kept in registers */
};

const char *cbrng_version(void);
const char *cbrng_last_error(void);
int cbrng_device_sm_count(int device);

/* ---------------- single-stream fills (Generator.words & distributions) ----------------
 * Stream (alg, seed, stream_ctr) positioned at stream word `word_pos`
 * (Philox/Threefry: block (word_pos >> 2) mod 2^32, word word_pos & 3 of it —
 * a generator resumed mid-block, generators.py:306-311; Squares: counter
 * word_pos mod 2^32). Block counters wrap mod 2^32 (bulk.py:215-217, :268).
 * For Tyche, `tyche_state` [host, 4 x u32] is the serial state to continue from
 * (generators.py:221-224; seed/stream_ctr/word_pos are ignored) and the state
 * after the last word is written to `tyche_state_out` [dev, 4 x u32] if non-NULL.
 * Output pointers must be 16-byte aligned (8 for normal2). */

/* bulk.generator_words (bulk.py:223-281) -> out[dev] u32[n] */
int cbrng_words(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos,
                const uint32_t *tyche_state, uint64_t n, uint32_t *out,
                uint32_t *tyche_state_out, void *stream);

/* distributions.uniform_f32_array (distributions.py:105-107): 1 word / value */
int cbrng_uniform_f32(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos,
                      const uint32_t *tyche_state, uint64_t n, float *out,
                      uint32_t *tyche_state_out, void *stream);

/* distributions.uniform_f64_array (distributions.py:99-102): 2 words / value, low first */
int cbrng_uniform_f64(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos,
                      const uint32_t *tyche_state, uint64_t n, double *out,
                      uint32_t *tyche_state_out, void *stream);

/* distributions.normal2_array (distributions.py:110-120): 4 words / pair,
 * two output arrays z0[n_pairs], z1[n_pairs] */
int cbrng_normal2_f64(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos,
                      const uint32_t *tyche_state, uint64_t n_pairs, double *z0, double *z1,
                      uint32_t *tyche_state_out, void *stream);

/* Box-Muller of caller-supplied words, 4 per pair (normal2, distributions.py:72-81,
 * applied to any word source: the reference's scripted-generator tests,
 * test_distributions.py:29-40, 178-186). words [dev, u32, 16-byte aligned],
 * z0/z1 [dev, f64]. Same arithmetic and tolerance as cbrng_normal2_f64. */
int cbrng_normal2_from_words(const uint32_t *words, uint64_t n_pairs, double *z0, double *z1, void *stream);

/* Batched fills: job i = cbrng_words / cbrng_uniform_f32 of (algs[i], seeds[i],
 * stream_ctrs[i] (NULL: all 0), word_pos[i], n[i]) into outs[i] [dev], in
 * order, same results as the per-job calls. Counter-based generators only
 * (Tyche: CBRNG_EINVAL). With CBRNG_MULTI=1 a Philox, a Threefry and a Squares
 * job run interleaved in one kernel (measured no faster than back-to-back
 * launches on B200, the default). No reference counterpart: the reference
 * fills generators one call at a time (bulk.py:223-281); this is the batched
 * form of that call. Job arrays are host memory. */
int cbrng_words_multi(int n_jobs, const int *algs, const uint64_t *seeds, const uint32_t *stream_ctrs,
                      const uint64_t *word_pos, const uint64_t *n, uint32_t *const *outs, void *stream);
int cbrng_uniform_f32_multi(int n_jobs, const int *algs, const uint64_t *seeds, const uint32_t *stream_ctrs,
                            const uint64_t *word_pos, const uint64_t *n, float *const *outs, void *stream);

/* _kernels.tyche_fill (_kernels.py:22-44): state [host, 4 x u64 < 2^32] in/out.
 * SYNCHRONOUS: waits for the stream so the final state is back in `state`. */
int cbrng_tyche_fill(uint64_t *state, uint64_t n, uint32_t *out, void *stream);

/* ---------------- multi-stream fills ----------------
 * bulk.prefix_words (bulk.py:162-207): out[i*nwords + j] = word j of stream
 * (seeds[i], ctrs[i]). seeds == NULL -> seeds[i] = seed_base + i (the
 * np.arange(n) pid layout, brownian.py:118); ctrs == NULL -> ctr_scalar for all.
 * seeds [dev, u64], ctrs [dev, u32], out [dev]. */
int cbrng_prefix_words(int alg, const uint64_t *seeds, uint64_t seed_base, const uint32_t *ctrs,
                       uint32_t ctr_scalar, uint64_t n_streams, uint32_t nwords, uint32_t *out,
                       void *stream);

/* same streams mapped through uniform_f32 (one word per value). */
int cbrng_prefix_uniform_f32(int alg, const uint64_t *seeds, uint64_t seed_base, const uint32_t *ctrs,
                             uint32_t ctr_scalar, uint64_t n_streams, uint32_t nvalues, float *out,
                             void *stream);

/* _kernels.philox_block_lanes (_kernels.py:54-86): out[dev] u32[n][4] = Philox
 * block `block_ctr` of stream (seeds[i], stream_ctrs[i]). */
int cbrng_philox_block_lanes(const uint64_t *seeds, const uint64_t *stream_ctrs, uint64_t block_ctr,
                             uint64_t n, uint32_t *out, void *stream);

/* ---------------- vector block functions (bulk.py:49-159) ----------------
 * Structure-of-arrays [dev] inputs/outputs, one cipher evaluation per lane. */
/* bulk.philox4x32 (bulk.py:49-66): ctr u32[4][n], key u32[2][n] -> out u32[4][n] */
int cbrng_philox4x32(const uint32_t *ctr, const uint32_t *key, uint64_t n, uint32_t *out, void *stream);
/* bulk.threefry4x32 (bulk.py:69-92) + threefry_block(rounds=) (generators.py:125-127):
 * ctr u32[4][n], key u32[4][n] */
int cbrng_threefry4x32(const uint32_t *ctr, const uint32_t *key, int rounds, uint64_t n, uint32_t *out,
                       void *stream);
/* bulk.squares32 (bulk.py:95-108): ctr u64[n], key u64[n] -> out u32[n] */
int cbrng_squares32(const uint64_t *ctr, const uint64_t *key, uint64_t n, uint32_t *out, void *stream);
/* bulk.squares_keys (bulk.py:111-118) */
int cbrng_squares_keys(const uint64_t *seeds, uint64_t n, uint64_t *keys, void *stream);
/* bulk.tyche_mix (bulk.py:121-131) applied `rounds` times: state u32[4][n] in/out */
int cbrng_tyche_mix(uint32_t *state, uint64_t n, uint32_t rounds, void *stream);
/* bulk.tyche_init (bulk.py:134-146): seeds u64[n] (or seed_base+i), ctrs u32[n] (or scalar) -> state u32[4][n] */
int cbrng_tyche_init(const uint64_t *seeds, uint64_t seed_base, const uint32_t *ctrs, uint32_t ctr_scalar,
                     uint64_t n, uint32_t *state, void *stream);

/* ---------------- scalar calls (generators.py:101-224, 295-320) ----------------
 * One synchronous round trip for the reference's scalar API: args and the result
 * are HOST memory; the library stages them through a mapped pinned buffer and
 * runs the vector kernels above on one lane on an internal per-device stream.
 * nargs / nout per op:
 *   PHILOX_BLOCK   ctr0..3, key0..1                      -> 4 words   (generators.py:101-122)
 *   THREEFRY_BLOCK ctr0..3, key0..3, rounds              -> 4 words   (generators.py:125-154)
 *   SQUARES_KEY    seed                                  -> key lo, hi (generators.py:157-170)
 *   SQUARES_ROUND  key, ctr                              -> 1 word    (generators.py:173-187)
 *   TYCHE_INIT     seed, stream_ctr                      -> state[4]  (generators.py:190-218)
 *   TYCHE_MIX      state0..3, rounds                     -> state[4]  (generators.py:201-210)
 *   STREAM_WORDS   alg (0-2), seed, stream_ctr, word_pos -> nout words (<= 2^18) of cbrng_words
 *   TYCHE_WORDS    state0..3                             -> nout-4 words, then the state after them
 *   TYCHE_SEED_WORDS seed, stream_ctr                    -> the state after tyche_init (4), nout-8 words,
 *                                                           then the state after them (a fresh stream's
 *                                                           first window in one round trip) */
enum {
    CBRNG_SCALAR_PHILOX_BLOCK = 0, CBRNG_SCALAR_THREEFRY_BLOCK = 1, CBRNG_SCALAR_SQUARES_KEY = 2,
    CBRNG_SCALAR_SQUARES_ROUND = 3, CBRNG_SCALAR_TYCHE_INIT = 4, CBRNG_SCALAR_TYCHE_MIX = 5,
    CBRNG_SCALAR_STREAM_WORDS = 6, CBRNG_SCALAR_TYCHE_WORDS = 7, CBRNG_SCALAR_TYCHE_SEED_WORDS = 8
};
int cbrng_scalar(int op, const uint64_t *args, uint32_t nargs, uint32_t *out, uint64_t nout);

/* ---------------- Brownian walk (brownian.py) ----------------
 * SoA float64 particle arrays [dev]. pid == NULL -> pid[i] = pid_base + i. */
/* init_particles (brownian.py:112-126) */
int cbrng_brownian_init(int alg, uint64_t n, const uint64_t *pid, uint64_t pid_base, uint32_t init_ctr,
                        double *x, double *y, double *vx, double *vy, void *stream);
/* nsteps x _step_slice (brownian.py:129-142) for iterations first_it..first_it+nsteps-1,
 * counter = (init_ctr + it) mod 2^32. first_it >= 1 (brownian.py:151-152). */
int cbrng_brownian_steps(int alg, uint64_t n, const uint64_t *pid, uint64_t pid_base,
                         double *x, double *y, double *vx, double *vy, uint32_t init_ctr,
                         uint64_t first_it, uint64_t nsteps, double gamma, double mass, double dt,
                         int mode, void *stream);
/* Deterministic statistics of a particle range, accumulated (+=, mod 2^64) into
 * acc[dev, 8 x i64]: [0] n, [1] sum x, [2] sum y, [3] sum vx, [4] sum vy (fixed point
 * 2^-32), [5] sum x^2+y^2, [6] sum vx^2+vy^2 (fixed point 2^-24), [7] order-free
 * position-aware digest of the (pid, x, y, vx, vy) bits. Integer sums are
 * associative, so any sharding gives identical bits. */
int cbrng_brownian_stats(uint64_t n, const uint64_t *pid, uint64_t pid_base, const double *x,
                         const double *y, const double *vx, const double *vy, int64_t *acc,
                         void *stream);

/* Snapshot / checksum records (brownian.py:198-250): n pid-ordered 40-byte `<Qdddd`
 * records (pid u64, x, y, vx, vy f64, little-endian) packed from / unpacked to the SoA
 * arrays, all [dev]; rec must be 8-byte aligned. unpack: pid may be NULL (dropped). */
int cbrng_pack_records(uint64_t n, const uint64_t *pid, uint64_t pid_base, const double *x, const double *y,
                       const double *vx, const double *vy, uint8_t *rec, void *stream);
int cbrng_unpack_records(uint64_t n, const uint8_t *rec, uint64_t *pid, double *x, double *y, double *vx,
                         double *vy, void *stream);
/* *bad [dev, u32] is set to 1 if pid[0..n) is not strictly increasing (checksum
 * precondition, brownian.py:209-212); it is never cleared. */
int cbrng_pid_order_check(uint64_t n, const uint64_t *pid, uint32_t *bad, void *stream);

/* ---------------- invariance digest ----------------
 * acc[dev, u64] += sum_i mix64(global_offset + i, words[i]) mod 2^64: an order-free,
 * position-aware digest used to prove results are identical for any GPU count. */
int cbrng_digest_u32(const uint32_t *words, uint64_t n, uint64_t global_offset, uint64_t *acc, void *stream);

/* ---------------- statistical-battery producers ----------------
 * Generators fused with the reductions of stats.py; counts are u64 [dev] and
 * accumulated (+=), exact and order-independent. */
/* byte histogram of n_words words of one stream (monobit / chi_square_bytes on
 * run_battery's stream, stats.py:117-139, :300-306); same stream addressing and
 * Tyche state convention as cbrng_words. counts: u64[256]. */
int cbrng_stream_byte_histogram(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos,
                                const uint32_t *tyche_state, uint64_t n_words, uint64_t *counts,
                                uint32_t *tyche_state_out, void *stream);
/* byte histogram of prefix_words(alg, seed_base + arange(n_streams), ctr0 + t, nwords) over
 * t = 0..n_ctrs-1, i.e. n_ctrs iterations of iter_interleave_chunks (stats.py:276-286), one launch. */
int cbrng_prefix_byte_histogram(int alg, uint64_t seed_base, uint32_t ctr0, uint32_t n_ctrs, uint64_t n_streams,
                                uint32_t nwords, uint64_t *counts, void *stream);
/* byte histogram of n bytes at data [dev, 4-byte aligned] (monobit(data), stats.py:117). */
int cbrng_buffer_byte_histogram(const uint8_t *data, uint64_t n, uint64_t *counts, void *stream);
/* avalanche_stats (stats.py:171-192): out[0] += sum popcount(w0 ^ w1), out[1 + b] += trials whose
 * bit b differs, w0/w1 = first word of (seeds[i], ctrs[i]) / (seeds[i] ^ flips[i], ctrs[i]). */
int cbrng_avalanche(int alg, const uint64_t *seeds, const uint32_t *ctrs, const uint64_t *flips, uint64_t n,
                    uint64_t *out, void *stream);
/* Pearson sums for interstream_correlation (stats.py:205-246): partials[k*5 + (0..4)] =
 * (sum a, sum b, sum a^2, sum b^2, sum ab) of block k; reduce blocks in order on the host. */
int cbrng_pearson_partials(const double *a, const double *b, uint64_t n, uint32_t n_blocks, double *partials,
                           void *stream);

/* _kernels.fnv1a64 (_kernels.py:89-96): byte-serial by definition, host only. */
uint64_t cbrng_fnv1a64(const uint8_t *data, uint64_t n, uint64_t h);

#ifdef __cplusplus
}
#endif
#endif /* CBRNG_B200_H */
