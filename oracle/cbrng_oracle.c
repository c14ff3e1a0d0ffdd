/*
 * cbrng_oracle.c — CPU restatement of the OpenRAND/cbrng reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker and the CPU
 * baseline ("cpu_baseline.kind = port"). Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The product
 * (paper_2310_19925_b200) never links or calls it.
 *
 * Parity pinned: every function below is checked against fixtures frozen from
 * the reference package itself (tests/golden/make_golden.py ->
 * tests/golden/golden.{json,npz}); see tests/test_oracle.py.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/cbrng/).
 *
 * Build: oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off). FP contraction
 * is disabled because the reference's float64 arithmetic is numpy/CPython
 * double ops, each individually rounded.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define M32 0xFFFFFFFFu

enum { ALG_PHILOX = 0, ALG_THREEFRY = 1, ALG_SQUARES = 2, ALG_TYCHE = 3 };

/* generators.py:35-54 */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u
#define THREEFRY_PARITY 0x1BD11BDAu
#define TYCHE_INIT_CONST 0x9E3779B9u
#define GOLDEN64 0x9E3779B97F4A7C15ull
#define SPLITMIX_M1 0xBF58476D1CE4E5B9ull
#define SPLITMIX_M2 0x94D049BB133111EBull

static const int TF_ROT[8][2] = {{10, 26}, {11, 21}, {13, 27}, {23, 5},
                                 {6, 20},  {17, 11}, {25, 10}, {18, 20}};

static inline uint32_t rotl32(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* generators.py:101-122 — Philox4x32-10. */
void orc_philox_block(const uint32_t key[2], const uint32_t ctr[4], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
        uint64_t p0 = (uint64_t)PHILOX_M0 * c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n1 = (uint32_t)p1;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* generators.py:125-154 — Threefry4x32 with key injection every 4 rounds. */
void orc_threefry_block(const uint32_t key[4], const uint32_t ctr[4], int rounds, uint32_t out[4]) {
    uint32_t ks[5] = {key[0], key[1], key[2], key[3],
                      THREEFRY_PARITY ^ key[0] ^ key[1] ^ key[2] ^ key[3]};
    uint32_t x[4];
    for (int i = 0; i < 4; i++) x[i] = ctr[i] + ks[i];
    for (int r = 0; r < rounds; r++) {
        int r0 = TF_ROT[r % 8][0], r1 = TF_ROT[r % 8][1];
        if (r % 2 == 0) {
            x[0] += x[1]; x[1] = rotl32(x[1], r0) ^ x[0];
            x[2] += x[3]; x[3] = rotl32(x[3], r1) ^ x[2];
        } else {
            x[0] += x[3]; x[3] = rotl32(x[3], r0) ^ x[0];
            x[2] += x[1]; x[1] = rotl32(x[1], r1) ^ x[2];
        }
        if ((r + 1) % 4 == 0) {
            uint32_t j = (uint32_t)((r + 1) / 4);
            for (int i = 0; i < 4; i++) x[i] += ks[(j + i) % 5];
            x[3] += j;
        }
    }
    for (int i = 0; i < 4; i++) out[i] = x[i];
}

/* generators.py:157-170 — SplitMix-style 32->64-bit odd key. */
uint64_t orc_squares_key(uint64_t seed) {
    uint64_t s = seed & M32;
    uint64_t z = s + GOLDEN64;
    z = (z ^ (z >> 30)) * SPLITMIX_M1;
    z = (z ^ (z >> 27)) * SPLITMIX_M2;
    z ^= z >> 31;
    return (z ^ (s << 32)) | 1ull;
}

/* generators.py:173-187 — squares32. */
uint32_t orc_squares_round(uint64_t key, uint64_t ctr) {
    uint64_t x = ctr * key, y = x, z = y + key;
    x = x * x + y; x = (x >> 32) | (x << 32);
    x = x * x + z; x = (x >> 32) | (x << 32);
    x = x * x + y; x = (x >> 32) | (x << 32);
    return (uint32_t)((x * x + z) >> 32);
}

/* generators.py:190-201 — one ChaCha quarter round over (a, b, c, d). */
void orc_tyche_mix(uint32_t s[4]) {
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3];
    a += b; d = rotl32(d ^ a, 16);
    c += d; b = rotl32(b ^ c, 12);
    a += b; d = rotl32(d ^ a, 8);
    c += d; b = rotl32(b ^ c, 7);
    s[0] = a; s[1] = b; s[2] = c; s[3] = d;
}

/* generators.py:204-218 */
void orc_tyche_init(uint64_t seed, uint32_t sc, uint32_t s[4]) {
    s[0] = (uint32_t)(seed >> 32); s[1] = (uint32_t)seed; s[2] = TYCHE_INIT_CONST; s[3] = sc;
    for (int i = 0; i < 20; i++) orc_tyche_mix(s);
}

/* Stream mapping, generators.py:267-275 and :285-312: block `bc` of stream
 * (seed, sc) for the 4-word algorithms. */
static inline void block_of(int alg, uint64_t seed, uint32_t sc, uint32_t bc, uint32_t out[4]) {
    if (alg == ALG_PHILOX) {
        uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
        uint32_t ctr[4] = {sc, bc, 0, 0};
        orc_philox_block(key, ctr, out);
    } else {
        uint32_t key[4] = {(uint32_t)seed, (uint32_t)(seed >> 32), sc, 0};
        uint32_t ctr[4] = {bc, 0, 0, 0};
        orc_threefry_block(key, ctr, 20, out);
    }
}

/*
 * Single stream, the semantics of n x Generator.next_u32 (generators.py:295-312;
 * bulk path bulk.py:223-281): start at block counter `bc0` with `lane` words of
 * that block already served (0..3, 4-word algorithms only), emit n words. Block
 * counters wrap mod 2^32 (bulk.py:215-217, :268). Tyche runs serially from
 * tyche_state (in/out, _kernels.py:22-44). Returns 0, or -1 on a bad argument.
 */
int orc_words(int alg, uint64_t seed, uint32_t sc, uint32_t bc0, uint32_t lane, uint64_t n,
              uint32_t *out, uint32_t *tyche_state) {
    if (alg == ALG_PHILOX || alg == ALG_THREEFRY) {
        if (lane > 3) return -1;
        uint64_t total = (uint64_t)lane + n;
        int64_t nblocks = (int64_t)((total + 3) / 4);
#pragma omp parallel for schedule(static)
        for (int64_t b = 0; b < nblocks; b++) {
            uint32_t blk[4];
            block_of(alg, seed, sc, (uint32_t)(bc0 + (uint64_t)b), blk);
            for (int j = 0; j < 4; j++) {
                int64_t pos = b * 4 + j - (int64_t)lane;
                if (pos >= 0 && (uint64_t)pos < n) out[pos] = blk[j];
            }
        }
        return 0;
    }
    if (alg == ALG_SQUARES) {
        uint64_t key = orc_squares_key(seed);
        uint64_t base = (uint64_t)sc << 32;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < (int64_t)n; i++)
            out[i] = orc_squares_round(key, base | (uint32_t)(bc0 + (uint64_t)i));
        return 0;
    }
    if (alg == ALG_TYCHE) {
        uint32_t s[4];
        if (tyche_state) memcpy(s, tyche_state, sizeof s);
        else orc_tyche_init(seed, sc, s);
        for (uint64_t i = 0; i < n; i++) { orc_tyche_mix(s); out[i] = s[1]; }
        if (tyche_state) memcpy(tyche_state, s, sizeof s);
        return 0;
    }
    return -1;
}

/*
 * Multi-stream prefix words, bulk.py:162-207: out[i*nwords + j] = word j of
 * stream (seeds[i], ctrs[i]). seeds == NULL means seeds[i] = seed_base + i;
 * ctrs == NULL means every stream uses ctr_scalar.
 */
int orc_prefix_words(int alg, const uint64_t *seeds, uint64_t seed_base, const uint32_t *ctrs,
                     uint32_t ctr_scalar, uint64_t n_streams, uint32_t nwords, uint32_t *out) {
    if (alg < 0 || alg > 3) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n_streams; i++) {
        uint64_t seed = seeds ? seeds[i] : seed_base + (uint64_t)i;
        uint32_t sc = ctrs ? ctrs[i] : ctr_scalar;
        uint32_t *row = out + (uint64_t)i * nwords;
        if (alg == ALG_SQUARES) seed &= M32; /* generators.py:256-257 */
        orc_words(alg, seed, sc, 0, 0, nwords, row, NULL);
    }
    return 0;
}

/* distributions.py:105-107 — (w >> 8) * 2^-24, computed in double then cast. */
void orc_words_to_f32(const uint32_t *w, uint64_t n, float *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) out[i] = (float)((double)(w[i] >> 8) * 0x1p-24);
}

/* distributions.py:99-102 — ((lo | hi << 32) >> 11) * 2^-53, low word first. */
void orc_words_to_f64(const uint32_t *w, uint64_t n, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) {
        uint64_t u = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
        out[i] = (double)(u >> 11) * 0x1p-53;
    }
}

/* distributions.py:110-120 — bulk Box-Muller over 4 words per pair, libm. */
void orc_words_to_normal2(const uint32_t *w, uint64_t n_pairs, double *z0, double *z1) {
    const double two_pi = 2.0 * M_PI;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n_pairs; i++) {
        const uint32_t *q = w + 4 * i;
        uint64_t a = (uint64_t)q[0] | ((uint64_t)q[1] << 32);
        uint64_t b = (uint64_t)q[2] | ((uint64_t)q[3] << 32);
        double u1 = 1.0 - (double)(a >> 11) * 0x1p-53;
        double u2 = (double)(b >> 11) * 0x1p-53;
        double r = sqrt(-2.0 * log(u1));
        double t = two_pi * u2;
        z0[i] = r * cos(t);
        z1[i] = r * sin(t);
    }
}

/* Fused CPU fill (the CPU-baseline shape): uniform f32 of one stream, chunked so
 * no intermediate word array is materialised beyond 4096 words per thread. */
int orc_uniform_f32(int alg, uint64_t seed, uint32_t sc, uint64_t n, float *out) {
    if (alg == ALG_TYCHE) {
        uint32_t s[4], buf[4096];
        orc_tyche_init(seed, sc, s);
        for (uint64_t lo = 0; lo < n; lo += 4096) {
            uint64_t k = n - lo < 4096 ? n - lo : 4096;
            for (uint64_t i = 0; i < k; i++) { orc_tyche_mix(s); buf[i] = s[1]; }
            for (uint64_t i = 0; i < k; i++) out[lo + i] = (float)((double)(buf[i] >> 8) * 0x1p-24);
        }
        return 0;
    }
    if (alg < 0 || alg > 3) return -1;
    int64_t nchunks = (int64_t)((n + 4095) / 4096);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nchunks; c++) {
        uint32_t buf[4096];
        uint64_t lo = (uint64_t)c * 4096, k = n - lo < 4096 ? n - lo : 4096;
        /* chunk start is a multiple of 4 words -> block boundary */
        uint32_t bc = (alg == ALG_SQUARES) ? (uint32_t)lo : (uint32_t)(lo / 4);
        if (alg == ALG_SQUARES) {
            uint64_t key = orc_squares_key(seed), base = (uint64_t)sc << 32;
            for (uint64_t i = 0; i < k; i++) buf[i] = orc_squares_round(key, base | (uint32_t)(bc + i));
        } else {
            for (uint64_t b = 0; b < (k + 3) / 4; b++) {
                uint32_t blk[4];
                block_of(alg, seed, sc, bc + (uint32_t)b, blk);
                for (int j = 0; j < 4 && b * 4 + j < k; j++) buf[b * 4 + j] = blk[j];
            }
        }
        for (uint64_t i = 0; i < k; i++) out[lo + i] = (float)((double)(buf[i] >> 8) * 0x1p-24);
    }
    return 0;
}

static inline double unit_double(uint32_t lo, uint32_t hi) {
    /* brownian.py:107-109 */
    uint64_t u = (uint64_t)lo | ((uint64_t)hi << 32);
    return (double)(u >> 11) * 0x1p-53;
}

/* brownian.py:112-126 — 8 words of stream (pid, init_counter) per particle.
 * pid == NULL means pid[i] = i (brownian.py:118). */
int orc_brownian_init(int alg, uint64_t n, const uint64_t *pid, uint32_t init_ctr,
                      double *x, double *y, double *vx, double *vy) {
    if (alg < 0 || alg > 3) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) {
        uint32_t w[8];
        uint64_t seed = pid ? pid[i] : (uint64_t)i;
        if (alg == ALG_SQUARES) seed &= M32;
        orc_words(alg, seed, init_ctr, 0, 0, 8, w, NULL);
        x[i] = unit_double(w[0], w[1]);
        y[i] = unit_double(w[2], w[3]);
        vx[i] = unit_double(w[4], w[5]) * 2.0 - 1.0;
        vy[i] = unit_double(w[6], w[7]) * 2.0 - 1.0;
    }
    return 0;
}

/* brownian.py:129-142 (_step_slice) for iterations first_it .. first_it+nsteps-1,
 * counter = (init_ctr + it) mod 2^32 (brownian.py:153, :182). Association order
 * follows numpy: vx -= ((gamma/mass) * vx) * dt; vx += (r*2 - 1) * sqrt(dt);
 * x += vx * dt. Particles are independent, so the step loop is innermost. */
int orc_brownian_steps(int alg, uint64_t n, const uint64_t *pid, double *x, double *y,
                       double *vx, double *vy, uint32_t init_ctr, uint64_t first_it,
                       uint64_t nsteps, double gamma, double mass, double dt) {
    if (alg < 0 || alg > 3) return -1;
    const double gm = gamma / mass;
    const double sqrt_dt = sqrt(dt);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; i++) {
        uint64_t seed = pid ? pid[i] : (uint64_t)i;
        if (alg == ALG_SQUARES) seed &= M32;
        double px = x[i], py = y[i], qx = vx[i], qy = vy[i];
        for (uint64_t s = 0; s < nsteps; s++) {
            uint32_t ctr = (uint32_t)(init_ctr + first_it + s);
            uint32_t w[4];
            qx -= (gm * qx) * dt;
            qy -= (gm * qy) * dt;
            orc_words(alg, seed, ctr, 0, 0, 4, w, NULL);
            double rx = unit_double(w[0], w[1]);
            double ry = unit_double(w[2], w[3]);
            qx += (rx * 2.0 - 1.0) * sqrt_dt;
            qy += (ry * 2.0 - 1.0) * sqrt_dt;
            px += qx * dt;
            py += qy * dt;
        }
        x[i] = px; y[i] = py; vx[i] = qx; vy[i] = qy;
    }
    return 0;
}

/* _kernels.py:89-96 — FNV-1a 64. */
uint64_t orc_fnv1a64(const uint8_t *data, uint64_t n) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (uint64_t i = 0; i < n; i++) h = (h ^ data[i]) * 0x100000001B3ull;
    return h;
}

/* brownian.py:198-223 — FNV over pid-ordered <Qdddd records (little-endian host). */
uint64_t orc_brownian_checksum(uint64_t n, const uint64_t *pid, const double *x, const double *y,
                               const double *vx, const double *vy) {
    uint64_t h = 0xCBF29CE484222325ull;
    for (uint64_t i = 0; i < n; i++) {
        uint64_t rec[5];
        rec[0] = pid ? pid[i] : i;
        memcpy(&rec[1], &x[i], 8); memcpy(&rec[2], &y[i], 8);
        memcpy(&rec[3], &vx[i], 8); memcpy(&rec[4], &vy[i], 8);
        const uint8_t *b = (const uint8_t *)rec;
        for (int k = 0; k < 40; k++) h = (h ^ b[k]) * 0x100000001B3ull;
    }
    return h;
}

/* ------------------------------------------------------------------------- */
/* Full-size checks (tests/test_gpu_fullsize.py). Not reference functions: the
 * order-free position-aware digest sum_i mix64(mix64(i) ^ w_i) mod 2^64 that
 * the GPU side computes (paper_2310_19925_b200/sharding.py), streamed over the
 * reference's outputs without materialising them, and the Box-Muller error of
 * a device array against the reference's formula.                            */

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint32_t f32_bits_of_word(uint32_t w) {
    /* distributions.py:105-107 */
    float f = (float)((double)(w >> 8) * 0x1p-24);
    uint32_t b;
    memcpy(&b, &f, 4);
    return b;
}

/* Digest of words (as_f32 = 0) or of their uniform f32 bit patterns (as_f32 = 1)
 * at stream word positions [word0, word0 + n) of stream (seed, sc) — the values
 * uniform_f32_array / words would return for a generator positioned at word0
 * (bulk.py:223-281; block counter = word0 / 4 for Philox/Threefry, = word0 for
 * Squares, wrapping mod 2^32) — with global index offset `index0`. */
uint64_t orc_digest_stream(int alg, uint64_t seed, uint32_t sc, uint64_t word0, uint64_t n, uint64_t index0,
                           int as_f32) {
    if (alg < 0 || alg > 2) return 0;
    if (alg == ALG_SQUARES) seed &= M32;
    const uint64_t key = orc_squares_key(seed);
    uint64_t acc = 0;
    const int64_t nchunks = (int64_t)((n + 4095) / 4096);
#pragma omp parallel for schedule(static) reduction(+ : acc)
    for (int64_t c = 0; c < nchunks; c++) {
        const uint64_t lo = (uint64_t)c * 4096, k = n - lo < 4096 ? n - lo : 4096;
        uint32_t blk[4];
        uint64_t have = ~0ull;  /* block index held in blk */
        for (uint64_t i = 0; i < k; i++) {
            const uint64_t pos = word0 + lo + i;
            uint32_t w;
            if (alg == ALG_SQUARES) {
                w = orc_squares_round(key, ((uint64_t)sc << 32) | (uint32_t)pos);
            } else {
                if ((pos >> 2) != have) {
                    have = pos >> 2;
                    block_of(alg, seed, sc, (uint32_t)have, blk);
                }
                w = blk[pos & 3];
            }
            if (as_f32) w = f32_bits_of_word(w);
            acc += mix64(mix64(index0 + lo + i) ^ (uint64_t)w);
        }
    }
    return acc;
}

/* Digest of prefix_words(alg, arange(seed_base, seed_base + n_streams), ctr, nwords)
 * (bulk.py:162-207), optionally as uniform f32 bits; index i = stream * nwords + j
 * counted from index0. */
uint64_t orc_digest_prefix(int alg, uint64_t seed_base, uint64_t n_streams, uint32_t ctr, uint32_t nwords,
                           uint64_t index0, int as_f32) {
    if (alg < 0 || alg > 3 || nwords > 4096) return 0;
    uint64_t acc = 0;
#pragma omp parallel for schedule(static) reduction(+ : acc)
    for (int64_t s = 0; s < (int64_t)n_streams; s++) {
        uint32_t row[4096];
        uint64_t seed = seed_base + (uint64_t)s;
        if (alg == ALG_SQUARES) seed &= M32;
        orc_words(alg, seed, ctr, 0, 0, nwords, row, NULL);
        for (uint32_t j = 0; j < nwords; j++) {
            const uint32_t w = as_f32 ? f32_bits_of_word(row[j]) : row[j];
            acc += mix64(mix64(index0 + (uint64_t)s * nwords + j) ^ (uint64_t)w);
        }
    }
    return acc;
}

/* Box-Muller error of device results z0/z1 for pairs [0, n_pairs) of stream
 * (seed, sc) starting at block bc0 (one 4-word block per pair, distributions.py:
 * 72-81, 110-120, libm as the reference's scalar normal2): out[0] = max error in
 * units of ulp(max(|z|, 1)) (the parity tolerance's unit), out[1] = max error in
 * ulps of z itself (z != 0), out[2] = count of values above `tol` units.
 * Philox/Threefry only (the long-stream layout of configs[3]). */
int orc_normal2_error(int alg, uint64_t seed, uint32_t sc, uint32_t bc0, uint64_t n_pairs, const double *z0,
                      const double *z1, double tol, double out[3]) {
    if (alg != ALG_PHILOX && alg != ALG_THREEFRY) return -1;
    const double two_pi = 2.0 * M_PI;
    double m_abs = 0.0, m_rel = 0.0, over = 0.0;
#pragma omp parallel for schedule(static) reduction(max : m_abs, m_rel) reduction(+ : over)
    for (int64_t i = 0; i < (int64_t)n_pairs; i++) {
        uint32_t q[4];
        block_of(alg, seed, sc, (uint32_t)(bc0 + (uint64_t)i), q);
        const uint64_t a = (uint64_t)q[0] | ((uint64_t)q[1] << 32);
        const uint64_t b = (uint64_t)q[2] | ((uint64_t)q[3] << 32);
        const double u1 = 1.0 - (double)(a >> 11) * 0x1p-53;
        const double u2 = (double)(b >> 11) * 0x1p-53;
        const double r = sqrt(-2.0 * log(u1));
        const double t = two_pi * u2;
        const double ref[2] = {r * cos(t), r * sin(t)};
        const double got[2] = {z0[i], z1[i]};
        for (int k = 0; k < 2; k++) {
            const double d = fabs(got[k] - ref[k]);
            const double ua = d / (nextafter(fmax(fabs(ref[k]), 1.0), INFINITY) - fmax(fabs(ref[k]), 1.0));
            if (ua > m_abs) m_abs = ua;
            if (ua > tol) over += 1.0;
            if (ref[k] != 0.0) {
                const double ar = fabs(ref[k]);
                const double ur = d / (nextafter(ar, INFINITY) - ar);
                if (ur > m_rel) m_rel = ur;
            }
        }
    }
    out[0] = m_abs; out[1] = m_rel; out[2] = over;
    return 0;
}
