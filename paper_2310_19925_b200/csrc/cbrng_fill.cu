// cbrng_fill.cu — single-stream bulk fills: Generator.words and the fused
// distribution fills (bulk.py:223-281, distributions.py:99-120).
//
// Layout: one "unit" = 4 consecutive words of the stream (one Philox/Threefry
// block, or 4 Squares counters). Lane l of a warp owns units base + l + 32j
// (j < ILP), so every store instruction of a warp writes one contiguous
// 512-byte run (128-bit st.global.cs per lane) and each thread keeps ILP
// independent cipher evaluations in flight. The grid is the resident grid
// (SMs x CTAs/SM), persistent over the output.
//
// Counter arithmetic: the fill starts at stream word `word_pos`. For Philox/Threefry
// that is block b0 = (word_pos >> 2) mod 2^32 (bulk.py:215-217) at word skip =
// word_pos & 3; unit u is block (b0 + u) when skip == 0, otherwise the last
// 4 - skip words of block b0 + u followed by the first skip words of block
// b0 + u + 1 (a resumed, mid-block generator: 2 cipher calls per unit).
// Squares word k of unit u uses counter (word_pos + 4u + k) mod 2^32 (bulk.py:268).
#include <cstdlib>
#include <type_traits>

#include "cbrng_internal.cuh"
#include "cbrng_bm.cuh"
#include "cbrng_stream.cuh"

namespace cbrng {

enum Out : int { OUT_U32 = 0, OUT_F32 = 1, OUT_F64 = 2, OUT_NORMAL = 3 };

template <int ALG>
struct FillArgs {
    typename StreamOf<ALG>::T p;
    uint32_t bc0;
    uint32_t skip;     // 0..3: words of block bc0 already consumed (Philox/Threefry)
    uint32_t tail;     // trailing output elements after the last full unit
    uint64_t n_units;  // full units
    void *out0;
    void *out1;
    uint32_t m24;      // 1 << 24 at run time (u32_to_f32_mul)
};

// CV: where the f32 map's shift / convert / scale run (u32_to_f32_cv).
// BV: the lane's view of the Box-Muller tables (OUT_NORMAL only).
// CV & 8 (tuning build, CBRNG_NOSTORE=1) or CBRNG_CEILING (the measurement-only
// libcbrng_ceiling.so that bench.py times live): HBM-free ceiling of the same kernel.
// Unit u is stored at u mod 2^16 (a 1-2 MB ring that stays in L2), so the
// instruction stream is the product's plus one LOP3 per store, and no output
// reaches HBM. (A value-dependent store predicate instead splits the unrolled
// tile into branches and serialises it.)
template <int OUT, int CV = 0, class BV = BmView<>>
__device__ __forceinline__ void store_unit(void *out0, void *out1, uint64_t u, uint4 w, uint32_t m24 = 0,
                                           const BV &bm = BV{}) {
    if constexpr ((CV & 8) != 0 || CBRNG_CEILING) u &= 0xFFFFu;
    if constexpr (OUT == OUT_U32) {
        __stcs(reinterpret_cast<uint4 *>(out0) + u, w);
    } else if constexpr (OUT == OUT_F32) {
        __stcs(reinterpret_cast<float4 *>(out0) + u, u32x4_to_f32x4<CV & 7>(w, m24));
    } else if constexpr (OUT == OUT_F64) {
        __stcs(reinterpret_cast<double2 *>(out0) + u, make_double2(u32x2_to_f64(w.x, w.y), u32x2_to_f64(w.z, w.w)));
    } else {
        double z0, z1;
        box_muller_fast(w, z0, z1, bm);
        __stcs(reinterpret_cast<double *>(out0) + u, z0);
        __stcs(reinterpret_cast<double *>(out1) + u, z1);
    }
}

// Partial trailing unit (1-3 words, or 1 double): element-wise stores.
template <int OUT>
__device__ __forceinline__ void store_tail(void *out0, uint64_t u, uint32_t tail, uint4 w) {
    uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    if constexpr (OUT == OUT_U32) {
        for (uint32_t k = 0; k < tail; k++) reinterpret_cast<uint32_t *>(out0)[4 * u + k] = ws[k];
    } else if constexpr (OUT == OUT_F32) {
        for (uint32_t k = 0; k < tail; k++) reinterpret_cast<float *>(out0)[4 * u + k] = u32_to_f32(ws[k]);
    } else if constexpr (OUT == OUT_F64) {
        if (tail) reinterpret_cast<double *>(out0)[2 * u] = u32x2_to_f64(w.x, w.y);
    }
}

// One fill job, warp-strided: warp `warp` of `nwarps` takes tiles warp,
// warp + nwarps, ...; the last warp also writes the remainder and the tail.
// PIPE (Box-Muller): software-pipelined tiles, the cipher blocks of the warp's
// next tile are generated in the same loop body as the current tile's FP64
// transform, so one warp's instruction stream mixes FMA-heavy (IMAD.WIDE) and
// FP64 work instead of alternating between a cipher phase and a transform phase.
template <int ALG, int OUT, int ILP, bool SKIP, int V, int CV, class BV = BmView<>, bool PIPE = false>
__device__ __forceinline__ void fill_job(const FillArgs<ALG> &a, uint64_t warp, uint64_t nwarps, uint32_t lane,
                                         const BV &bmt = BV{}) {
    constexpr uint32_t TILE = 32 * ILP;
    // Full warp tiles: no bounds checks, all ILP cipher evaluations issued
    // before the stores.
    const uint64_t n_full = a.n_units / TILE;
    if constexpr (PIPE) {
        uint4 wn[ILP];
        if (warp < n_full) {
#pragma unroll
            for (int j = 0; j < ILP; j++) wn[j] = unit_words<ALG, SKIP, V>(a.p, a.bc0, a.skip, warp * TILE + lane + 32 * j);
        }
        for (uint64_t t = warp; t < n_full; t += nwarps) {
            uint4 w[ILP];
#pragma unroll
            for (int j = 0; j < ILP; j++) w[j] = wn[j];
            // the next tile (the last iteration recomputes its own: a select, not a branch)
            const uint64_t tn = t + nwarps < n_full ? t + nwarps : t;
#pragma unroll
            for (int j = 0; j < ILP; j++) wn[j] = unit_words<ALG, SKIP, V>(a.p, a.bc0, a.skip, tn * TILE + lane + 32 * j);
#pragma unroll
            for (int j = 0; j < ILP; j++)
                store_unit<OUT, CV, BV>(a.out0, a.out1, t * TILE + lane + 32 * j, w[j], a.m24, bmt);
        }
    }
    for (uint64_t t = PIPE ? n_full : warp; t < n_full; t += nwarps) {
        const uint64_t base = t * TILE + lane;
        uint4 w[ILP];
        if constexpr (ALG == SQUARES && (V == 2 || V == 6)) {
            // no counter wrap, round 1 by finite differences (squares_x4_inc):
            // x and E for the lane's first unit, then +128 counters per j
            // (V 6, tuning: carries forced onto the ALU pipe)
            const uint32_t c0 = a.bc0 + 4u * (uint32_t)base;
            uint64_t x = (uint64_t)c0 * a.p.key + a.p.base;
            uint64_t e = (uint64_t)c0 * a.p.k2x2 + a.p.ebase;
            const uint64_t sx = a.p.key << 7, se = a.p.k2x2 << 7;
#pragma unroll
            for (int j = 0; j < ILP; j++) {
                w[j] = squares_x4_inc<V == 6>(x, e, a.p.key, a.p.k2x2, a.p.k2x4);
                if constexpr (V == 6) {
                    x = add64_alu(x, sx);
                    e = add64_alu(e, se);
                } else {
                    x = add64_opaque(x, sx);
                    e = add64_opaque(e, se);
                }
            }
        } else if constexpr (ALG == SQUARES && V == 1) {
            // no counter wrap anywhere in the fill: unit u's first product
            // x = ctr * key steps by 32 units = 128 counters per j with one
            // 64-bit add (ALU) instead of a 64-bit multiply (FMA-heavy)
            uint64_t x = (uint64_t)(a.bc0 + 4u * (uint32_t)base) * a.p.key + a.p.base;
            const uint64_t step = a.p.key << 7;
#pragma unroll
            for (int j = 0; j < ILP; j++) {
                w[j] = squares_x4(x, a.p.key);
                x = add64_opaque(x, step);
            }
        } else {
#pragma unroll
            for (int j = 0; j < ILP; j++) w[j] = unit_words<ALG, SKIP, V>(a.p, a.bc0, a.skip, base + 32 * j);
        }
#pragma unroll
        for (int j = 0; j < ILP; j++)
            store_unit<OUT, CV, BV>(a.out0, a.out1, base + 32 * j, w[j], a.m24, bmt);
    }
    // Remainder (< one tile) and the partial trailing unit: the last warp of the grid.
    if (warp == nwarps - 1) {
        for (uint64_t u = n_full * TILE + lane; u < a.n_units; u += 32)
            store_unit<OUT, 0, BV>(a.out0, a.out1, u, unit_words<ALG, SKIP, V>(a.p, a.bc0, a.skip, u), 0, bmt);
        if (a.tail && lane == 0)
            store_tail<OUT>(a.out0, a.n_units, a.tail, unit_words<ALG, SKIP, V>(a.p, a.bc0, a.skip, a.n_units));
    }
}

// MB: minimum resident CTAs per SM for the register allocator (0 = unconstrained).
template <int ALG, int OUT, int ILP, bool SKIP, int V, int CV, int MB = 0>
__global__ void __launch_bounds__(256, MB) fill_kernel(const __grid_constant__ FillArgs<ALG> a) {
    static_assert(OUT != OUT_NORMAL, "normal_fill_kernel");
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    fill_job<ALG, OUT, ILP, SKIP, V, CV>(a, warp, nwarps, lane);
}

// Box-Muller fill: NT threads per CTA, LC / SC interleaved copies of the log /
// sincos tables in shared memory (cbrng_bm.cuh), MB CTAs per SM for the
// register allocator.
template <int ALG, int ILP, bool SKIP, int V, int LC, int SC, int NT, int MB, bool PIPE = false, int CV = 0>
__global__ void __launch_bounds__(NT, MB) normal_fill_kernel(const __grid_constant__ FillArgs<ALG> a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const BmView<LC, SC> v = bm_stage_table(reinterpret_cast<BmTables<LC, SC> *>(s_dyn));
    fill_job<ALG, OUT_NORMAL, ILP, SKIP, V, CV, BmView<LC, SC>, PIPE>(a, warp, nwarps, lane, v);
}

// Several counter-based fills in one launch (cbrng_words_multi /
// cbrng_uniform_f32_multi with CBRNG_MULTI=1). The generators bind different
// pipes (Philox: HBM and the FMA-heavy pipe; Threefry: ALU; Squares:
// FMA-heavy), so the kernel interleaves them on every SM: warp w runs its
// share of each job in the order starting at job w mod 3, so about a third of
// the resident warps run each generator at any time. Each warp's total work
// is the same share of every job, so the warps finish together. Jobs with
// n_units == 0 and tail == 0 are absent. Only the default fast paths:
// block-aligned Philox/Threefry (skip 0) and non-wrapping Squares (V 2).
template <int OUT>
struct MultiFillArgs {
    FillArgs<PHILOX> ph;
    FillArgs<THREEFRY> tf;
    FillArgs<SQUARES> sq;
};

constexpr int TF_V_DEFAULT = 4;

template <int OUT, int CV, int IP, int IT, int IS, int MB>
__global__ void __launch_bounds__(256, MB) multi_fill_kernel(const __grid_constant__ MultiFillArgs<OUT> m) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t first = (uint32_t)(warp % 3);
#pragma unroll 1
    for (uint32_t k = 0; k < 3; k++) {
        const uint32_t j = first + k >= 3 ? first + k - 3 : first + k;
        if (j == 0) fill_job<PHILOX, OUT, IP, false, 0, CV>(m.ph, warp, nwarps, lane, nullptr);
        else if (j == 1) fill_job<THREEFRY, OUT, IT, false, TF_V_DEFAULT, CV>(m.tf, warp, nwarps, lane, nullptr);
        else fill_job<SQUARES, OUT, IS, false, 2, CV>(m.sq, warp, nwarps, lane, nullptr);
    }
}

// Tyche is sequential within a stream (generators.py:221-224; _kernels.py:3-5):
// one thread walks the chain. Latency-bound (~12 dependent ALU ops per word).
template <int OUT>
__global__ void tyche_stream_kernel(uint4 s, uint64_t n, void *out0, void *out1, uint32_t *state_out, uint32_t z) {
    __shared__ std::conditional_t<OUT == OUT_NORMAL, BmTables<>, char> s_bm;
    BmView<> bv{};
    if constexpr (OUT == OUT_NORMAL) bv = bm_stage_table(&s_bm);
    uint32_t a = s.x, b = s.y, c = s.z, d = s.w;
    for (uint64_t i = 0; i < n; i++) {
        if constexpr (OUT == OUT_U32) {
            tyche_mix_alu(a, b, c, d, z);
            reinterpret_cast<uint32_t *>(out0)[i] = b;
        } else if constexpr (OUT == OUT_F32) {
            tyche_mix_alu(a, b, c, d, z);
            reinterpret_cast<float *>(out0)[i] = u32_to_f32(b);
        } else if constexpr (OUT == OUT_F64) {
            tyche_mix_alu(a, b, c, d, z);
            uint32_t lo = b;
            tyche_mix_alu(a, b, c, d, z);
            reinterpret_cast<double *>(out0)[i] = u32x2_to_f64(lo, b);
        } else {
            uint4 w;
            tyche_mix_alu(a, b, c, d, z); w.x = b;
            tyche_mix_alu(a, b, c, d, z); w.y = b;
            tyche_mix_alu(a, b, c, d, z); w.z = b;
            tyche_mix_alu(a, b, c, d, z); w.w = b;
            double z0, z1;
            box_muller_fast(w, z0, z1, bv);
            reinterpret_cast<double *>(out0)[i] = z0;
            reinterpret_cast<double *>(out1)[i] = z1;
        }
    }
    if (state_out) {
        state_out[0] = a; state_out[1] = b; state_out[2] = c; state_out[3] = d;
    }
}

// A fresh Tyche stream's first words in one launch (cbrng_scalar op
// TYCHE_SEED_WORDS): out = [state after tyche_init (4), n words, final state (4)].
__global__ void tyche_seed_words_kernel(uint64_t seed, uint32_t sc, uint64_t n, uint32_t *out, uint32_t z) {
    const uint4 s = tyche_init(seed, sc);
    out[0] = s.x; out[1] = s.y; out[2] = s.z; out[3] = s.w;
    uint32_t a = s.x, b = s.y, c = s.z, d = s.w;
    for (uint64_t i = 0; i < n; i++) {
        tyche_mix_alu(a, b, c, d, z);
        out[4 + i] = b;
    }
    out[4 + n] = a; out[5 + n] = b; out[6 + n] = c; out[7 + n] = d;
}

int launch_tyche_seed_words(uint64_t seed, uint32_t sc, uint64_t n, uint32_t *out, cudaStream_t st) {
    tyche_seed_words_kernel<<<1, 1, 0, st>>>(seed, sc, n, out, 0u);
    return check_launch("tyche_seed_words_kernel");
}

// Box-Muller over caller-supplied words (4 per pair): the transform of
// normal2 / normal2_array applied to any word source (the reference tests it
// with scripted generators, test_distributions.py:29-40, 178-186).
__global__ void __launch_bounds__(256) normal2_words_kernel(const uint4 *__restrict__ w, uint64_t n_pairs,
                                                            double *__restrict__ z0, double *__restrict__ z1) {
    __shared__ BmTables<> s_bm;
    const BmView<> bv = bm_stage_table(&s_bm);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pairs;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double a, b;
        box_muller_fast(w[i], a, b, bv);
        z0[i] = a;
        z1[i] = b;
    }
}

constexpr int FILL_BLOCK = 256;

template <int ALG, int OUT, bool SKIP, int ILP, int V, int CV, int MB = 0>
static int launch_fill_ilp(const FillArgs<ALG> &a, cudaStream_t st) {
    auto k = fill_kernel<ALG, OUT, ILP, SKIP, V, CV, MB>;
    if constexpr (TUNING && !SKIP) {
        if (tuning_knob("CBRNG_NOSTORE", 0, 0, 1)) k = fill_kernel<ALG, OUT, ILP, SKIP, V, CV | 8, MB>;
    }
    uint64_t work = (a.n_units + (FILL_BLOCK * ILP) - 1) / (FILL_BLOCK * ILP);
    unsigned grid = grid_for(k, FILL_BLOCK, 0, work ? work : 1);
    k<<<grid, FILL_BLOCK, 0, st>>>(a);
    return check_launch("fill_kernel");
}

// Units per thread per tile (independent cipher chains in flight per thread).
// B200 sweeps: 4 -> 8 lifts Philox 6411 -> 6575 GB/s, Squares 4329 -> 4416,
// Box-Muller 2526 -> 2655 (profiles/r1o_tune.md); 8 -> 16 adds 2 % for the
// Philox word and f32 fills and costs Squares 1.5 % (r1p_tune.md) and, with the
// XU conversion, Threefry 2 % (r1r_tune.md); 12 is 1 % faster than 8 for
// Threefry and Squares (r1t_tune.md); after Squares' finite-difference round 1,
// 16 edges 12 for the Squares f32 fill (4826 vs 4807-4809 GB/s) while 12 stays
// ahead for its u32 words (5302-5304 vs 5180-5181).
// Box-Muller stays at 8: more pairs per thread hide the long FP64 dependency
// chains (ncu r1e at one pair: issue 64 %, "wait" the top stall), 16 spills.
template <int ALG, int OUT>
constexpr int fill_ilp_default() {
    constexpr bool WORDS = OUT == OUT_U32 || OUT == OUT_F32;
    return WORDS ? ((ALG == THREEFRY || (ALG == SQUARES && OUT == OUT_U32)) ? 12 : 16) : 8;
}

// Default code variants (B200 sweeps, profiles/r1r_tune.md): Threefry V (see
// block_at) and the f32 conversion placement CV (see u32_to_f32_cv) per
// generator. Tuning build: CBRNG_FILL_ILP=8|12|16, CBRNG_TF_VARIANT=0..8,
// CBRNG_CVT=0..5, CBRNG_SQ_INC=0..2, CBRNG_SQ_MINB=0|6, CBRNG_MULTI=0|1,
// CBRNG_BM_LAYOUT=0..12, CBRNG_BM_SPLIT=0|1, CBRNG_BM_GRID, CBRNG_NOSTORE=0|1.

// Box-Muller fill shape (normal_fill_kernel): ILP pairs per thread, LC / SC
// table copies, NT threads per CTA, MB CTAs per SM (profiles/r2d_tune.md).
constexpr int BM_ILP = 8, BM_LC = 8, BM_SC = 2, BM_NT = 1024, BM_MB = 2, BM_LAYOUT_DEFAULT = 5;

template <int ALG, bool SKIP, int V, int ILP, int LC, int SC, int NT, int MB, bool PIPE = false>
static int launch_normal(const FillArgs<ALG> &a, cudaStream_t st) {
    auto k = normal_fill_kernel<ALG, ILP, SKIP, V, LC, SC, NT, MB, PIPE>;
    if constexpr (TUNING && !SKIP) {
        if (tuning_knob("CBRNG_NOSTORE", 0, 0, 1)) k = normal_fill_kernel<ALG, ILP, SKIP, V, LC, SC, NT, MB, PIPE, 8>;
    }
    constexpr size_t smem = sizeof(BmTables<LC, SC>);
    // per launch: the attribute is per device and the ABI serves any current device
    if (smem > 48 * 1024) {
        const int rc = check_cuda(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                                  "normal_fill_kernel shared-memory attribute");
        if (rc) return rc;
    }
    // persistent: one resident grid (each CTA stages smem bytes of tables once)
    const uint64_t work = (a.n_units + (NT * ILP) - 1) / (NT * ILP);
    uint64_t g = (uint64_t)resident_blocks(reinterpret_cast<const void *>(k), NT, smem);
    if constexpr (TUNING) g *= (uint64_t)tuning_knob("CBRNG_BM_GRID", 1, 1, 8);
    if (work < g) g = work;
    k<<<(unsigned)(g ? g : 1), NT, smem, st>>>(a);
    return check_launch("normal_fill_kernel");
}

template <int ALG> constexpr int cv_default() { return 4; }  // all three fills: SHF + I2F (XU) + FMUL

// Tuning build: the Box-Muller fill shapes of CBRNG_BM_LAYOUT (profiles/r2d_tune.md).
template <int ALG, bool SKIP, int VS>
static int launch_normal_layout(const FillArgs<ALG> &a, cudaStream_t st, int lay) {
    switch (lay) {
        case 8: return launch_normal<ALG, SKIP, VS, 4, 8, 2, 512, 2, true>(a, st);
        case 9: return launch_normal<ALG, SKIP, VS, 4, 8, 4, 1024, 1, true>(a, st);
        case 10: return launch_normal<ALG, SKIP, VS, 2, 8, 2, 1024, 2, true>(a, st);
        case 11: return launch_normal<ALG, SKIP, VS, 4, 8, 2, 1024, 2, true>(a, st);
        case 12: return launch_normal<ALG, SKIP, VS, 8, 8, 2, 1024, 1>(a, st);
        case 0: return launch_normal<ALG, SKIP, VS, 8, 1, 1, 256, 8>(a, st);
        case 1: return launch_normal<ALG, SKIP, VS, 8, 2, 1, 256, 8>(a, st);
        case 2: return launch_normal<ALG, SKIP, VS, 8, 8, 1, 512, 4>(a, st);
        case 3: return launch_normal<ALG, SKIP, VS, 8, 4, 2, 512, 4>(a, st);
        case 4: return launch_normal<ALG, SKIP, VS, 8, 8, 4, 1024, 2>(a, st);
        case 5: return launch_normal<ALG, SKIP, VS, 8, 8, 2, 1024, 2>(a, st);
        case 6: return launch_normal<ALG, SKIP, VS, 4, 8, 2, 1024, 2>(a, st);
        default: return launch_normal<ALG, SKIP, VS, 8, 8, 1, 256, 0>(a, st);
    }
}

template <int ALG, int OUT, bool SKIP, int V, int CV>
static int launch_fill_v(const FillArgs<ALG> &a, cudaStream_t st) {
    if constexpr (SKIP && OUT == OUT_NORMAL) {
        return launch_normal<ALG, SKIP, V, 2, 1, 1, 256, 0>(a, st);  // resumed mid-block: rare, 2 blocks per unit
    } else if constexpr (SKIP) {
        return launch_fill_ilp<ALG, OUT, SKIP, 2, V, CV>(a, st);  // resumed mid-block: rare, 2 blocks per unit
    } else if constexpr (OUT == OUT_U32 || OUT == OUT_F32) {
        constexpr int I0 = fill_ilp_default<ALG, OUT>();
        if constexpr (TUNING && ALG == SQUARES) {
            // register cap: 6 CTAs/SM (<= 40 registers) instead of 5 at 48
            static const int mb = tuning_knob("CBRNG_SQ_MINB", 0, 0, 8);
            if (mb == 6) {
                static const int ilp = tuning_knob("CBRNG_FILL_ILP", I0, 8, 16);
                if (ilp == 12) return launch_fill_ilp<ALG, OUT, SKIP, 12, V, CV, 6>(a, st);
                return launch_fill_ilp<ALG, OUT, SKIP, 16, V, CV, 6>(a, st);
            }
        }
        if constexpr (TUNING) {
            static const int ilp = tuning_knob("CBRNG_FILL_ILP", I0, 8, 16);
            if (ilp == 16) return launch_fill_ilp<ALG, OUT, SKIP, 16, V, CV>(a, st);
            if (ilp == 12) return launch_fill_ilp<ALG, OUT, SKIP, 12, V, CV>(a, st);
            return launch_fill_ilp<ALG, OUT, SKIP, 8, V, CV>(a, st);
        }
        return launch_fill_ilp<ALG, OUT, SKIP, I0, V, CV>(a, st);
    } else if constexpr (OUT == OUT_NORMAL) {
        if constexpr (TUNING && ALG == PHILOX && !SKIP) {
            // CBRNG_BM_SPLIT=1: Philox mulhilo as IMAD.HI + IMAD (V 1), measured 10 % slower (profiles/r2d_tune.md)
            // 2..5: only some rounds split (round bit masks 0x2AA, 0x154, 0x3F0, 0x00E)
            static const int split = tuning_knob("CBRNG_BM_SPLIT", 0, 0, 5);
            static const int lay = tuning_knob("CBRNG_BM_LAYOUT", BM_LAYOUT_DEFAULT, 0, 12);
            switch (split) {
                case 1: return launch_normal_layout<ALG, SKIP, 1>(a, st, lay);
                case 2: return launch_normal<ALG, SKIP, 0x2AA, BM_ILP, BM_LC, BM_SC, BM_NT, BM_MB>(a, st);
                case 3: return launch_normal<ALG, SKIP, 0x154, BM_ILP, BM_LC, BM_SC, BM_NT, BM_MB>(a, st);
                case 4: return launch_normal<ALG, SKIP, 0x3F0, BM_ILP, BM_LC, BM_SC, BM_NT, BM_MB>(a, st);
                case 5: return launch_normal<ALG, SKIP, 0x00E, BM_ILP, BM_LC, BM_SC, BM_NT, BM_MB>(a, st);
                default: return launch_normal_layout<ALG, SKIP, V>(a, st, lay);
            }
        } else if constexpr (ALG != PHILOX) {
            return launch_normal<ALG, SKIP, V, 4, 8, 2, 512, 0>(a, st);  // wider cipher state
        } else {
            return launch_normal<ALG, SKIP, V, BM_ILP, BM_LC, BM_SC, BM_NT, BM_MB>(a, st);
        }
    } else {
        return launch_fill_ilp<ALG, OUT, SKIP, 8, V, CV>(a, st);
    }
}

// Tuning dispatch: either the code variant V or the conversion CV departs from
// its default (never both), which keeps the instantiation count linear.
template <int ALG, int OUT, bool SKIP, int V0>
static int launch_fill_cv(const FillArgs<ALG> &a, cudaStream_t st) {
    constexpr int C0 = cv_default<ALG>();
    if constexpr (TUNING && OUT == OUT_F32 && !SKIP) {
        static const int cv = tuning_knob("CBRNG_CVT", C0, 0, 5);
        switch (cv) {
            case 0: return launch_fill_v<ALG, OUT, SKIP, V0, 0>(a, st);
            case 1: return launch_fill_v<ALG, OUT, SKIP, V0, 1>(a, st);
            case 2: return launch_fill_v<ALG, OUT, SKIP, V0, 2>(a, st);
            case 3: return launch_fill_v<ALG, OUT, SKIP, V0, 3>(a, st);
            case 4: return launch_fill_v<ALG, OUT, SKIP, V0, 4>(a, st);
            default: return launch_fill_v<ALG, OUT, SKIP, V0, 5>(a, st);
        }
    }
    return launch_fill_v<ALG, OUT, SKIP, V0, C0>(a, st);
}

template <int ALG, int OUT, bool SKIP>
static int launch_fill_k(const FillArgs<ALG> &a, cudaStream_t st) {
    constexpr int C0 = cv_default<ALG>();
    if constexpr (ALG == SQUARES) {
        // counters bc0 .. bc0 + 4*(n_units+1) - 1 never wrap: drop the per-unit check
        if ((uint64_t)a.bc0 + 4ull * (a.n_units + 1) <= (1ull << 32)) {
            // V 2: round 1 by finite differences (tuning: CBRNG_SQ_INC=0 -> V 1)
            if constexpr (TUNING) {
                // CBRNG_SQ_INC: 0 -> V 1 (no finite differences), 2 -> V 6 (ALU-forced carries)
                static const int inc = tuning_knob("CBRNG_SQ_INC", 1, 0, 2);
                if (inc == 0) return launch_fill_cv<ALG, OUT, SKIP, 1>(a, st);
                if (inc == 2) return launch_fill_cv<ALG, OUT, SKIP, 6>(a, st);
            }
            return launch_fill_cv<ALG, OUT, SKIP, 2>(a, st);
        }
        return launch_fill_v<ALG, OUT, SKIP, 0, C0>(a, st);  // the fill crosses the counter wrap
    } else if constexpr (ALG == THREEFRY) {
        if constexpr (TUNING && (OUT == OUT_U32 || OUT == OUT_F32) && !SKIP) {
            static const int tfv = tuning_knob("CBRNG_TF_VARIANT", TF_V_DEFAULT, 0, 8);
            switch (tfv) {
                case 0: return launch_fill_v<ALG, OUT, SKIP, 0, C0>(a, st);
                case 1: return launch_fill_v<ALG, OUT, SKIP, 1, C0>(a, st);
                case 2: return launch_fill_v<ALG, OUT, SKIP, 2, C0>(a, st);
                case 3: return launch_fill_v<ALG, OUT, SKIP, 3, C0>(a, st);
                case 5: return launch_fill_v<ALG, OUT, SKIP, 5, C0>(a, st);
                case 6: return launch_fill_v<ALG, OUT, SKIP, 6, C0>(a, st);
                case 7: return launch_fill_v<ALG, OUT, SKIP, 7, C0>(a, st);
                case 8: return launch_fill_v<ALG, OUT, SKIP, 8, C0>(a, st);
                default: break;
            }
        }
        return launch_fill_cv<ALG, OUT, SKIP, TF_V_DEFAULT>(a, st);
    } else {
        return launch_fill_cv<ALG, OUT, SKIP, 0>(a, st);
    }
}

template <int ALG>
static FillArgs<ALG> make_fill_args(uint64_t seed, uint32_t sc, uint64_t word_pos, uint64_t n_units, uint32_t tail,
                                    void *out0, void *out1) {
    FillArgs<ALG> a;
    if constexpr (ALG == PHILOX) a.p = philox_stream_setup(seed, sc);
    else if constexpr (ALG == THREEFRY) a.p = threefry_stream_setup(seed, sc);
    else a.p = squares_stream_setup(seed, sc);
    if constexpr (ALG == SQUARES) {
        a.bc0 = (uint32_t)word_pos;
        a.skip = 0;
    } else {
        a.bc0 = (uint32_t)(word_pos >> 2);
        a.skip = (uint32_t)(word_pos & 3);
    }
    a.tail = tail;
    a.n_units = n_units;
    a.out0 = out0;
    a.out1 = out1;
    a.m24 = 1u << 24;
    return a;
}

template <int ALG, int OUT>
static int launch_fill(uint64_t seed, uint32_t sc, uint64_t word_pos, uint64_t n_units, uint32_t tail, void *out0,
                       void *out1, cudaStream_t st) {
    if (n_units == 0 && tail == 0) return CBRNG_OK;
    const FillArgs<ALG> a = make_fill_args<ALG>(seed, sc, word_pos, n_units, tail, out0, out1);
    if constexpr (ALG != SQUARES) {
        if (a.skip) return launch_fill_k<ALG, OUT, true>(a, st);  // resumed mid-block
    }
    return launch_fill_k<ALG, OUT, false>(a, st);
}

template <int OUT>
static int dispatch_fill(int alg, uint64_t seed, uint32_t sc, uint64_t word_pos, const uint32_t *tyche_state,
                         uint64_t n_elems, void *out0, void *out1, uint32_t *tyche_state_out, void *stream) {
    CBRNG_CHECK_ALG(alg);
    clear_error();
    cudaStream_t st = as_stream(stream);
    if (alg == TYCHE) {
        CBRNG_REQUIRE(tyche_state != nullptr, "tyche fills need the serial state (tyche_state)");
        uint4 s = make_uint4(tyche_state[0], tyche_state[1], tyche_state[2], tyche_state[3]);
        if (n_elems == 0 && tyche_state_out == nullptr) return CBRNG_OK;
        tyche_stream_kernel<OUT><<<1, 1, 0, st>>>(s, n_elems, out0, out1, tyche_state_out, 0u);
        return check_launch("tyche_stream_kernel");
    }
    if (alg == SQUARES) seed &= 0xFFFFFFFFull;  // generators.py:256-257
    // elements per 4-word unit: u32/f32 4, f64 2, normal pairs 1
    const uint64_t per = (OUT == OUT_U32 || OUT == OUT_F32) ? 4 : (OUT == OUT_F64 ? 2 : 1);
    const size_t align = (OUT == OUT_NORMAL) ? 8 : 16;
    if (n_elems >= per) {
        if (!aligned(out0, align) || (out1 && !aligned(out1, align))) {
            set_error("output pointer not %zu-byte aligned", align);
            return CBRNG_EALIGN;
        }
    }
    uint64_t n_units = n_elems / per;
    uint32_t tail = (uint32_t)(n_elems % per);
    switch (alg) {
        case PHILOX: return launch_fill<PHILOX, OUT>(seed, sc, word_pos, n_units, tail, out0, out1, st);
        case THREEFRY: return launch_fill<THREEFRY, OUT>(seed, sc, word_pos, n_units, tail, out0, out1, st);
        default: return launch_fill<SQUARES, OUT>(seed, sc, word_pos, n_units, tail, out0, out1, st);
    }
}

// Fused launch of up to one Philox, one Threefry and one Squares job
// (multi_fill_kernel), opt-in with CBRNG_MULTI=1. Measured on B200 it does not
// beat back-to-back launches (2.77 vs 2.74 ms for the three 2^30 f32 fills of
// configs[1], profiles/r1t_tune.md): every generator already keeps both
// integer pipes busy and the SM's issue rate binds the mix.
template <int OUT, int IP, int IT, int IS, int MB>
static int launch_multi_k(const MultiFillArgs<OUT> &m, cudaStream_t st) {
    constexpr int CV = cv_default<PHILOX>();
    auto k = multi_fill_kernel<OUT, CV, IP, IT, IS, MB>;
    const uint64_t units = m.ph.n_units + m.tf.n_units + m.sq.n_units;
    const uint64_t work = (units + (FILL_BLOCK * IT) - 1) / (FILL_BLOCK * IT);
    k<<<grid_for(k, FILL_BLOCK, 0, work ? work : 1), FILL_BLOCK, 0, st>>>(m);
    return check_launch("multi_fill_kernel");
}

// Units per thread per tile in the fused kernel: Philox 8, Threefry 4, Squares
// 8. The standalone ILPs (16/12/12) make the three hot loops 55 KB of code that
// run at once and thrash the instruction cache (3.35 ms vs 2.77, r1t_tune).
template <int OUT>
static int launch_multi(const MultiFillArgs<OUT> &m, cudaStream_t st) {
    return launch_multi_k<OUT, 8, 4, 8, 0>(m, st);
}

struct MultiJob {
    int alg;
    uint64_t seed;
    uint32_t sc;
    uint64_t word_pos, n;
    void *out;
};

// Jobs are taken in order; a job joins the pending fused batch when it is on
// the fast path (block-aligned Philox/Threefry, non-wrapping Squares) and its
// generator's slot is free, otherwise the batch is flushed first. Off-path jobs
// launch on their own (dispatch_fill). Results equal the per-job calls.
template <int OUT>
static int dispatch_multi(int n_jobs, const int *algs, const uint64_t *seeds, const uint32_t *ctrs,
                          const uint64_t *word_pos, const uint64_t *n, void *const *outs, void *stream) {
    clear_error();
    CBRNG_REQUIRE(n_jobs >= 0, "n_jobs < 0");
    if (n_jobs == 0) return CBRNG_OK;
    CBRNG_REQUIRE(algs && seeds && word_pos && n && outs, "NULL job array");
    for (int i = 0; i < n_jobs; i++) {
        CBRNG_CHECK_ALG(algs[i]);
        CBRNG_REQUIRE(algs[i] != TYCHE, "job %d: tyche is serial within a stream; use the per-stream fill", i);
        if (n[i] >= 4 && !aligned(outs[i], 16)) {
            set_error("job %d: output pointer not 16-byte aligned", i);
            return CBRNG_EALIGN;
        }
    }
    cudaStream_t st = as_stream(stream);
    // the fused multi-generator kernel measured no faster (tuning build only)
    static const bool fused = TUNING && tuning_knob("CBRNG_MULTI", 0, 0, 1) == 1;
    MultiFillArgs<OUT> m{};
    int pending = 0;  // bit per generator slot
    MultiJob single[3];
    auto flush = [&]() -> int {
        int rc = CBRNG_OK;
        if (__builtin_popcount(pending) >= 2) {
            if constexpr (TUNING) rc = launch_multi<OUT>(m, st);
        } else {
            for (int g = 0; g < 3 && rc == CBRNG_OK; g++)
                if (pending & (1 << g))
                    rc = dispatch_fill<OUT>(g, single[g].seed, single[g].sc, single[g].word_pos, nullptr, single[g].n,
                                            single[g].out, nullptr, nullptr, stream);
        }
        m = MultiFillArgs<OUT>{};
        pending = 0;
        return rc;
    };
    for (int i = 0; i < n_jobs; i++) {
        const int g = algs[i];
        const uint64_t seed = g == SQUARES ? (seeds[i] & 0xFFFFFFFFull) : seeds[i];  // generators.py:256-257
        const uint32_t sc = ctrs ? ctrs[i] : 0u;
        const uint64_t units = n[i] / 4;
        const uint32_t tail = (uint32_t)(n[i] % 4);
        const bool fast = fused && (units > 0) &&
                          (g == SQUARES ? (uint64_t)(uint32_t)word_pos[i] + 4ull * (units + 1) <= (1ull << 32)
                                        : (word_pos[i] & 3) == 0);
        if (!fast) {
            const int rc = dispatch_fill<OUT>(g, seed, sc, word_pos[i], nullptr, n[i], outs[i], nullptr, nullptr, stream);
            if (rc != CBRNG_OK) return rc;
            continue;
        }
        if (pending & (1 << g)) {
            const int rc = flush();
            if (rc != CBRNG_OK) return rc;
        }
        pending |= 1 << g;
        single[g] = MultiJob{g, seed, sc, word_pos[i], n[i], outs[i]};
        if (g == PHILOX) m.ph = make_fill_args<PHILOX>(seed, sc, word_pos[i], units, tail, outs[i], nullptr);
        else if (g == THREEFRY) m.tf = make_fill_args<THREEFRY>(seed, sc, word_pos[i], units, tail, outs[i], nullptr);
        else m.sq = make_fill_args<SQUARES>(seed, sc, word_pos[i], units, tail, outs[i], nullptr);
    }
    return flush();
}

}  // namespace cbrng

using namespace cbrng;

extern "C" {

int cbrng_words(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos, const uint32_t *tyche_state,
                uint64_t n, uint32_t *out, uint32_t *tyche_state_out, void *stream) {
    const DeviceGuard device_guard(stream);
    return dispatch_fill<OUT_U32>(alg, seed, stream_ctr, word_pos, tyche_state, n, out, nullptr, tyche_state_out,
                                  stream);
}

int cbrng_uniform_f32(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos, const uint32_t *tyche_state,
                      uint64_t n, float *out, uint32_t *tyche_state_out, void *stream) {
    const DeviceGuard device_guard(stream);
    return dispatch_fill<OUT_F32>(alg, seed, stream_ctr, word_pos, tyche_state, n, out, nullptr, tyche_state_out,
                                  stream);
}

int cbrng_uniform_f64(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos, const uint32_t *tyche_state,
                      uint64_t n, double *out, uint32_t *tyche_state_out, void *stream) {
    const DeviceGuard device_guard(stream);
    return dispatch_fill<OUT_F64>(alg, seed, stream_ctr, word_pos, tyche_state, n, out, nullptr, tyche_state_out,
                                  stream);
}

int cbrng_normal2_f64(int alg, uint64_t seed, uint32_t stream_ctr, uint64_t word_pos, const uint32_t *tyche_state,
                      uint64_t n_pairs, double *z0, double *z1, uint32_t *tyche_state_out, void *stream) {
    const DeviceGuard device_guard(stream);
    return dispatch_fill<OUT_NORMAL>(alg, seed, stream_ctr, word_pos, tyche_state, n_pairs, z0, z1,
                                     tyche_state_out, stream);
}

int cbrng_words_multi(int n_jobs, const int *algs, const uint64_t *seeds, const uint32_t *stream_ctrs,
                      const uint64_t *word_pos, const uint64_t *n, uint32_t *const *outs, void *stream) {
    const DeviceGuard device_guard(stream);
    return dispatch_multi<OUT_U32>(n_jobs, algs, seeds, stream_ctrs, word_pos, n,
                                   reinterpret_cast<void *const *>(outs), stream);
}

int cbrng_uniform_f32_multi(int n_jobs, const int *algs, const uint64_t *seeds, const uint32_t *stream_ctrs,
                            const uint64_t *word_pos, const uint64_t *n, float *const *outs, void *stream) {
    const DeviceGuard device_guard(stream);
    return dispatch_multi<OUT_F32>(n_jobs, algs, seeds, stream_ctrs, word_pos, n,
                                   reinterpret_cast<void *const *>(outs), stream);
}

int cbrng_normal2_from_words(const uint32_t *words, uint64_t n_pairs, double *z0, double *z1, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    if (n_pairs == 0) return CBRNG_OK;
    CBRNG_REQUIRE(words && z0 && z1, "NULL pointer");
    if (!aligned(words, 16)) {
        set_error("words pointer not 16-byte aligned");
        return CBRNG_EALIGN;
    }
    cudaStream_t st = as_stream(stream);
    normal2_words_kernel<<<grid_for(normal2_words_kernel, 256, 0, (n_pairs + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const uint4 *>(words), n_pairs, z0, z1);
    return check_launch("normal2_words_kernel");
}

int cbrng_tyche_fill(uint64_t *state, uint64_t n, uint32_t *out, void *stream) {
    const DeviceGuard device_guard(stream);
    CBRNG_REQUIRE(state != nullptr, "state is NULL");
    uint32_t s[4] = {(uint32_t)state[0], (uint32_t)state[1], (uint32_t)state[2], (uint32_t)state[3]};
    uint32_t *dev_state = nullptr;
    cudaStream_t st = as_stream(stream);
    int rc = check_cuda(cudaMallocAsync(&dev_state, 16, st), "cudaMallocAsync");
    if (rc) return rc;
    rc = cbrng_words(TYCHE, 0, 0, 0, s, n, out, dev_state, stream);
    uint32_t back[4] = {s[0], s[1], s[2], s[3]};
    if (rc == 0) rc = check_cuda(cudaMemcpyAsync(back, dev_state, 16, cudaMemcpyDeviceToHost, st), "copy state");
    cudaFreeAsync(dev_state, st);
    if (rc == 0) rc = check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize");
    if (rc == 0)
        for (int i = 0; i < 4; i++) state[i] = back[i];
    return rc;
}

}  // extern "C"
