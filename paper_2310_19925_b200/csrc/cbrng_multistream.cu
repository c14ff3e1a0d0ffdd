// cbrng_multistream.cu — many streams at once: bulk.prefix_words (bulk.py:162-207),
// _kernels.philox_block_lanes (_kernels.py:54-86) and the vector block functions
// (bulk.py:49-159).
//
// Output is row-major out[stream][word] exactly as the reference returns it.
//   * rows of >= 16 words (and every Tyche row: serial within a stream,
//     bulk.py:9-11): one thread per stream walks its row with the stream-only
//     cipher setup folded once per row; a warp transposes its 32 streams x 16
//     words through swizzled shared memory, so each store instruction writes
//     8 rows x 64 contiguous bytes (staged_prefix_kernel);
//   * shorter rows: lanes map to contiguous 16-byte chunks of consecutive rows
//     (prefix_kernel).
#include <cstdlib>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "cbrng_internal.cuh"
#include "cbrng_stream.cuh"

namespace cbrng {

struct PrefixArgs {
    const uint64_t *seeds;
    uint64_t seed_base;
    const uint32_t *ctrs;
    uint32_t ctr_scalar;
    uint32_t nwords;
    uint64_t n_streams;
    void *out;
    uint32_t m24;  // 1 << 24 at run time (u32_to_f32_mul)
};

__device__ __forceinline__ uint64_t seed_of(const PrefixArgs &a, uint64_t i) {
    return a.seeds ? a.seeds[i] : a.seed_base + i;
}
__device__ __forceinline__ uint32_t ctr_of(const PrefixArgs &a, uint64_t i) {
    return a.ctrs ? a.ctrs[i] : a.ctr_scalar;
}

// Per-stream key material for the counter-based algorithms.
template <int ALG> struct StreamKey;
template <> struct StreamKey<PHILOX> {
    uint32_t k0, k1, sc;
    __device__ __forceinline__ StreamKey(uint64_t seed, uint32_t c) : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)), sc(c) {}
    __device__ __forceinline__ uint4 block(uint32_t b) const { return philox_block(make_uint4(sc, b, 0, 0), k0, k1); }
};
template <> struct StreamKey<THREEFRY> {
    uint32_t k0, k1, sc;
    __device__ __forceinline__ StreamKey(uint64_t seed, uint32_t c) : k0((uint32_t)seed), k1((uint32_t)(seed >> 32)), sc(c) {}
    __device__ __forceinline__ uint4 block(uint32_t b) const { return threefry_block(make_uint4(b, 0, 0, 0), k0, k1, sc, 0); }
};
template <> struct StreamKey<SQUARES> {
    SquaresStream p;
    __device__ __forceinline__ StreamKey(uint64_t seed, uint32_t c) {
        p.key = squares_key(seed);
        p.base = ((uint64_t)c << 32) * p.key;
    }
    __device__ __forceinline__ uint32_t word(uint32_t j) const { return squares_stream_word(p, j); }
    __device__ __forceinline__ uint4 block(uint32_t b) const { return squares_stream_word4(p, 4 * b); }
};

template <int ALG>
__device__ __forceinline__ uint32_t single_word(const StreamKey<ALG> &k, uint32_t j) {
    if constexpr (ALG == SQUARES) {
        return k.word(j);
    } else {
        uint4 b = k.block(j >> 2);
        uint32_t r = b.x;
        r = ((j & 3) == 1) ? b.y : r;
        r = ((j & 3) == 2) ? b.z : r;
        r = ((j & 3) == 3) ? b.w : r;
        return r;
    }
}

// OUT: 0 = u32 words, 1 = uniform f32 (conversion placement CV, u32_to_f32_cv).
template <int OUT, int CV = 0>
__device__ __forceinline__ void store4(void *out, uint64_t word_index, uint4 w, uint32_t m24 = 0) {
    if constexpr (OUT == 0) {
        __stcs(reinterpret_cast<uint4 *>(reinterpret_cast<uint32_t *>(out) + word_index), w);
    } else {
        __stcs(reinterpret_cast<float4 *>(reinterpret_cast<float *>(out) + word_index), u32x4_to_f32x4<CV>(w, m24));
    }
}
template <int OUT>
__device__ __forceinline__ void store1(void *out, uint64_t word_index, uint32_t w) {
    if constexpr (OUT == 0) reinterpret_cast<uint32_t *>(out)[word_index] = w;
    else reinterpret_cast<float *>(out)[word_index] = u32_to_f32(w);
}

// Short rows (< 16 words: Brownian init's 8, first_words' 1, ...): a warp covers
// floor(32 / chunks_per_row) whole rows per pass, lane -> (row, chunk), so the
// warp's stores are one contiguous run. CW = words per chunk: 4 (nwords % 4 == 0,
// 16-byte stores) or 1 (generic). Longer rows take staged_prefix_kernel.
template <int ALG, int OUT, int CW>
__global__ void __launch_bounds__(256) prefix_kernel(const __grid_constant__ PrefixArgs a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t cpr = a.nwords / CW;  // chunks per row, < 32 here
    const uint32_t rpp = 32 / cpr;       // rows per pass
    const uint32_t roff = lane / cpr, ch = lane - roff * cpr;
    if (roff >= rpp) return;
    for (uint64_t r0 = warp * rpp; r0 < a.n_streams; r0 += nwarps * rpp) {
        const uint64_t row = r0 + roff;
        if (row >= a.n_streams) break;
        const StreamKey<ALG> k(seed_of(a, row), ctr_of(a, row));
        if constexpr (CW == 4) store4<OUT>(a.out, row * a.nwords + 4ull * ch, k.block(ch));
        else store1<OUT>(a.out, row * a.nwords + ch, single_word<ALG>(k, ch));
    }
}

constexpr int TY_WARPS = 8;  // 256 threads

// One stream walked word by word by one thread (the staged kernel below).
// Counter-based algorithms fold the stream-only rounds once per row
// (philox/threefry_stream_setup), so a 256-word row pays the setup once instead
// of once per 4-word block; Tyche is serial anyway.
template <int ALG> struct RowGen;
template <> struct RowGen<PHILOX> {
    PhiloxStream p;
    uint32_t b = 0;
    __device__ __forceinline__ RowGen(uint64_t seed, uint32_t c) : p(philox_stream_setup(seed, c)) {}
    __device__ __forceinline__ uint4 next4() { return philox_stream_block(p, b++); }
};
template <> struct RowGen<THREEFRY> {
    ThreefryStream p;
    uint32_t b = 0;
    // p.one from the constant bank: set up on the device, a literal 1 would let
    // ptxas fold the forced IMAD adds back into IADD3s on the ALU pipe, the pipe
    // that bounds Threefry
    __device__ __forceinline__ RowGen(uint64_t seed, uint32_t c) : p(threefry_stream_setup(seed, c)) { p.one = c_one; }
    __device__ __forceinline__ uint4 next4() { return threefry_stream_block<0, true, true>(p, b++); }
};
template <> struct RowGen<SQUARES> {
    // x = ctr * key and E = 2 key x + key^2 + key for the row's next counter,
    // stepped by 4 counters per call (64-bit adds; rows never wrap the 32-bit
    // counter); round 1 of the 4 words by finite differences (squares_x4_inc)
    uint64_t key, k2x2, k2x4, x, e;
    __device__ __forceinline__ RowGen(uint64_t seed, uint32_t c) {
        key = squares_key(seed);
        const uint64_t k2 = key * key;
        k2x2 = 2 * k2;
        k2x4 = 4 * k2;
        x = ((uint64_t)c << 32) * key;
        e = (((uint64_t)c << 33) + 1) * k2 + key;
    }
    __device__ __forceinline__ uint4 next4() {
        const uint4 w = squares_x4_inc(x, e, key, k2x2, k2x4, &x);  // x <- x_4, the next call's x_0
        e = add64_opaque(e, k2x4 << 1);                               // E_4 = E_0 + 8 key^2
        return w;
    }
};
template <> struct RowGen<TYCHE> {
    uint32_t A, B, C, D;
    __device__ __forceinline__ RowGen(uint64_t seed, uint32_t c) {
        const uint4 s = tyche_init(seed, c);
        A = s.x; B = s.y; C = s.z; D = s.w;
    }
    __device__ __forceinline__ uint4 next4() {
        uint4 w;
        tyche_mix(A, B, C, D); w.x = B;
        tyche_mix(A, B, C, D); w.y = B;
        tyche_mix(A, B, C, D); w.z = B;
        tyche_mix(A, B, C, D); w.w = B;
        return w;
    }
};


// One thread per stream; a warp transposes its 32 streams x 16 words through
// shared memory so each global store instruction writes 8 rows x 64 B.
// VEC: rows are 16-byte aligned (nwords % 4 == 0) -> 128-bit stores. CV: the
// f32 conversion placement (u32_to_f32_cv). Compile-time so the copy-out is
// branch-free.
// Occupancy: Tyche's row state is 4 registers (32-register cap, 8 CTAs/SM).
// Philox / Threefry keep the folded stream setup live and run best uncapped
// (86 registers, 2 CTAs/SM: the 4 staged blocks' rounds interleave; Philox rows
// +7.5 % over the 64-register cap, profiles/r1t_tune.md); Squares 5 CTAs/SM.
// (Squares: 3 CTAs/SM = 80 registers, which the 8 registers of finite-difference
// row state need without spilling; Threefry: 4 CTAs/SM, 64 registers, +0.5 % on
// u32 rows over uncapped; profiles/r1t_tune.md)
template <int ALG, bool VEC = true> constexpr int staged_min_blocks() {
    return ALG == TYCHE ? 8 : (ALG == SQUARES ? 3 : (ALG == THREEFRY ? 4 : 2));
}

// CH: 16-byte chunks staged per row per round: 4 (64 B of each row per store
// instruction, 8 rows; 16 KB/CTA) or 8 (full 128 B lines, 4 rows; 32 KB/CTA).
// NW: the row length when known at compile time (256: configs[1]'s Tyche rows
// and configs[4]); a full warp's copy-out then stores through one pointer with
// immediate row offsets and no per-row predicates.
template <int ALG, int OUT, bool VEC, int CV, int CH = 4, int NW = 0>
__global__ void __launch_bounds__(256, staged_min_blocks<ALG, VEC>()) staged_prefix_kernel(const __grid_constant__ PrefixArgs a) {
    static_assert(CH == 4 || CH == 8, "CH");
    constexpr uint32_t RPI = 32 / CH;  // rows per copy-out instruction
    __shared__ uint4 tile[TY_WARPS][32 * CH];
    // Tyche u32 rows of NW words: a second staging buffer, so the copy-out of
    // group g - 1 interleaves with the generation of group g (without the f32
    // conversion between them the staging's LDS/STG bursts fill the MIO queue)
    constexpr bool DB = ALG == TYCHE && OUT == 0 && NW != 0 && VEC && CH == 4;
    __shared__ std::conditional_t<DB, uint4[TY_WARPS][32 * 4], uint4[1][1]> tile2;
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t groups = a.nwords / (4 * CH), rem = a.nwords % (4 * CH);
    uint4 *const my = tile[wib];
    // Staging slots (XOR swizzle, conflict-free STS.128 row-wise and LDS.128
    // column-wise): lane writes row `lane`, chunk c at lane*CH + (c ^ wx); for
    // the copy-out, lane reads row r = RPI*k + rrow, chunk rc. CH = 4: swizzle
    // (r >> 1) & 3, independent of k; CH = 8: swizzle r & 7 = rrow ^ 4(k & 1).
    const uint32_t wx = CH == 4 ? (lane >> 1) & 3 : lane & 7;
    const uint32_t rrow = lane / CH, rc = lane % CH;
    const uint32_t rslot = CH == 4 ? rrow * CH + (rc ^ ((lane >> 3) & 3)) : rrow * CH + (rc ^ rrow);
    for (uint64_t s0 = warp * 32; s0 < a.n_streams; s0 += nwarps * 32) {
        const uint64_t sid = s0 + lane;
        const bool valid = sid < a.n_streams;
        RowGen<ALG> gen(valid ? seed_of(a, sid) : 0, valid ? ctr_of(a, sid) : 0);
        // output word index of (row rrow + RPI k, chunk rc) in group g: at + k*rstride
        // (CBRNG_CEILING: rows of 2048-stream blocks overwrite one L2-resident ring)
        uint64_t at = ((CBRNG_CEILING ? (s0 & 2047u) : s0) + rrow) * a.nwords + rc * 4;
        const uint64_t rstride = (uint64_t)RPI * a.nwords;
        const uint32_t rows_left = a.n_streams - s0 < 32 ? (uint32_t)(a.n_streams - s0) : 32u;
        if constexpr (NW != 0 && VEC && CH == 4) {
            if (rows_left == 32) {
                // full warp, compile-time row length: rows rrow + 8k sit at
                // immediate offsets k * 8 * NW words from one pointer
                using V4 = typename std::conditional<OUT == 0, uint4, float4>::type;
                V4 *ptr = reinterpret_cast<V4 *>(a.out) + at / 4;
                if constexpr (DB) {
                    uint4 *const b1 = tile2[wib];
#pragma unroll
                    for (int c = 0; c < 4; c++) my[lane * 4 + (c ^ wx)] = gen.next4();
                    __syncwarp();
                    // ptr: the group being copied out (g - 1)
                    for (uint32_t g = 1; g < (uint32_t)NW / 16; g++, ptr += 4) {
                        uint4 *const cur = (g & 1) ? b1 : my;
                        const uint4 *const prev = (g & 1) ? my : b1;
#pragma unroll
                        for (int c = 0; c < 4; c++) {
                            cur[lane * 4 + (c ^ wx)] = gen.next4();
                            __stcs(reinterpret_cast<uint4 *>(ptr) + c * 2 * NW, prev[rslot + 32 * c]);
                        }
                        __syncwarp();
                    }
                    const uint4 *const last = ((NW / 16 - 1) & 1) ? b1 : my;
#pragma unroll
                    for (int k = 0; k < 4; k++) __stcs(reinterpret_cast<uint4 *>(ptr) + k * 2 * NW, last[rslot + 32 * k]);
                    __syncwarp();
                } else {
                    for (uint32_t g = 0; g < (uint32_t)NW / 16; g++, ptr += 4) {
#pragma unroll
                        for (int c = 0; c < CH; c++) my[lane * CH + (c ^ wx)] = gen.next4();
                        __syncwarp();
#pragma unroll
                        for (int k = 0; k < 4; k++) {
                            const uint4 v = my[rslot + 32 * k];
                            if constexpr (OUT == 0) __stcs(reinterpret_cast<uint4 *>(ptr) + k * 2 * NW, v);
                            else __stcs(reinterpret_cast<float4 *>(ptr) + k * 2 * NW, u32x4_to_f32x4<CV>(v, a.m24));
                        }
                        __syncwarp();
                    }
                }
                continue;
            }
        }
        for (uint32_t g = 0; g < groups; g++, at += 4 * CH) {
#pragma unroll
            for (int c = 0; c < CH; c++) my[lane * CH + (c ^ wx)] = gen.next4();
            __syncwarp();
#pragma unroll
            for (int k = 0; k < (int)CH; k++) {
                if (rrow + RPI * k < rows_left) {
                    const uint32_t slot = CH == 4 ? rslot + 32 * k : (rslot + 32 * k) ^ (4 * (k & 1));
                    const uint4 v = my[slot];
                    if constexpr (VEC) {
                        store4<OUT, CV>(a.out, at + k * rstride, v, a.m24);
                    } else {  // rows not 16-byte aligned (nwords % 4 != 0)
                        const uint64_t o = at + k * rstride;
                        store1<OUT>(a.out, o, v.x); store1<OUT>(a.out, o + 1, v.y);
                        store1<OUT>(a.out, o + 2, v.z); store1<OUT>(a.out, o + 3, v.w);
                    }
                }
            }
            __syncwarp();
        }
        for (uint32_t j = 0; j < rem; j += 4) {
            const uint4 w = gen.next4();  // may run up to 3 words past the row end: discarded
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
            if (valid)
                for (uint32_t q = 0; q < 4 && j + q < rem; q++)
                    store1<OUT>(a.out, sid * a.nwords + groups * 4 * CH + j + q, ws[q]);
        }
    }
}

// Grid: Tyche uses the resident x8 persistent grid like the fills; the
// counter-based row generators one CTA per 256 streams (every thread one row):
// Philox 1e8 x 256 words 5386 -> 5689 GB/s (profiles/r1t_tune.md).
// 256-word rows with the copy-out done by the tensor-memory accelerator: the
// warp stages its 32 rows x 16 words in shared memory exactly as
// staged_prefix_kernel does (16-byte chunk c of row r at c ^ ((r >> 1) & 3),
// which is the hardware's SWIZZLE_64B pattern for 64-byte rows), then one lane
// issues a single 2 KB cp.async.bulk.tensor store of the [32 x 16] box. No
// LDS/STG per lane, no row predicates: the TMA clips rows past n_streams.
// The f32 map is applied before staging.
template <int ALG, int OUT, int CV>
__global__ void __launch_bounds__(256, staged_min_blocks<ALG>())
    staged_tma_kernel(const __grid_constant__ PrefixArgs a, const __grid_constant__ CUtensorMap tmap) {
    __shared__ __align__(1024) uint4 tile[TY_WARPS][32 * 4];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint4 *const my = tile[wib];
    const uint32_t smem = (uint32_t)__cvta_generic_to_shared(my);
    const uint32_t wx = (lane >> 1) & 3;
    for (uint64_t s0 = warp * 32; s0 < a.n_streams; s0 += nwarps * 32) {
        const uint64_t sid = s0 + lane;
        const bool valid = sid < a.n_streams;
        RowGen<ALG> gen(valid ? seed_of(a, sid) : 0, valid ? ctr_of(a, sid) : 0);
        for (uint32_t g = 0; g < a.nwords / 16; g++) {
            // the previous store of this warp's tile must have read it
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 4; c++) {
                uint4 w = gen.next4();
                if constexpr (OUT == 1) {
                    const float4 f = u32x4_to_f32x4<CV>(w, a.m24);
                    w = make_uint4(__float_as_uint(f.x), __float_as_uint(f.y), __float_as_uint(f.z), __float_as_uint(f.w));
                }
                my[lane * 4 + (c ^ wx)] = w;
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> TMA
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n\t"
                    "cp.async.bulk.commit_group;"
                    :
                    : "l"(reinterpret_cast<uint64_t>(&tmap)), "r"((int)(16 * g)), "r"((int)s0), "r"(smem)
                    : "memory");
            }
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

[[maybe_unused]] static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// [n_streams][nwords] 4-byte elements, box 32 rows x 16 words, 64-byte swizzle.
[[maybe_unused]] static bool rows_tensor_map(CUtensorMap *m, void *out, uint64_t n_streams, uint32_t nwords, bool f32) {
    const auto encode = tensor_map_encoder();
    if (!encode || n_streams > 0x7FFFFFFFull) return false;
    const cuuint64_t dims[2] = {nwords, n_streams};
    const cuuint64_t strides[1] = {(cuuint64_t)nwords * 4};
    const cuuint32_t box[2] = {16, 32};
    const cuuint32_t estr[2] = {1, 1};
    return encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// f32 conversion placement per generator (B200 sweeps, profiles/r1r_tune.md,
// r1t_tune.md); tuning build: CBRNG_CVT_MS=0..5. Tyche's lean
// 256-word copy-out prefers the shift on the multiplier (IMAD.HI) and I2FP.
// Re-swept after the NW=256 Threefry rows and the stepped Squares rows (r1t_tune.md):
// Philox rows f32 CV 0 (+2.4 % over CV 4), Squares CV 4 (+0.7 % over CV 0).
template <int ALG> constexpr int ms_cv_default() { return ALG == PHILOX ? 0 : ALG == TYCHE ? 1 : 4; }

constexpr bool MS_TMA_DEFAULT = false;

// Tyche (tuning build): CBRNG_TY_GRID = k -> k x resident CTAs (persistent), 0 ->
// one CTA per 256 streams.
constexpr int TY_GRID_DEFAULT = 0;  // one CTA per 256 streams: robust across boxes (r1t_tune.md)

template <int ALG>
static unsigned staged_grid(const void *kernel, uint64_t n_streams) {
    const uint64_t work = (n_streams + 255) / 256;
    if constexpr (TUNING && ALG == TYCHE) {
        static const int k = tuning_knob("CBRNG_TY_GRID", TY_GRID_DEFAULT, 0, 64);
        if (k > 0) {
            const uint64_t g = (uint64_t)resident_blocks(kernel, 256, 0) * k;
            return (unsigned)(g < work ? g : work);
        }
    } else {
        (void)kernel;
    }
    return (unsigned)(work < 0x7FFFFFFFull ? work : 0x7FFFFFFFull);
}

template <int ALG, int OUT, int CV, int CH>
static int launch_staged_ch(const PrefixArgs &a, cudaStream_t st) {
    if constexpr (TUNING && CH == 4 && ALG != THREEFRY) {
        // TMA copy-out (tuning build, CBRNG_MS_TMA=1; measured no faster than the LDS/STG copy-out)
        static const bool tma = tuning_knob("CBRNG_MS_TMA", MS_TMA_DEFAULT, 0, 1) != 0;
        CUtensorMap m;
        if (tma && a.nwords == 256 && rows_tensor_map(&m, a.out, a.n_streams, a.nwords, OUT == 1)) {
            auto k = staged_tma_kernel<ALG, OUT, CV>;
            k<<<staged_grid<ALG>(reinterpret_cast<const void *>(k), a.n_streams), 256, 0, st>>>(a, m);
            return check_launch("staged_tma_kernel");
        }
    }
    if constexpr (CH == 4) {
        if (a.nwords == 256) {
            auto k = staged_prefix_kernel<ALG, OUT, true, CV, CH, 256>;
            k<<<staged_grid<ALG>(reinterpret_cast<const void *>(k), a.n_streams), 256, 0, st>>>(a);
            return check_launch("staged_prefix_kernel");
        }
    }
    if (a.nwords % 4 == 0) {
        auto k = staged_prefix_kernel<ALG, OUT, true, CV, CH>;
        k<<<staged_grid<ALG>(reinterpret_cast<const void *>(k), a.n_streams), 256, 0, st>>>(a);
    } else {
        auto k = staged_prefix_kernel<ALG, OUT, false, CV, CH>;
        k<<<staged_grid<ALG>(reinterpret_cast<const void *>(k), a.n_streams), 256, 0, st>>>(a);
    }
    return check_launch("staged_prefix_kernel");
}

// Staging width (tuning build: CBRNG_TY_CH=4|8; Tyche only).
constexpr int TY_CH_DEFAULT = 4;

template <int ALG, int OUT, int CV>
static int launch_staged_cv(const PrefixArgs &a, cudaStream_t st) {
    if constexpr (TUNING && ALG == TYCHE && OUT == 1) {  // (the u32 variant spills at CH 8)
        static const int ch = tuning_knob("CBRNG_TY_CH", TY_CH_DEFAULT, 4, 8);
        if (ch == 8) return launch_staged_ch<ALG, OUT, CV, 8>(a, st);
    }
    return launch_staged_ch<ALG, OUT, CV, 4>(a, st);
}


template <int ALG, int OUT>
static int launch_staged(const PrefixArgs &a, cudaStream_t st) {
    constexpr int C0 = ms_cv_default<ALG>();
    if constexpr (TUNING && OUT == 1) {
        static const int cv = tuning_knob("CBRNG_CVT_MS", C0, 0, 5);
        switch (cv) {
            case 0: return launch_staged_cv<ALG, OUT, 0>(a, st);
            case 1: return launch_staged_cv<ALG, OUT, 1>(a, st);
            case 2: return launch_staged_cv<ALG, OUT, 2>(a, st);
            case 3: return launch_staged_cv<ALG, OUT, 3>(a, st);
            case 4: return launch_staged_cv<ALG, OUT, 4>(a, st);
            default: return launch_staged_cv<ALG, OUT, 5>(a, st);
        }
    }
    return launch_staged_cv<ALG, OUT, C0>(a, st);
}

// Rows of 256 words of a block cipher (configs[4]) with LPR lanes per row and
// no staging: the LPR lanes of a row each set up the row's stream (the folded
// key material of philox/threefry_stream_setup, LPR-fold redundant) and take
// blocks sub, sub + LPR, ... (64 / LPR blocks in flight per lane), so each
// store instruction writes 32 / LPR rows x LPR consecutive 16-byte blocks
// (64-byte row segments at LPR = 4, full 128-byte lines at 8) straight from
// registers. Against the one-thread-per-row staged kernel (B200, 2^22 x 256,
// profiles/r2k_tune.md): Philox u32 6174 -> 7120 GB/s at LPR 4, f32 6084 ->
// 6424; Threefry u32 3510 -> 3652 and f32 3202 -> 3357 at LPR 8.
template <int ALG, int OUT, int CV, int LPR, int MB>
__global__ void __launch_bounds__(256, MB) rowsplit_kernel(const __grid_constant__ PrefixArgs a) {
    static_assert(ALG == PHILOX || ALG == THREEFRY, "block ciphers only");
    constexpr uint32_t NB = 64, RPW = 32 / LPR, ILP = NB / LPR;
    const uint32_t lane = threadIdx.x & 31, sub = lane % LPR, rw = lane / LPR;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r0 = warp * RPW; r0 < a.n_streams; r0 += nwarps * RPW) {
        const uint64_t r = r0 + rw;
        if (r >= a.n_streams) continue;
        uint4 w[ILP];
        if constexpr (ALG == PHILOX) {
            const PhiloxStream p = philox_stream_setup(seed_of(a, r), ctr_of(a, r));
#pragma unroll
            for (uint32_t j = 0; j < ILP; j++) w[j] = philox_stream_block(p, sub + LPR * j);
        } else {
            ThreefryStream p = threefry_stream_setup(seed_of(a, r), ctr_of(a, r));
            p.one = c_one;  // keep the forced adds on the FMA-heavy pipe (RowGen<THREEFRY>)
#pragma unroll
            for (uint32_t j = 0; j < ILP; j++) w[j] = threefry_stream_block<0, true, true>(p, sub + LPR * j);
        }
        const uint64_t row = CBRNG_CEILING ? (r & 2047u) : r;  // ceiling build: one L2-resident ring
#pragma unroll
        for (uint32_t j = 0; j < ILP; j++) store4<OUT, CV>(a.out, row * 256 + 4ull * (sub + LPR * j), w[j], a.m24);
    }
}

template <int ALG, int OUT, int LPR>
static int launch_rowsplit(const PrefixArgs &a, cudaStream_t st) {
    constexpr int CV = ms_cv_default<ALG>();
    auto k = rowsplit_kernel<ALG, OUT, CV, LPR, 0>;
    const uint64_t work = (a.n_streams + 8 * (32 / LPR) - 1) / (8 * (32 / LPR));
    k<<<grid_for(k, 256, 0, work ? work : 1), 256, 0, st>>>(a);
    return check_launch("rowsplit_kernel");
}

// Lanes per 256-word row of the block ciphers (0: the staged kernel).
template <int ALG> constexpr int ms_split_default() { return ALG == PHILOX ? 4 : ALG == THREEFRY ? 8 : 0; }

template <int ALG, int OUT>
static int launch_prefix(const PrefixArgs &a, cudaStream_t st) {
    if constexpr (ALG == PHILOX || ALG == THREEFRY) {
        if (a.nwords == 256 && a.n_streams > 0) {
            if constexpr (TUNING) {  // CBRNG_MS_SPLIT = 0 (staged) / 4 / 8 / 16
                static const int lpr = tuning_knob("CBRNG_MS_SPLIT", ms_split_default<ALG>(), 0, 16);
                if (lpr == 4) return launch_rowsplit<ALG, OUT, 4>(a, st);
                if (lpr == 8) return launch_rowsplit<ALG, OUT, 8>(a, st);
                if (lpr == 16) return launch_rowsplit<ALG, OUT, 16>(a, st);
            } else {
                return launch_rowsplit<ALG, OUT, ms_split_default<ALG>()>(a, st);
            }
        }
    }
    // Rows of >= 16 words: one thread per stream with the stream setup folded
    // once per row, staged through shared memory (ncu: the warp-per-row kernel
    // spends ~20 % of its FMA-heavy cycles re-deriving the key schedule).
    if constexpr (ALG == TYCHE) {
        return launch_staged<ALG, OUT>(a, st);
    } else {
        if (a.nwords >= 16) return launch_staged<ALG, OUT>(a, st);
        if (a.nwords % 4 == 0) {
            auto k = prefix_kernel<ALG, OUT, 4>;
            uint64_t chunks = a.n_streams * (a.nwords / 4);
            k<<<grid_for(k, 256, 0, (chunks + 255) / 256), 256, 0, st>>>(a);
        } else {
            auto k = prefix_kernel<ALG, OUT, 1>;
            uint64_t chunks = a.n_streams * a.nwords;
            k<<<grid_for(k, 256, 0, (chunks + 255) / 256), 256, 0, st>>>(a);
        }
        return check_launch("prefix_kernel");
    }
}

template <int OUT>
static int dispatch_prefix(int alg, const uint64_t *seeds, uint64_t seed_base, const uint32_t *ctrs,
                           uint32_t ctr_scalar, uint64_t n_streams, uint32_t nwords, void *out, void *stream) {
    CBRNG_CHECK_ALG(alg);
    clear_error();
    if (n_streams == 0 || nwords == 0) return CBRNG_OK;
    CBRNG_REQUIRE(out != nullptr, "out is NULL");
    if (nwords % 4 == 0 && !aligned(out, 16)) {
        set_error("output pointer not 16-byte aligned");
        return CBRNG_EALIGN;
    }
    PrefixArgs a{seeds, seed_base, ctrs, ctr_scalar, nwords, n_streams, out, 1u << 24};
    cudaStream_t st = as_stream(stream);
    switch (alg) {
        case PHILOX: return launch_prefix<PHILOX, OUT>(a, st);
        case THREEFRY: return launch_prefix<THREEFRY, OUT>(a, st);
        case SQUARES: return launch_prefix<SQUARES, OUT>(a, st);
        default: return launch_prefix<TYCHE, OUT>(a, st);
    }
}

// ---------------- vector block functions ----------------
__global__ void philox4x32_kernel(const uint32_t *ctr, const uint32_t *key, uint64_t n, uint32_t *out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 r = philox_block(make_uint4(ctr[i], ctr[n + i], ctr[2 * n + i], ctr[3 * n + i]), key[i], key[n + i]);
        out[i] = r.x; out[n + i] = r.y; out[2 * n + i] = r.z; out[3 * n + i] = r.w;
    }
}

__global__ void threefry4x32_kernel(const uint32_t *ctr, const uint32_t *key, int rounds, uint64_t n, uint32_t *out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 c = make_uint4(ctr[i], ctr[n + i], ctr[2 * n + i], ctr[3 * n + i]);
        uint4 r;
        if (rounds == 20) {
            r = threefry_block(c, key[i], key[n + i], key[2 * n + i], key[3 * n + i]);
        } else {
            uint32_t k[4] = {key[i], key[n + i], key[2 * n + i], key[3 * n + i]};
            r = threefry_block_rounds(c, k, rounds);
        }
        out[i] = r.x; out[n + i] = r.y; out[2 * n + i] = r.z; out[3 * n + i] = r.w;
    }
}

__global__ void squares32_kernel(const uint64_t *ctr, const uint64_t *key, uint64_t n, uint32_t *out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = squares_round(key[i], ctr[i]);
}

__global__ void squares_keys_kernel(const uint64_t *seeds, uint64_t n, uint64_t *keys) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = squares_key(seeds[i]);
}

__global__ void tyche_mix_kernel(uint32_t *s, uint64_t n, uint32_t rounds) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t a = s[i], b = s[n + i], c = s[2 * n + i], d = s[3 * n + i];
        for (uint32_t r = 0; r < rounds; r++) tyche_mix(a, b, c, d);
        s[i] = a; s[n + i] = b; s[2 * n + i] = c; s[3 * n + i] = d;
    }
}

__global__ void tyche_init_kernel(const uint64_t *seeds, uint64_t seed_base, const uint32_t *ctrs, uint32_t ctr_scalar,
                                  uint64_t n, uint32_t *s) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 t = tyche_init(seeds ? seeds[i] : seed_base + i, ctrs ? ctrs[i] : ctr_scalar);
        s[i] = t.x; s[n + i] = t.y; s[2 * n + i] = t.z; s[3 * n + i] = t.w;
    }
}

// One scalar block function with its arguments by value (cbrng_scalar ops 0-5):
// the result goes straight into the caller's mapped pinned buffer, so a call
// costs one launch and one synchronisation and reads nothing over PCIe.
struct ScalarArgs {
    uint64_t a[9];
};

__global__ void scalar_kernel(int op, const __grid_constant__ ScalarArgs s, uint32_t *out) {
    const uint64_t *a = s.a;
    switch (op) {
        case 0: {  // philox_block: ctr0..3, key0..1
            const uint4 r = philox_block(make_uint4((uint32_t)a[0], (uint32_t)a[1], (uint32_t)a[2], (uint32_t)a[3]),
                                         (uint32_t)a[4], (uint32_t)a[5]);
            out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
            break;
        }
        case 1: {  // threefry_block: ctr0..3, key0..3, rounds
            const uint4 c = make_uint4((uint32_t)a[0], (uint32_t)a[1], (uint32_t)a[2], (uint32_t)a[3]);
            uint32_t k[4] = {(uint32_t)a[4], (uint32_t)a[5], (uint32_t)a[6], (uint32_t)a[7]};
            const uint4 r = threefry_block_rounds(c, k, (int)a[8]);
            out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
            break;
        }
        case 2: {  // squares_key: seed -> (lo, hi)
            const uint64_t k = squares_key(a[0]);
            out[0] = (uint32_t)k; out[1] = (uint32_t)(k >> 32);
            break;
        }
        case 3: out[0] = squares_round(a[0], a[1]); break;  // key, ctr
        case 4: {  // tyche_init: seed, stream counter
            const uint4 t = tyche_init(a[0], (uint32_t)a[1]);
            out[0] = t.x; out[1] = t.y; out[2] = t.z; out[3] = t.w;
            break;
        }
        default: {  // tyche_mix x rounds: state0..3, rounds
            uint32_t w = (uint32_t)a[0], x = (uint32_t)a[1], y = (uint32_t)a[2], z = (uint32_t)a[3];
            for (uint64_t r = 0; r < a[4]; r++) tyche_mix(w, x, y, z);
            out[0] = w; out[1] = x; out[2] = y; out[3] = z;
            break;
        }
    }
}

int launch_scalar(int op, const uint64_t *args, uint32_t nargs, uint32_t *out, cudaStream_t st) {
    ScalarArgs s = {};
    for (uint32_t i = 0; i < nargs && i < 9; i++) s.a[i] = args[i];
    scalar_kernel<<<1, 1, 0, st>>>(op, s, out);
    return check_launch("scalar_kernel");
}

__global__ void philox_block_lanes_kernel(const uint64_t *seeds, const uint64_t *scs, uint64_t block_ctr, uint64_t n,
                                          uint32_t *out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s = seeds[i];
        uint4 r = philox_block(make_uint4((uint32_t)scs[i], (uint32_t)block_ctr, 0, 0), (uint32_t)s, (uint32_t)(s >> 32));
        reinterpret_cast<uint4 *>(out)[i] = r;
    }
}

template <typename K>
static unsigned lanes_grid(K k, uint64_t n) { return grid_for(k, 256, 0, (n + 255) / 256); }

}  // namespace cbrng

using namespace cbrng;

extern "C" {

int cbrng_prefix_words(int alg, const uint64_t *seeds, uint64_t seed_base, const uint32_t *ctrs, uint32_t ctr_scalar,
                       uint64_t n_streams, uint32_t nwords, uint32_t *out, void *stream) {
    const DeviceGuard device_guard(stream);
    return dispatch_prefix<0>(alg, seeds, seed_base, ctrs, ctr_scalar, n_streams, nwords, out, stream);
}

int cbrng_prefix_uniform_f32(int alg, const uint64_t *seeds, uint64_t seed_base, const uint32_t *ctrs,
                             uint32_t ctr_scalar, uint64_t n_streams, uint32_t nvalues, float *out, void *stream) {
    const DeviceGuard device_guard(stream);
    return dispatch_prefix<1>(alg, seeds, seed_base, ctrs, ctr_scalar, n_streams, nvalues, out, stream);
}

int cbrng_philox_block_lanes(const uint64_t *seeds, const uint64_t *stream_ctrs, uint64_t block_ctr, uint64_t n,
                             uint32_t *out, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(seeds && stream_ctrs && out, "NULL pointer");
    if (!aligned(out, 16)) { set_error("out not 16-byte aligned"); return CBRNG_EALIGN; }
    philox_block_lanes_kernel<<<lanes_grid(philox_block_lanes_kernel, n), 256, 0, as_stream(stream)>>>(
        seeds, stream_ctrs, block_ctr, n, out);
    return check_launch("philox_block_lanes_kernel");
}

int cbrng_philox4x32(const uint32_t *ctr, const uint32_t *key, uint64_t n, uint32_t *out, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(ctr && key && out, "NULL pointer");
    philox4x32_kernel<<<lanes_grid(philox4x32_kernel, n), 256, 0, as_stream(stream)>>>(ctr, key, n, out);
    return check_launch("philox4x32_kernel");
}

int cbrng_threefry4x32(const uint32_t *ctr, const uint32_t *key, int rounds, uint64_t n, uint32_t *out, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    CBRNG_REQUIRE(rounds >= 0, "rounds must be >= 0");
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(ctr && key && out, "NULL pointer");
    threefry4x32_kernel<<<lanes_grid(threefry4x32_kernel, n), 256, 0, as_stream(stream)>>>(ctr, key, rounds, n, out);
    return check_launch("threefry4x32_kernel");
}

int cbrng_squares32(const uint64_t *ctr, const uint64_t *key, uint64_t n, uint32_t *out, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(ctr && key && out, "NULL pointer");
    squares32_kernel<<<lanes_grid(squares32_kernel, n), 256, 0, as_stream(stream)>>>(ctr, key, n, out);
    return check_launch("squares32_kernel");
}

int cbrng_squares_keys(const uint64_t *seeds, uint64_t n, uint64_t *keys, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(seeds && keys, "NULL pointer");
    squares_keys_kernel<<<lanes_grid(squares_keys_kernel, n), 256, 0, as_stream(stream)>>>(seeds, n, keys);
    return check_launch("squares_keys_kernel");
}

int cbrng_tyche_mix(uint32_t *state, uint64_t n, uint32_t rounds, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    if (n == 0 || rounds == 0) return CBRNG_OK;
    CBRNG_REQUIRE(state, "NULL pointer");
    tyche_mix_kernel<<<lanes_grid(tyche_mix_kernel, n), 256, 0, as_stream(stream)>>>(state, n, rounds);
    return check_launch("tyche_mix_kernel");
}

int cbrng_tyche_init(const uint64_t *seeds, uint64_t seed_base, const uint32_t *ctrs, uint32_t ctr_scalar, uint64_t n,
                     uint32_t *state, void *stream) {
    const DeviceGuard device_guard(stream);
    clear_error();
    if (n == 0) return CBRNG_OK;
    CBRNG_REQUIRE(state, "NULL pointer");
    tyche_init_kernel<<<lanes_grid(tyche_init_kernel, n), 256, 0, as_stream(stream)>>>(seeds, seed_base, ctrs,
                                                                                        ctr_scalar, n, state);
    return check_launch("tyche_init_kernel");
}

}  // extern "C"
