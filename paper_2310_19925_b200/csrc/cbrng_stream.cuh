// cbrng_stream.cuh — one single-stream "unit" (4 consecutive words) of any
// counter-based generator, shared by the fill kernels (cbrng_fill.cu) and the
// fused battery producers (cbrng_stats.cu).
#pragma once
#include "cbrng_cores.cuh"

namespace cbrng {

template <int ALG> struct StreamOf;
template <> struct StreamOf<PHILOX> { using T = PhiloxStream; };
template <> struct StreamOf<THREEFRY> { using T = ThreefryStream; };
template <> struct StreamOf<SQUARES> { using T = SquaresStream; };


// V selects a code variant per algorithm. Philox: V = 1 splits each mulhilo
// into IMAD.HI + IMAD, V > 1 the rounds of the bit mask V (philox_stream_block). Threefry (adds "forced" = emitted as
// IMAD on the FMA-heavy pipe instead of IADD3 on the ALU pipe; "mul" rotations
// = IMAD.WIDE by 2^r instead of SHF.L.W):
//   V = 0 compiler-scheduled;             V = 1: forced round adds + 10 mul rotations;
//   V = 2: forced round adds;             V = 3: forced round adds + 6 mul rotations;
//   V = 4: forced round + injection adds; V = 5/6/7/8: V4 + 2/4/6/8 mul rotations.
template <int ALG, int V>
__device__ __forceinline__ uint4 block_at(const typename StreamOf<ALG>::T &p, uint32_t bc) {
    if constexpr (ALG == PHILOX) return philox_stream_block<V>(p, bc);  // V: split-mulhilo round mask (1 = all)
    else if constexpr (V == 0) return threefry_stream_block<0, false>(p, bc);
    else if constexpr (V == 1) return threefry_stream_block<10, true>(p, bc);
    else if constexpr (V == 2) return threefry_stream_block<0, true>(p, bc);
    else if constexpr (V == 3) return threefry_stream_block<6, true>(p, bc);
    else if constexpr (V == 4) return threefry_stream_block<0, true, true>(p, bc);
    else if constexpr (V == 5) return threefry_stream_block<2, true, true>(p, bc);
    else if constexpr (V == 6) return threefry_stream_block<4, true, true>(p, bc);
    else if constexpr (V == 7) return threefry_stream_block<6, true, true>(p, bc);
    else return threefry_stream_block<8, true, true>(p, bc);
}

template <int ALG, bool SKIP, int V = 0>
__device__ __forceinline__ uint4 unit_words(const typename StreamOf<ALG>::T &p, uint32_t bc0, uint32_t skip, uint64_t u) {
    if constexpr (ALG == SQUARES) {
        // V == 1: the host proved the fill never wraps the 32-bit counter
        return squares_stream_word4<V == 1>(p, bc0 + 4u * (uint32_t)u);
    } else if constexpr (!SKIP) {
        return block_at<ALG, V>(p, bc0 + (uint32_t)u);
    } else {
        uint4 a = block_at<ALG, V>(p, bc0 + (uint32_t)u), b = block_at<ALG, V>(p, bc0 + (uint32_t)u + 1);
        if (skip == 1) return make_uint4(a.y, a.z, a.w, b.x);
        if (skip == 2) return make_uint4(a.z, a.w, b.x, b.y);
        return make_uint4(a.w, b.x, b.y, b.z);
    }
}


// Launch-uniform setup of a single stream (host): the folded key material.
template <int ALG>
inline typename StreamOf<ALG>::T stream_setup(uint64_t seed, uint32_t sc) {
    if constexpr (ALG == PHILOX) return philox_stream_setup(seed, sc);
    else if constexpr (ALG == THREEFRY) return threefry_stream_setup(seed, sc);
    else return squares_stream_setup(seed, sc);
}

}  // namespace cbrng
