// Pipe-throughput probes (one B200): instructions/clk/SM for DFMA (register
// and uniform-register operands), DMUL, IMAD, IMAD.WIDE, IMAD.HI, LOP3, SHF, I2F.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_pipes probe_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8;       // independent chains per thread
constexpr int IT = 4096;    // iterations

__global__ void k_dfma(double *out, double a, double b) {
    double x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = fma(x[c], a, b);
    double s = 0;
    for (int c = 0; c < CH; c++) s += x[c];
    if (s == 1.2345) out[0] = s;
}
__global__ void k_dfma_reg(double *out, const double *ab) {
    double a = ab[threadIdx.x & 1], b = ab[2 + (threadIdx.x & 1)];  // non-uniform -> regular registers
    double x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = fma(x[c], a, b);
    double s = 0;
    for (int c = 0; c < CH; c++) s += x[c];
    if (s == 1.2345) out[0] = s;
}
__global__ void k_dmul(double *out, double a) {
    double x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 1e-9 + c;
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = x[c] * a;
    double s = 0;
    for (int c = 0; c < CH; c++) s += x[c];
    if (s == 1.2345) out[0] = s;
}
template <int OP>
__global__ void k_int(uint32_t *out, uint32_t a, uint32_t b) {
    uint32_t x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 7 + c;
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) {
            if constexpr (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
            else if constexpr (OP == 1) { uint64_t p; asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(x[c]), "r"(a), "l"((uint64_t)b)); x[c] = (uint32_t)p ^ (uint32_t)(p >> 32); }
            else if constexpr (OP == 2) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
            else if constexpr (OP == 3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
            else if constexpr (OP == 4) asm volatile("shf.l.wrap.b32 %0, %0, %0, 13;" : "+r"(x[c]));
            else { float f; asm volatile("cvt.rm.f32.u32 %0, %1;" : "=f"(f) : "r"(x[c])); x[c] = __float_as_uint(f) + b; }
        }
    uint32_t s = 0;
    for (int c = 0; c < CH; c++) s += x[c];
    if (s == 12345) out[0] = s;
}

// Pipe-sharing probe: CH/2 DFMA chains and CH/2 IMAD chains interleaved.
__global__ void k_mix(double *out, double a, double b, uint32_t ia, uint32_t ib) {
    double x[CH / 2];
    uint32_t y[CH / 2];
    for (int c = 0; c < CH / 2; c++) { x[c] = threadIdx.x * 1e-9 + c; y[c] = threadIdx.x * 3 + c; }
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH / 2; c++) {
            x[c] = fma(x[c], a, b);
            asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[c]) : "r"(ia), "r"(ib));
        }
    double s = 0;
    for (int c = 0; c < CH / 2; c++) s += x[c] + y[c];
    if (s == 1.2345) out[0] = s;
}
// DFMA interleaved with LOP3 (ALU pipe) as a control.
__global__ void k_mix_alu(double *out, double a, double b, uint32_t ia, uint32_t ib) {
    double x[CH / 2];
    uint32_t y[CH / 2];
    for (int c = 0; c < CH / 2; c++) { x[c] = threadIdx.x * 1e-9 + c; y[c] = threadIdx.x * 3 + c; }
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH / 2; c++) {
            x[c] = fma(x[c], a, b);
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[c]) : "r"(ia), "r"(ib));
        }
    double s = 0;
    for (int c = 0; c < CH / 2; c++) s += x[c] + y[c];
    if (s == 1.2345) out[0] = s;
}
__global__ void k_i2f64(double *out, uint32_t b) {
    uint64_t x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 7ull + c;
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) {
            double d;
            asm volatile("cvt.rn.f64.u64 %0, %1;" : "=d"(d) : "l"(x[c]));
            x[c] = (uint64_t)__double_as_longlong(d) + b;
        }
    uint64_t s = 0;
    for (int c = 0; c < CH; c++) s += x[c];
    if (s == 12345) out[0] = (double)s;
}

// IMAD.WIDE alone: 64-bit accumulator chains x = lo32(x) * a + x (mad.wide.u32 with a 64-bit addend).
__global__ void k_wide(uint64_t *out, uint32_t a) {
    uint64_t x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 7ull + c;
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(x[c]) : "r"((uint32_t)x[c]), "r"(a));
    uint64_t s = 0;
    for (int c = 0; c < CH; c++) s += x[c];
    if (s == 12345) out[0] = s;
}

// IMAD.WIDE without an addend: x = lo32(x) * a as a 64-bit product (mul.wide.u32),
// chains fed through lo32 so only the multiply sits on the loop.
__global__ void k_wide_noadd(uint64_t *out, uint32_t a) {
    uint64_t x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 7ull + c + 1;
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(x[c]) : "r"((uint32_t)(x[c] >> 7)), "r"(a));
    uint64_t s = 0;
    for (int c = 0; c < CH; c++) s += x[c];
    if (s == 12345) out[0] = s;
}


// Mixes (r2f): per chain and iteration NW mul.wide.u32 (IMAD.WIDE, no addend),
// NL lop3 (ALU) and ND DFMA with register operands, round-robin in program order
// (asm volatile): which combinations of the Box-Muller fill's pipes co-issue.
template <int NW, int NL, int ND>
__global__ void k_ratio(double *out, const double *ab, uint32_t ia, uint32_t ib) {
    const double a = ab[threadIdx.x & 1], b = ab[2 + (threadIdx.x & 1)];
    double x[CH / 2];
    uint32_t y[CH / 2], z[CH / 2];
    for (int c = 0; c < CH / 2; c++) { x[c] = threadIdx.x * 1e-9 + c; y[c] = threadIdx.x * 3 + c; z[c] = c; }
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH / 2; c++) {
#pragma unroll
            for (int k = 0; k < (NW > NL ? (NW > ND ? NW : ND) : (NL > ND ? NL : ND)); k++) {
                if (k < NW) { uint64_t p; asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(y[c]), "r"(ia)); y[c] = (uint32_t)(p >> 32); z[c] ^= (uint32_t)p; }
                if (k < NL) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(z[c]) : "r"(ia), "r"(ib));
                if (k < ND) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(a), "d"(b));
            }
        }
    double s = 0;
    for (int c = 0; c < CH / 2; c++) s += x[c] + y[c] + z[c];
    if (s == 1.2345) out[0] = s;
}

// r2f op-mix probe: per chain-iteration NW IMAD.WIDE (hi feeds the chain, lo
// xor-folded), NH IMAD.HI, NI IMAD, NL LOP3, ND DFMA (register operands), NU
// DFMA (uniform operands); asm volatile keeps the program order round-robin.
template <int NW, int NH, int NI, int NL, int ND, int NU>
__global__ void k_ops(double *out, const double *ab, uint32_t ia, uint32_t ib, double ua, double ub) {
    const double a = ab[threadIdx.x & 1], b = ab[2 + (threadIdx.x & 1)];
    constexpr int M0 = NW > NH ? NW : NH, M1 = NI > NL ? NI : NL, M2 = ND > NU ? ND : NU;
    constexpr int MX = M0 > M1 ? (M0 > M2 ? M0 : M2) : (M1 > M2 ? M1 : M2);
    double x[CH / 2], v[CH / 2];
    uint32_t y[CH / 2], z[CH / 2], q[CH / 2];
    for (int c = 0; c < CH / 2; c++) { x[c] = threadIdx.x * 1e-9 + c; v[c] = x[c] + 1; y[c] = threadIdx.x * 3 + c; z[c] = threadIdx.x ^ c; q[c] = 5 * threadIdx.x + c + 1; }
    for (int i = 0; i < IT; i++)
#pragma unroll
        for (int c = 0; c < CH / 2; c++) {
#pragma unroll
            for (int k = 0; k < MX; k++) {
                if (k < NW) { uint32_t lo, hi; asm volatile("{.reg .b64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;}" : "=r"(lo), "=r"(hi) : "r"(y[c]), "r"(ia)); y[c] = hi; z[c] ^= lo; }
                if (k < NH) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(q[c]) : "r"(ia));
                if (k < NI) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[c]) : "r"(ia), "r"(ib));
                if (k < NL) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(z[c]) : "r"(ia), "r"(ib));
                if (k < ND) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[c]) : "d"(a), "d"(b));
                if (k < NU) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(v[c]) : "d"(ua), "d"(ub));
            }
        }
    double s = 0;
    for (int c = 0; c < CH / 2; c++) s += x[c] + v[c] + y[c] + z[c] + q[c];
    if (s == 1.2345) out[0] = s;
}

template <typename K, typename... A>
static void run(const char *name, double per_iter_instr, K k, A... args) {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);  // kHz
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, 256, 0);
    dim3 grid(sms * blocks);
    k<<<grid, 256>>>(args...);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) k<<<grid, 256>>>(args...);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double instr = 5.0 * grid.x * 256.0 * IT * CH * per_iter_instr;
    double per_clk_sm = instr / (ms * 1e-3) / sms / (clk * 1e3);
    printf("{\"probe\": \"%s\", \"thread_ops_per_clk_per_sm_at_max_clock\": %.1f, \"blocks_per_sm\": %d}\n", name, per_clk_sm, blocks);
}

int main() {
    double *d; uint32_t *u; double *ab;
    cudaMalloc(&d, 64); cudaMalloc(&u, 64); cudaMalloc(&ab, 64);
    double h[4] = {1.0000001, 0.9999999, 1e-9, 2e-9};
    cudaMemcpy(ab, h, 32, cudaMemcpyHostToDevice);
    run("DFMA (uniform operands)", 1, k_dfma, d, 1.0000001, 1e-9);
    run("DFMA (register operands)", 1, k_dfma_reg, d, (const double *)ab);
    run("DMUL", 1, k_dmul, d, 1.0000001);
    run("IMAD", 1, k_int<0>, u, 0x12345u, 7u);
    run("IMAD.WIDE (+LOP3)", 2, k_int<1>, u, 0x12345u, 7u);
    run("IMAD.HI", 1, k_int<2>, u, 0x12345u, 7u);
    run("LOP3", 1, k_int<3>, u, 0x12345u, 7u);
    run("SHF.L.W", 1, k_int<4>, u, 0x12345u, 7u);
    run("I2F.RM (+IADD)", 2, k_int<5>, u, 0x12345u, 7u);
    run("DFMA + IMAD interleaved (1:1)", 1, k_mix, d, 1.0000001, 1e-9, 0x12345u, 7u);
    run("DFMA + LOP3 interleaved (1:1)", 1, k_mix_alu, d, 1.0000001, 1e-9, 0x12345u, 7u);
    run("I2F.F64.U64 (+IADD 64)", 1, k_i2f64, d, 7u);
    run("IMAD.WIDE (64-bit addend, alone)", 1, k_wide, (uint64_t *)u, 0x12345u);
    run("IMAD.WIDE (no addend, + SHF)", 2, k_wide_noadd, (uint64_t *)u, 0x12345u);
    // k_ratio<NW, NL, ND>: thread-ops per chain-iteration = 2 NW (IMAD.WIDE + its XOR) + NL + ND, CH/2 chains
    run("mix W1 (IMAD.WIDE + LOP3 xor)", 1, k_ratio<1, 0, 0>, d, (const double *)ab, 0x12345u, 7u);
    run("mix D1 (DFMA reg)", 0.5, k_ratio<0, 0, 1>, d, (const double *)ab, 0x12345u, 7u);
    run("mix W1 D1 (3 ops)", 1.5, k_ratio<1, 0, 1>, d, (const double *)ab, 0x12345u, 7u);
    run("mix W1 D2 (4 ops)", 2, k_ratio<1, 0, 2>, d, (const double *)ab, 0x12345u, 7u);
    run("mix W2 L2 D2 (8 ops)", 4, k_ratio<2, 2, 2>, d, (const double *)ab, 0x12345u, 7u);
    run("mix W2 L0 D2 (6 ops)", 3, k_ratio<2, 0, 2>, d, (const double *)ab, 0x12345u, 7u);
    run("mix W1 L2 D2 (6 ops)", 3, k_ratio<1, 2, 2>, d, (const double *)ab, 0x12345u, 7u);
    // k_ops<NW, NH, NI, NL, ND, NU>: per_iter = (ops per chain-iteration) / 2; the true
    // SASS mix of each loop is read back with tools/sass_pipes.py
#define OPS(nw, nh, ni, nl, nd, nu) \
    run("ops W" #nw " H" #nh " I" #ni " L" #nl " D" #nd " U" #nu, (nw + nh + ni + nl + nd + nu) / 2.0, \
        k_ops<nw, nh, ni, nl, nd, nu>, d, (const double *)ab, 0x12345u, 7u, 1.0000001, 1e-9)
    OPS(0, 1, 0, 0, 1, 0);
    OPS(0, 1, 1, 0, 2, 0);
    OPS(0, 0, 1, 0, 1, 0);
    OPS(0, 0, 0, 1, 1, 0);
    OPS(1, 0, 0, 0, 0, 1);
    OPS(1, 0, 0, 0, 0, 2);
    OPS(0, 1, 1, 0, 0, 2);
    OPS(0, 0, 0, 0, 0, 1);
    OPS(0, 1, 0, 0, 0, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("# %s\n", cudaGetErrorString(e));
    return 0;
}
