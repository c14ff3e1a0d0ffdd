// Launch-to-result latency on one B200 (host wall clock, median of 2000):
//   empty kernel + cudaStreamSynchronize; a one-thread kernel writing 4 words to mapped
//   pinned memory + sync; the same reading 6 args from mapped memory first; and the
//   same with args by value polling a completion flag instead of synchronising.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_latency probe_latency.cu
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_empty() {}
__global__ void k_write(uint32_t *out, uint4 v) { out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w; }
__global__ void k_readwrite(const uint32_t *in, uint32_t *out) {
    uint32_t a = in[0], b = in[1], c = in[2], d = in[3], e = in[4], f = in[5];
    out[0] = a ^ e; out[1] = b ^ f; out[2] = c; out[3] = d;
}
__global__ void k_write_flag(uint32_t *out, uint4 v, volatile uint32_t *flag, uint32_t seq) {
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
    __threadfence_system();
    *flag = seq;
}

template <typename F>
static double med_us(F f, int n = 2000) {
    std::vector<double> t;
    for (int i = 0; i < 50; i++) f();
    for (int i = 0; i < n; i++) {
        auto a = std::chrono::steady_clock::now();
        f();
        auto b = std::chrono::steady_clock::now();
        t.push_back(std::chrono::duration<double, std::micro>(b - a).count());
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    uint32_t *h, *d;
    cudaHostAlloc((void **)&h, 4096, cudaHostAllocMapped);
    cudaHostGetDevicePointer((void **)&d, h, 0);
    volatile uint32_t *hflag = h + 512;
    uint32_t *dflag = d + 512;
    uint32_t seq = 0;
    printf("{\"empty+sync_us\": %.2f, ", med_us([&] { k_empty<<<1, 1, 0, s>>>(); cudaStreamSynchronize(s); }));
    printf("\"write_mapped+sync_us\": %.2f, ", med_us([&] { k_write<<<1, 1, 0, s>>>(d, make_uint4(1, 2, 3, 4)); cudaStreamSynchronize(s); }));
    printf("\"read6_write_mapped+sync_us\": %.2f, ", med_us([&] { k_readwrite<<<1, 1, 0, s>>>(d + 64, d); cudaStreamSynchronize(s); }));
    printf("\"write_mapped+poll_flag_us\": %.2f, ", med_us([&] {
        ++seq;
        k_write_flag<<<1, 1, 0, s>>>(d, make_uint4(1, 2, 3, seq), dflag, seq);
        while (*hflag != seq) {
        }
    }));
    printf("\"launch_only_us\": %.2f}\n", med_us([&] { k_empty<<<1, 1, 0, s>>>(); }));
    cudaStreamSynchronize(s);
    return 0;
}
