// gather_l2.cu -- measurement tool (not product code): can an explicit L2 prefetch turn the
// bucket-order random row gather into a DRAM stream?  X (2^24 x 128 B rows) is processed in
// windows of W rows, windows in order, rows in random order inside a window (the order a
// region-major CountSketch permutation gives).  One launch per window; at the start of
// window w every CTA issues cp.async.bulk.prefetch.L2 for its slice of window w+PD.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_l2 gather_l2.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void window_gather(const float* __restrict__ x, const uint32_t* __restrict__ perm, int64_t r0, int64_t w,
                              int ld, float* out, const char* pf, int64_t pf_bytes) {
    if (pf && threadIdx.x == 0 && pf_bytes > 0) {
        const int64_t slice = (pf_bytes / gridDim.x + 15) / 16 * 16;
        const int64_t a = (int64_t)blockIdx.x * slice;
        if (a < pf_bytes) {
            const uint32_t sz = (uint32_t)min(slice, pf_bytes - a);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf + a), "r"(sz) : "memory");
        }
    }
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float acc = 0.f;
    for (int64_t base = r0 + warp * 32; base < r0 + w; base += nwarps * 32) {
        const uint32_t p = perm[base + lane];
        float v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] = __ldcs(x + (int64_t)__shfl_sync(0xffffffff, p, u) * ld + lane);
#pragma unroll
        for (int u = 0; u < 32; ++u) acc += v[u];
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    const int64_t nrows = 1 << 24;
    const int ld = 32;
    float *x, *out;
    uint32_t* perm;
    cudaMalloc(&x, nrows * ld * 4);
    cudaMalloc(&perm, nrows * 4);
    cudaMalloc(&out, 4);
    cudaMemset(x, 0, nrows * ld * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::vector<uint32_t> h(nrows);
    std::mt19937_64 g(1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int64_t W : {1 << 16, 1 << 17, 1 << 18, 1 << 19}) {
        for (int64_t i = 0; i < nrows; ++i) h[i] = (uint32_t)i;
        for (int64_t s = 0; s < nrows; s += W) std::shuffle(h.begin() + s, h.begin() + std::min(nrows, s + W), g);
        cudaMemcpy(perm, h.data(), nrows * 4, cudaMemcpyHostToDevice);
        for (int pd : {0, 1, 2, 3}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                for (int64_t r0 = 0; r0 < nrows; r0 += W) {
                    const int64_t nxt = r0 + pd * W;
                    const char* pf = (pd > 0 && nxt < nrows) ? (const char*)(x + nxt * ld) : nullptr;
                    const int64_t pfb = pf ? std::min(W, nrows - nxt) * ld * 4 : 0;
                    window_gather<<<sms * 8, 256>>>(x, perm, r0, std::min(W, nrows - r0), ld, out, pf, pfb);
                }
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep == 1)
                    printf("window %7lld rows (%4lld MB) prefetch distance %d: %.3f ms  %.1f GB/s\n", (long long)W,
                           (long long)(W * 128 >> 20), pd, ms, nrows * 132.0 / ms / 1e6);
            }
        }
    }
    return 0;
}
