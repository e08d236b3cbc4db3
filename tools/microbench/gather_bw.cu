// gather_bw.cu -- measurement tool (not product code): HBM bandwidth of the access
// patterns the dense sketch can use, on this B200.
//   seq      : each warp streams contiguous 128 B rows
//   rand     : warps read rows in a uniformly random order over the whole buffer
//   window W : random order, but all concurrently-processed rows lie in a W-row window
//              (windows processed in order) -- the row-chunked gather
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U, typename A = float>
__global__ void gather(const float* __restrict__ x, const uint32_t* __restrict__ perm, int64_t nrows, int ld,
                       float* out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    A acc = 0.f;
    for (int64_t base = warp * 32; base < nrows; base += nwarps * 32) {
        uint32_t p = perm[base + lane];
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint32_t r = __shfl_sync(0xffffffff, p, u);
            v[u] = __ldcs(x + (int64_t)r * ld + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += (A)v[u];
        if (U < 32) {
#pragma unroll
            for (int u = U; u < 32; u += U) {
                float w[U];
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    uint32_t r = __shfl_sync(0xffffffff, p, u + k);
                    w[k] = __ldcs(x + (int64_t)r * ld + lane);
                }
#pragma unroll
                for (int k = 0; k < U; ++k) acc += (A)w[k];
            }
        }
    }
    if (acc == (A)12345.f) out[0] = (float)acc;
}

// Same gather, but each warp walks its own contiguous stretch of perm (the CountSketch
// kernel's assignment: a warp owns consecutive buckets) instead of a grid stride.
__global__ void gather_contig(const float* __restrict__ x, const uint32_t* __restrict__ perm, int64_t nrows, int ld,
                              float* out, int64_t per_warp) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    double acc = 0.0;
    const int64_t b = warp * per_warp, e = min(nrows, b + per_warp);
    for (int64_t base = b; base < e; base += 32) {
        uint32_t p = perm[base + lane];
        float v[16];
#pragma unroll
        for (int h = 0; h < 32; h += 16) {
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = __ldcs(x + (int64_t)__shfl_sync(0xffffffff, p, h + u) * ld + lane);
#pragma unroll
            for (int u = 0; u < 16; ++u) acc += (double)v[u];
        }
    }
    if (acc == 12345.0) out[0] = (float)acc;
}

int main() {
    const int64_t nrows = 1 << 24;
    const int ld = 32;
    float* x;
    uint32_t* perm;
    float* out;
    CK(cudaMalloc(&x, nrows * ld * 4));
    CK(cudaMalloc(&perm, nrows * 4));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemset(x, 0, nrows * ld * 4));
    std::vector<uint32_t> h(nrows);
    std::mt19937_64 g(1);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int variant = 0;
    auto launch = [&](int blocks, int threads) {
        if (variant == 0) gather<16><<<blocks, threads>>>(x, perm, nrows, ld, out);
        else if (variant == 1) gather<16, double><<<blocks, threads>>>(x, perm, nrows, ld, out);
        else if (variant == 2) gather<32, double><<<blocks, threads>>>(x, perm, nrows, ld, out);
        else gather<32, float><<<blocks, threads>>>(x, perm, nrows, ld, out);
    };
    auto run = [&](const char* name, int blocks, int threads) {
        CK(cudaMemcpy(perm, h.data(), nrows * 4, cudaMemcpyHostToDevice));
        for (int it = 0; it < 3; ++it) launch(blocks, threads);
        cudaEventRecord(a);
        const int reps = 10;
        for (int it = 0; it < reps; ++it) launch(blocks, threads);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        double bytes = (double)nrows * ld * 4 + nrows * 4.0;
        printf("v%d %-28s blocks=%6d thr=%4d  %8.3f ms  %8.1f GB/s\n", variant, name, blocks, threads, ms, bytes / ms / 1e6);
        return 0;
    };
    for (int64_t i = 0; i < nrows; ++i) h[i] = (uint32_t)i;
    for (int bl : {sms * 4, sms * 8, sms * 16}) run("seq", bl, 256);
    std::shuffle(h.begin(), h.end(), g);
    for (variant = 0; variant < 4; ++variant)
        for (int bl : {sms * 2, sms * 4, sms * 8, sms * 16}) run("rand(2GB)", bl, 256);
    variant = 0;
    // bucket-sorted order: rows grouped by a random bucket in [0, 65536), ascending within
    // a bucket -- the order the CountSketch gather walks
    {
        std::vector<uint32_t> key(nrows);
        for (int64_t i = 0; i < nrows; ++i) key[i] = (uint32_t)(g() & 0xffff);
        for (int64_t i = 0; i < nrows; ++i) h[i] = (uint32_t)i;
        std::stable_sort(h.begin(), h.end(), [&](uint32_t a, uint32_t b) { return key[a] < key[b]; });
        for (variant = 0; variant < 4; ++variant)
            for (int bl : {sms * 4, sms * 16}) run("bucket-sorted", bl, 256);
        variant = 0;
        CK(cudaMemcpy(perm, h.data(), nrows * 4, cudaMemcpyHostToDevice));
        for (int64_t per : {1024, 4096, 16384}) {
            const int64_t warps = (nrows + per - 1) / per;
            const int blocks = (int)((warps + 7) / 8);
            for (int it = 0; it < 3; ++it) gather_contig<<<blocks, 256>>>(x, perm, nrows, ld, out, per);
            cudaEventRecord(a);
            for (int it = 0; it < 10; ++it) gather_contig<<<blocks, 256>>>(x, perm, nrows, ld, out, per);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ms /= 10;
            printf("contig per_warp=%-6lld blocks=%6d  %8.3f ms  %8.1f GB/s\n", (long long)per, blocks, ms,
                   ((double)nrows * ld * 4 + nrows * 4.0) / ms / 1e6);
        }
    }
    for (int64_t W : {1 << 14, 1 << 16, 1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22}) {
        for (int64_t i = 0; i < nrows; ++i) h[i] = (uint32_t)i;
        for (int64_t s = 0; s < nrows; s += W) std::shuffle(h.begin() + s, h.begin() + std::min(nrows, s + W), g);
        char name[64];
        snprintf(name, sizeof name, "window %lld rows (%lld MB)", (long long)W, (long long)(W * 128 >> 20));
        run(name, sms * 8, 256);
    }
    return 0;
}
