// Measurement helper (not product code): throughput of random record writes -- thread i
// writes an R-byte record to slot (i * odd) mod n (a permutation of n = 2^26 slots), as a
// bucket-ordering scatter of CSR rows would.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int R>
__global__ void scatter(uint4* __restrict__ rec, int64_t n, uint64_t mul) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = (int64_t)(((uint64_t)i * mul) & (uint64_t)(n - 1));
        uint4* p = rec + k * (R / 16);
#pragma unroll
        for (int q = 0; q < R / 16; ++q) p[q] = make_uint4((uint32_t)i, (uint32_t)q, 1u, 2u);
    }
}
template <int R>
__global__ void seqwrite(uint4* __restrict__ rec, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * (R / 16); i += (int64_t)gridDim.x * blockDim.x)
        rec[i] = make_uint4((uint32_t)i, 0u, 1u, 2u);
}

int main() {
    const int64_t n = 1ll << 26;
    uint4* rec;
    cudaMalloc(&rec, (size_t)n * 64);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch, double bytes) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        printf("%-28s %.3f ms  %.1f G records/s  %.0f GB/s (%s)\n", name, ms, n / ms / 1e6, bytes / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    const int blocks = 148 * 8;
    run("random 16 B records", [&] { scatter<16><<<blocks, 256>>>(rec, n, 0x9E3779B97F4A7C15ull | 1); }, n * 16.0);
    run("random 32 B records", [&] { scatter<32><<<blocks, 256>>>(rec, n, 0x9E3779B97F4A7C15ull | 1); }, n * 32.0);
    run("random 64 B records", [&] { scatter<64><<<blocks, 256>>>(rec, n, 0x9E3779B97F4A7C15ull | 1); }, n * 64.0);
    run("sequential 64 B records", [&] { seqwrite<64><<<blocks, 256>>>(rec, n); }, n * 64.0);
    return 0;
}
