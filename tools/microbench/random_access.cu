// random_access.cu -- measurement tool (not product code): the rate of independent random
// DRAM accesses on this B200 -- the ceiling of a CSR gather whose rows cost three random
// reads each (row offsets, columns, values).  Each thread issues U independent 4 B loads
// (L1::no_allocate, L2::64B: one 64 B DRAM access each) at random 32 B-aligned positions of
// a `gb`-GB buffer (a power of two), then consumes them.  Prints loads/s and the implied 64 B-access GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o random_access random_access.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <int U>
__global__ void probe(const uint32_t* __restrict__ x, uint64_t nsect, int64_t rounds, uint32_t* out) {
    uint32_t acc = 0;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t r = 0; r < rounds; ++r) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t* p = x + (mix((uint64_t)(tid * rounds + r) * U + u) & (nsect - 1)) * 8;
            asm volatile("ld.global.L1::no_allocate.L2::64B.u32 %0, [%1];" : "=r"(v[u]) : "l"(p));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
    const int64_t gb = argc > 1 ? atoll(argv[1]) : 8;
    const int64_t bytes = gb << 30;
    const uint64_t nsect = (uint64_t)bytes / 32;
    uint32_t *x, *out;
    if (cudaMalloc(&x, bytes) != cudaSuccess) return 1;
    cudaMalloc(&out, 4);
    cudaMemset(x, 0, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int blocks_per_sm : {4, 8, 16}) {
        const int blocks = 148 * blocks_per_sm, threads = 256;
        const int64_t rounds = 64;
        constexpr int U = 8;
        const double loads = (double)blocks * threads * rounds * U;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            probe<U><<<blocks, threads>>>(x, nsect, rounds, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2)
                printf("buffer %lld GB, %d CTAs/SM x 256 thr x %d in flight: %.2f G random loads/s (%.0f GB/s of 64 B accesses)\n",
                       (long long)gb, blocks_per_sm, U, loads / ms / 1e6, loads * 64 / ms / 1e6);
        }
    }
    return 0;
}
