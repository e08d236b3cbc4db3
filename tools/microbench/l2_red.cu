// l2_red.cu -- measurement tool (not product code): throughput of fire-and-forget fp64
// atomic adds (RED.E.ADD.F64) at random addresses of a region of R MB, from every SM --
// the accumulate step of a bucket-range-partitioned CSR sketch whose S.X slice is meant to
// stay in L2.  Also: the same with u64 adds, and with a streaming 8 B/record read feeding
// the adds (records generated here, read from a 1.37 GB buffer as the real pass would).
// Build: make -C tools/microbench l2_red
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// n atomics, address = hash(e) mod words
__global__ void red_f64(double* acc, uint64_t words, int64_t n) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix((uint64_t)e);
        atomicAdd(acc + (h % words), (double)(h & 0xff));
    }
}

__global__ void red_u64(unsigned long long* acc, uint64_t words, int64_t n) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix((uint64_t)e);
        atomicAdd(acc + (h % words), (unsigned long long)(h & 0xff));
    }
}

// records: (index u32, value f32) streamed from HBM, RED into acc
__global__ void red_stream(const uint2* __restrict__ rec, double* acc, int64_t n) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const uint2 r = __ldcs(rec + e);
        atomicAdd(acc + r.x, (double)__uint_as_float(r.y));
    }
}

__global__ void make_records(uint2* rec, uint64_t words, int64_t n) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix((uint64_t)e);
        rec[e] = make_uint2((uint32_t)(h % words), __float_as_uint(1.0f + (float)(h >> 60)));
    }
}

int main() {
    const int64_t n = 171798691;  // c3's nnz
    double* acc;
    cudaMalloc(&acc, (size_t)1 << 30);
    uint2* rec;
    cudaMalloc(&rec, sizeof(uint2) * n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int64_t mb : {4, 16, 32, 48, 64, 96, 128, 512}) {
        const uint64_t words = (uint64_t)mb << 17;
        for (int cps : {4, 8}) {
            const int grid = 148 * cps;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(acc, 0, words * 8);
                cudaEventRecord(a);
                red_f64<<<grid, 256>>>(acc, words, n);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms, a, b);
            }
            printf("f64 RED  region %4lld MB, %d CTA/SM: %.3f ms = %.1f G atomics/s\n", (long long)mb, cps, ms,
                   n / ms / 1e6);
        }
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(acc, 0, words * 8);
            cudaEventRecord(a);
            red_u64<<<148 * 8, 256>>>((unsigned long long*)acc, words, n);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        printf("u64 RED  region %4lld MB: %.3f ms = %.1f G atomics/s\n", (long long)mb, ms, n / ms / 1e6);
        make_records<<<148 * 8, 256>>>(rec, words, n);
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(acc, 0, words * 8);
            cudaEventRecord(a);
            red_stream<<<148 * 8, 256>>>(rec, acc, n);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        printf("stream+RED region %4lld MB: %.3f ms = %.1f G atomics/s (%.0f GB/s of records)\n", (long long)mb, ms,
               n / ms / 1e6, n * 8.0 / ms / 1e6);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
