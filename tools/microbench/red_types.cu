// red_types.cu -- measurement tool (not product code): fire-and-forget L2 reduction rate by
// operand type (f64 / u64 / f32 / u32), random addresses in an L2-resident 8 MB region --
// would a fixed-point (integer) S.X accumulate add faster than RED.ADD.F64?
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
template <int T>
__global__ void red(int64_t n, uint64_t words, void* acc) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix((uint64_t)e);
        const uint64_t w = h % words;
        if (T == 0) asm volatile("red.global.add.f64 [%0], %1;" ::"l"((double*)acc + w), "d"(1.0) : "memory");
        if (T == 1) asm volatile("red.global.add.u64 [%0], %1;" ::"l"((unsigned long long*)acc + w), "l"(h) : "memory");
        if (T == 2) asm volatile("red.global.add.f32 [%0], %1;" ::"l"((float*)acc + 2 * w), "f"(1.0f) : "memory");
        if (T == 3) asm volatile("red.global.add.u32 [%0], %1;" ::"l"((unsigned*)acc + 2 * w), "r"((unsigned)h) : "memory");
    }
}
int main() {
    const int64_t n = 172 << 20;
    void* acc;
    cudaMalloc(&acc, 64 << 20);
    cudaMemset(acc, 0, 64 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[4] = {"f64", "u64", "f32", "u32"};
    for (uint64_t mb : {8, 32}) {
        const uint64_t words = (mb << 20) / 8;
        for (int rep = 0; rep < 2; ++rep)
            for (int t = 0; t < 4; ++t) {
                cudaEventRecord(a);
                switch (t) {
                    case 0: red<0><<<148 * 8, 256>>>(n, words, acc); break;
                    case 1: red<1><<<148 * 8, 256>>>(n, words, acc); break;
                    case 2: red<2><<<148 * 8, 256>>>(n, words, acc); break;
                    case 3: red<3><<<148 * 8, 256>>>(n, words, acc); break;
                }
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep) printf("%s region %lu MB: %.3f ms  %.1f G/s\n", names[t], mb, ms, n / ms / 1e6);
            }
    }
    return 0;
}
