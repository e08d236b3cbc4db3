// sector_fetch.cu -- measurement tool (not product code): how many DRAM bytes does one
// random 32 B-sector load cost on this B200, per load flavour and cudaLimitMaxL2FetchGranularity?
// Each thread reads one 4 B word at a random 32 B-aligned position of a 2 GB buffer.
// Run under ncu with --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sector_fetch sector_fetch.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <int KIND>
__global__ void probe(const uint32_t* __restrict__ x, int64_t nsect, int64_t loads, uint32_t* out) {
    uint32_t acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < loads; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t* p = x + (mix(i) % nsect) * 8;
        uint32_t v;
        if (KIND == 0) asm volatile("ld.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
        else if (KIND == 1) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
        else if (KIND == 2) asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
        else if (KIND == 3) asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(v) : "l"(p));
        else asm volatile("ld.global.L1::no_allocate.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
        acc += v;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
    const int gran = argc > 1 ? atoi(argv[1]) : -1;
    if (gran >= 0) {
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        printf("cudaLimitMaxL2FetchGranularity set %d -> %s, now %zu\n", gran, cudaGetErrorString(e), got);
    }
    const int64_t bytes = 2LL << 30, nsect = bytes / 32, loads = 64LL << 20;
    uint32_t *x, *out;
    cudaMalloc(&x, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(x, 0, bytes);
    probe<0><<<148 * 8, 256>>>(x, nsect, loads, out);
    probe<1><<<148 * 8, 256>>>(x, nsect, loads, out);
    probe<2><<<148 * 8, 256>>>(x, nsect, loads, out);
    probe<3><<<148 * 8, 256>>>(x, nsect, loads, out);
    probe<4><<<148 * 8, 256>>>(x, nsect, loads, out);
    cudaDeviceSynchronize();
    printf("done: %lld loads per kernel (%lld MB of sectors requested)\n", (long long)loads, (long long)(loads * 32 >> 20));
    return 0;
}
