// occupy.cu -- measurement tool (not product code): pins K SMs with one spinning CTA each
// (all of an SM's shared memory, so nothing else can land there) until the host clears a
// flag, so a kernel launched meanwhile runs on the remaining 148-K SMs.  Used by
// tools/prof_sm_partition.py to ask whether the CSR gather is SM-bound or DRAM-bound.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o occupy.so occupy.cu
#include <cuda_runtime.h>

__global__ void spin(volatile int* flag, int* started) {
    extern __shared__ int s[];
    if (threadIdx.x == 0) {
        s[0] = 1;
        atomicAdd(started, 1);
        while (*flag) __nanosleep(1000);
    }
}

extern "C" int occupy(int k, int* flag_dev, int* started_dev, void* stream) {
    const int smem = 227 * 1024;
    cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    spin<<<k, 32, smem, (cudaStream_t)stream>>>(flag_dev, started_dev);
    return (int)cudaGetLastError();
}
