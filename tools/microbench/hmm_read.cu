// hmm_read.cu -- measurement tool (not product code): can a kernel read a PAGEABLE host
// array (malloc) directly -- HMM / pageable memory access -- and how fast, with the pages
// advised to stay on the CPU?  The drop-in's full-fp64 path moves every byte through host
// memory three times (pageable read, pinned write, DMA read); a direct read would move it once.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__global__ void sum_kernel(const double4* __restrict__ p, size_t n4, double* out) {
    double s = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        const double4 v = p[i];
        s += v.x + v.y + v.z + v.w;
    }
    atomicAdd(out, s);
}

int main() {
    int dev = 0, pma = 0, pmahpt = 0, cma = 0;
    cudaDeviceGetAttribute(&pma, cudaDevAttrPageableMemoryAccess, dev);
    cudaDeviceGetAttribute(&pmahpt, cudaDevAttrPageableMemoryAccessUsesHostPageTables, dev);
    cudaDeviceGetAttribute(&cma, cudaDevAttrConcurrentManagedAccess, dev);
    printf("pageableMemoryAccess %d, usesHostPageTables %d, concurrentManagedAccess %d\n", pma, pmahpt, cma);
    if (!pma) return 0;
    const size_t bytes = (size_t)2 << 30;
    double* h = (double*)malloc(bytes);
    for (size_t i = 0; i < bytes / 8; ++i) h[i] = 1.0;
    double* out;
    cudaMalloc(&out, 8);
    for (int advise = 0; advise < 2; ++advise) {
        if (advise) {
            cudaMemLocation cpu{};
            cpu.type = cudaMemLocationTypeHost;
            cpu.id = 0;
            cudaMemAdvise_v2(h, bytes, cudaMemAdviseSetPreferredLocation, cpu);
            cudaMemLocation g{};
            g.type = cudaMemLocationTypeDevice;
            g.id = 0;
            cudaMemAdvise_v2(h, bytes, cudaMemAdviseSetAccessedBy, g);
            printf("advise: %s\n", cudaGetErrorString(cudaGetLastError()));
        }
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(out, 0, 8);
            cudaDeviceSynchronize();
            auto t0 = std::chrono::steady_clock::now();
            sum_kernel<<<148 * 8, 256>>>((const double4*)h, bytes / 32, out);
            cudaError_t e = cudaDeviceSynchronize();
            const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            double r = 0;
            cudaMemcpy(&r, out, 8, cudaMemcpyDeviceToHost);
            printf("advise %d rep %d: %s, %.1f GB/s (%.1f ms), sum %.0f (want %.0f)\n", advise, rep, cudaGetErrorString(e),
                   bytes / t / 1e9, t * 1e3, r, (double)(bytes / 8));
        }
    }
    return 0;
}
