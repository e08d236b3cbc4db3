// fp64_peak.cu -- measurement tool (not product code): B200 FP64 throughput of
//   (a) warp-level DMMA  mma.sync.m8n8k4.f64  (the only f64 tensor path on sm_100a), and
//   (b) plain DFMA,
// each with 8 independent accumulator chains per warp, all SMs, to pin the roofline
// denominators for the Gaussian GEMM stage.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x + i;
    const double a = 1.0000001, b = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {4, 8, 16, 32}) {
        const int blocks = sms * 2, threads = warps * 16;  // warps/SM = warps
        dmma_loop<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dmma_loop<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * threads / 32.0);
        printf("DMMA m8n8k4: %2d warps/SM  %8.3f ms  %7.2f TFLOP/s\n", warps, ms, flops / ms / 1e9);
    }
    for (int warps : {8, 16, 32, 64}) {
        const int blocks = sms * 2, threads = warps * 16;
        dfma_loop<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8.0 * iters * blocks * threads;
        printf("DFMA        : %2d warps/SM  %8.3f ms  %7.2f TFLOP/s\n", warps, ms, flops / ms / 1e9);
    }
    return 0;
}
