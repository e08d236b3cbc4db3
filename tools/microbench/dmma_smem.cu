// dmma_smem.cu -- measurement tool (not product code): DMMA throughput when the m8n8k4
// fragments come from shared memory the way gemm_dmma loads them (4 A + 4 B LDS.64 per
// 16 DMMAs), with no global traffic and no barriers -- separates the operand-feed cost
// from the cp.async pipeline cost in the stage-2 GEMM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_smem dmma_smem.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int FM, int FN>
__global__ void __launch_bounds__(256) kern(double* out, int iters) {
    constexpr int LD = 68;
    __shared__ double As[2 * 16 * LD], Bs[2 * 16 * LD];
    for (int e = threadIdx.x; e < 2 * 16 * LD; e += blockDim.x) {
        As[e] = 1e-3 * e;
        Bs[e] = 1.0 + 1e-4 * e;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* as = As + (warp & 1) * 32 + (lane >> 2);
    const double* bs = Bs + (warp >> 1 & 1) * 32 + (lane >> 2);
    double acc[FM][FN][2] = {};
    for (int it = 0; it < iters; ++it) {
        const int st = (it & 1) * 16 * LD;  // rotating stage: the loads cannot be hoisted
#pragma unroll
        for (int k4 = 0; k4 < 16; k4 += 4) {
            double a[FM], b[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) a[i] = as[st + (k4 + (lane & 3)) * LD + i * 8];
#pragma unroll
            for (int j = 0; j < FN; ++j) b[j] = bs[st + (k4 + (lane & 3)) * LD + j * 8];
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) s += acc[i][j][0] + acc[i][j][1];
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
    const int iters = 2000;
    for (int bps : {1, 2}) {
        const int blocks = sms * bps;
        kern<4, 4><<<blocks, 256>>>(out, 10);
        cudaEventRecord(e0);
        kern<4, 4><<<blocks, 256>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * 8 * 8 * 4 * 16 * 4.0 * iters * blocks * 8;
        printf("smem-fed DMMA 4x4 fragments, %d CTA(s)/SM: %.2f TFLOP/s\n", bps, flops / ms / 1e9);
    }
    return 0;
}
