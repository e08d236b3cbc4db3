// e2e_probe.cu -- measurement tool (not product code): the c2 e2e call (pinned host X through
// cgx_countgauss_apply_dense) against its parts, timed on the host: a bare pinned H2D of the
// same bytes, the stage-1 call on host X, and the apply on device X.
// Build: nvcc -o e2e_probe e2e_probe.cu -I../../include -L../../paper_1606_05732_b200 -lcgx
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

#include "cgx.h"

static double ms_since(std::chrono::steady_clock::time_point a) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
}
#define CK(x) do { int rc_ = (x); if (rc_) { printf("%s -> %d: %s\n", #x, rc_, cgx_last_error()); return 1; } } while (0)

int main() {
    const int64_t n = 1 << 24, d = 32, B = 65536, m = 64;
    cgx_ctx* ctx;
    CK(cgx_init(0, &ctx));
    cgx_xform* xf;
    CK(cgx_countgauss_new(ctx, 12345, m, B, n, &xf));
    const size_t bytes = sizeof(float) * n * d;
    float *xh, *xd;
    double *sx, *zd, zh[64 * 32];
    cudaMallocHost(&xh, bytes);
    cudaMalloc(&xd, bytes);
    cudaMalloc(&sx, sizeof(double) * B * d);
    cudaMalloc(&zd, sizeof(double) * m * d);
    CK(cgx_gen_dense_normal(ctx, 7, 0, n, d, CGX_F32, CGX_ROW_MAJOR, xd, nullptr));
    cudaDeviceSynchronize();
    cudaMemcpy(xh, xd, bytes, cudaMemcpyDeviceToHost);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int rep = 0; rep < 3; ++rep) {
        auto t = std::chrono::steady_clock::now();
        cudaMemcpyAsync(xd, xh, bytes, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
        const double h2da = ms_since(t);
        t = std::chrono::steady_clock::now();
        CK(cgx_memcpy(ctx, xd, xh, bytes, nullptr));
        const double h2dc = ms_since(t);
        t = std::chrono::steady_clock::now();
        CK(cgx_memcpy(ctx, xd, xh, bytes, st));
        const double h2dc2 = ms_since(t);
        printf("app async H2D %.2f ms | cgx_memcpy ctx stream %.2f ms | cgx_memcpy app stream %.2f ms\n", h2da, h2dc, h2dc2);
        {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, st);
            t = std::chrono::steady_clock::now();
            CK(cgx_countsketch_apply_dense(ctx, xf, xh, CGX_F32, CGX_ROW_MAJOR, d, n, d, CGX_MEM_HOST, sx, CGX_ROW_MAJOR,
                                           CGX_MEM_DEVICE, st));
            const double issue = ms_since(t);
            cudaEventRecord(e1, st);
            cudaStreamSynchronize(st);
            const double wall = ms_since(t);
            float dev = 0;
            cudaEventElapsedTime(&dev, e0, e1);
            printf("stage 1 on host X, app stream: call returns after %.2f ms, done at %.2f ms, device span %.2f ms\n", issue,
                   wall, dev);
            double sk = 0, sk2 = 0;
            int64_t nl = 0;
            CK(cgx_profile_enable(ctx, 1));
            CK(cgx_countsketch_apply_dense(ctx, xf, xh, CGX_F32, CGX_ROW_MAJOR, d, n, d, CGX_MEM_HOST, sx, CGX_ROW_MAJOR,
                                           CGX_MEM_DEVICE, st));
            CK(cgx_profile_read(ctx, 0, &sk, &nl));
            CK(cgx_countsketch_apply_dense(ctx, xf, xd, CGX_F32, CGX_ROW_MAJOR, d, n, d, CGX_MEM_DEVICE, sx, CGX_ROW_MAJOR,
                                           CGX_MEM_DEVICE, st));
            CK(cgx_profile_read(ctx, 0, &sk2, &nl));
            CK(cgx_profile_enable(ctx, 0));
            printf("sketch kernel: after host staging %.3f ms, on device X %.3f ms\n", sk, sk2);
        }
        t = std::chrono::steady_clock::now();
        cudaMemcpy(xd, xh, bytes, cudaMemcpyHostToDevice);
        const double h2d = ms_since(t);
        t = std::chrono::steady_clock::now();
        CK(cgx_countsketch_apply_dense(ctx, xf, xh, CGX_F32, CGX_ROW_MAJOR, d, n, d, CGX_MEM_HOST, sx, CGX_ROW_MAJOR,
                                       CGX_MEM_DEVICE, nullptr));
        cudaDeviceSynchronize();
        const double s1 = ms_since(t);
        t = std::chrono::steady_clock::now();
        CK(cgx_countgauss_apply_dense(ctx, xf, xh, CGX_F32, CGX_ROW_MAJOR, d, n, d, CGX_MEM_HOST, zh, CGX_MEM_HOST,
                                      nullptr));
        const double e2e = ms_since(t);
        t = std::chrono::steady_clock::now();
        CK(cgx_countgauss_apply_dense(ctx, xf, xd, CGX_F32, CGX_ROW_MAJOR, d, n, d, CGX_MEM_DEVICE, zh, CGX_MEM_HOST,
                                      nullptr));
        const double dev = ms_since(t);
        printf("bare H2D %.2f ms | stage 1 on host X %.2f ms | apply host X %.2f ms | apply device X %.2f ms\n", h2d, s1,
               e2e, dev);
    }
    return 0;
}
