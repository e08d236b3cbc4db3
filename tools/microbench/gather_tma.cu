// gather_tma.cu -- measurement tool (not product code): can the TMA engine fetch random
// 128 B rows of a 2 GB matrix faster than SM loads (gather_bw.cu, ~5.6-5.9 TB/s; the c2
// sketch's cp.async ring reaches 5.6 TB/s)?  Each CTA streams its share of a random row
// permutation into a shared-memory ring with one cp.async.bulk (1-D TMA) per 128 B row, N
// rows per ring slot completing on one mbarrier, and folds the slot into a checksum.
// Build: make -C tools/microbench gather_tma
#include <cstdint>
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("{.reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(sa(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void wait_phase(uint64_t* b, unsigned ph) {
    asm volatile("{.reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=;}" ::"r"(sa(b)),
                 "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
                 "l"(src), "r"(bytes), "r"(sa(b))
                 : "memory");
}

// one warp per CTA-slot producer: lane k issues row k of a 32-row group; S slots in flight
template <int S>
__global__ void __launch_bounds__(128) tma_gather(const float* __restrict__ x, const uint32_t* __restrict__ perm,
                                                  int64_t nrows, float* out) {
    extern __shared__ __align__(128) float ring[];  // S slots x 4 warps x 32 rows x 32 floats
    __shared__ uint64_t bar[4][S];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bar[w][s], 1);
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int64_t warp = (int64_t)blockIdx.x * 4 + w, nw = (int64_t)gridDim.x * 4;
    const int64_t ngroups = nrows / 32;
    float acc = 0.f;
    float* mine = ring + (size_t)w * S * 1024;
    int64_t g = warp;
    // prologue: S groups in flight
    for (int s = 0; s < S && g + (int64_t)s * nw < ngroups; ++s) {
        const int64_t gg = g + (int64_t)s * nw;
        if (lane == 0) expect_tx(&bar[w][s], 32 * 128);
        __syncwarp();
        const uint32_t r = perm[gg * 32 + lane];
        bulk(mine + s * 1024 + lane * 32, x + (int64_t)r * 32, 128, &bar[w][s]);
    }
    unsigned phase[S] = {};
    for (int64_t k = 0;; ++k) {
        const int s = (int)(k % S);
        const int64_t gg = g + k * nw;
        if (gg >= ngroups) break;
        wait_phase(&bar[w][s], phase[s]);
        phase[s] ^= 1u;
#pragma unroll 4
        for (int rr = 0; rr < 32; ++rr) acc += mine[s * 1024 + rr * 32 + lane];
        __syncwarp();
        const int64_t nx = gg + (int64_t)S * nw;
        if (nx < ngroups) {
            if (lane == 0) expect_tx(&bar[w][s], 32 * 128);
            __syncwarp();
            const uint32_t r = perm[nx * 32 + lane];
            bulk(mine + s * 1024 + lane * 32, x + (int64_t)r * 32, 128, &bar[w][s]);
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    const int64_t nrows = (int64_t)1 << 24;  // c2: 2^24 rows x 128 B = 2 GB
    float *x, *out;
    uint32_t* perm;
    cudaMalloc(&x, (size_t)nrows * 128);
    cudaMalloc(&out, 4);
    cudaMalloc(&perm, 4 * nrows);
    cudaMemset(x, 0, (size_t)nrows * 128);
    std::vector<uint32_t> h(nrows);
    for (int64_t i = 0; i < nrows; ++i) h[i] = (uint32_t)i;
    uint64_t st = 88172645463325252ull;
    for (int64_t i = nrows - 1; i > 0; --i) {
        st ^= st << 13;
        st ^= st >> 7;
        st ^= st << 17;
        std::swap(h[i], h[st % (uint64_t)(i + 1)]);
    }
    cudaMemcpy(perm, h.data(), 4 * nrows, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](auto kern, int S, int ctas_per_sm) {
        const size_t smem = (size_t)S * 4 * 1024 * 4;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            kern<<<148 * ctas_per_sm, 128, smem>>>(x, perm, nrows, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        printf("TMA rows: %d slots x 4 warps, %d CTAs/SM: %.3f ms = %.2f TB/s (%s)\n", S, ctas_per_sm, ms,
               nrows * 128.0 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    for (int c : {2, 4, 8}) {
        run(tma_gather<2>, 2, c);
        run(tma_gather<4>, 4, c);
    }
    run(tma_gather<8>, 8, 2);
    run(tma_gather<8>, 8, 3);
    return 0;
}
