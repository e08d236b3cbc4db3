// Measurement helper (not product code): one tcgen05.mma kind::i8 (M=128, N=64, K=32) on a
// canonical K-major no-swizzle smem image, read back through TMEM, against a CPU product --
// checks the descriptor encodings ozgemm.cu uses.   nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(const int8_t* aimg, const int8_t* bimg, int lbo, int sbo, uint32_t idesc, int* out) {
    __shared__ __align__(1024) int8_t sm[128 * 32 + 64 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < 128 * 32 + 64 * 32; i += blockDim.x) sm[i] = i < 4096 ? aimg[i] : bimg[i - 4096];
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(sa(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tm = slot;
    if (tid == 0) {
        unsigned a = sa(sm), b = sa(sm + 4096);
        uint64_t da = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
        uint64_t db = (uint64_t)((b >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
    }
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(sa(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int q = 0; q < 4; ++q) {
        int v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tm + ((uint32_t)(warp * 32) << 16) + q * 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) out[(warp * 32 + lane) * 64 + q * 16 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}


// A from TMEM (tcgen05.cp 128x256b from the canonical image), B from smem
__global__ void kts(const int8_t* aimg, const int8_t* bimg, int lbo, int sbo, uint32_t idesc, int* out) {
    __shared__ __align__(1024) int8_t sm[128 * 32 + 64 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < 128 * 32 + 64 * 32; i += blockDim.x) sm[i] = i < 4096 ? aimg[i] : bimg[i - 4096];
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tm = slot;
    if (tid == 0) {
        unsigned a = sa(sm), b = sa(sm + 4096);
        uint64_t da = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
        uint64_t db = (uint64_t)((b >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 64), "l"(da));
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tm), "r"(tm + 64), "l"(db), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
    }
    asm volatile("{\n\t.reg .pred p;\n\tW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n\t}" ::"r"(sa(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int q = 0; q < 4; ++q) {
        int v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tm + ((uint32_t)(warp * 32) << 16) + q * 16));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) out[(warp * 32 + lane) * 64 + q * 16 + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

// MMA issue rate: iters x 28 MMAs (M=128, N=64, K=32) from fixed operands; ts = A from TMEM
__global__ void krate(int ts, int iters, long long* cyc) {
    extern __shared__ __align__(1024) int8_t dsm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    int tid = threadIdx.x, warp = tid / 32;
    int8_t* sm = dsm + ((1024 - (sa(dsm) & 1023)) & 1023);
    for (int i = tid; i < 7 * 6144; i += blockDim.x) sm[i] = (int8_t)(i * 7);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tm = slot;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24);
    if (tid == 0) {
        unsigned base = sa(sm);
        auto desc = [](unsigned a) { return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)8 << 16) | ((uint64_t)16 << 32) | (1ull << 46); };
        if (ts) for (int s = 0; s < 7; ++s) asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 448 + 8 * s), "l"(desc(base + s * 4096)));
        long long t0 = clock64();
        if (ts >= 6) {  // calibration: N=256 MMAs of other kinds (bf16 K=16, e4m3 K=32, i8 K=32)
          const uint32_t id16 = (1u << 4) | (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24);
          const uint32_t id8 = (1u << 4) | (0u << 7) | (0u << 10) | (32u << 17) | (8u << 24);
          const uint32_t idi = (2u << 4) | (1u << 7) | (1u << 10) | (32u << 17) | (8u << 24);
          for (int it = 0; it < iters; ++it)
            for (int q = 0; q < 7; ++q) {
                uint64_t da = desc(base), db = desc(base + 28672);
                if (ts == 6) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(id16), "r"(1));
                else if (ts == 7) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(id8), "r"(1));
                else asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(idi), "r"(1));
            }
        } else
        if (ts >= 2) {  // stacked-N: for each A plane s, B planes t0.. as one N = 64 w operand
          const int wmax = ts - 1;  // planes per MMA (4 -> N = 256)
          for (int it = 0; it < iters; ++it)
            for (int s = 0; s < 7; ++s)
                for (int t0 = 0; t0 < 7 - s; t0 += wmax) {
                    const int w = 7 - s - t0 < wmax ? 7 - s - t0 : wmax;
                    const uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(8 * w) << 17) | (8u << 24);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                                 ::"r"(tm + (s + t0) * 64), "l"(desc(base + s * 4096)), "l"(desc(base + 28672 + t0 * 2048)), "r"(id), "r"(1));
                }
        } else
        for (int it = 0; it < iters; ++it) {
            for (int s = 0; s < 7; ++s)
                for (int t = 0; s + t < 7; ++t) {
                    uint64_t db = desc(base + 28672 + t * 2048);
                    if (ts)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                                     ::"r"(tm + (s + t) * 64), "r"(tm + 448 + 8 * s), "l"(db), "r"(idesc), "r"(1));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                                     ::"r"(tm + (s + t) * 64), "l"(desc(base + s * 4096)), "l"(db), "r"(idesc), "r"(1));
                }
            if (ts && (it & 1)) for (int s = 0; s < 7; ++s) asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 448 + 8 * s), "l"(desc(base + s * 4096)));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)));
        asm volatile("{\n\t.reg .pred p;\n\tW3:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W3;\n\t}" ::"r"(sa(&bar)));
        cyc[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static int off(int r, int kk) { return (r / 8) * 256 + (kk / 16) * 128 + (r % 8) * 16 + (kk % 16); }

int main() {
    static int8_t A[128][32], B[64][32], ai[4096], bi[2048];
    srand(1);
    for (int r = 0; r < 128; ++r) for (int kk = 0; kk < 32; ++kk) { A[r][kk] = (int8_t)(rand() % 255 - 127); ai[off(r, kk)] = A[r][kk]; }
    for (int r = 0; r < 64; ++r) for (int kk = 0; kk < 32; ++kk) { B[r][kk] = (int8_t)(rand() % 255 - 127); bi[off(r, kk)] = B[r][kk]; }
    static int ref[128][64], got[128 * 64];
    for (int i = 0; i < 128; ++i) for (int j = 0; j < 64; ++j) { int s = 0; for (int kk = 0; kk < 32; ++kk) s += A[i][kk] * B[j][kk]; ref[i][j] = s; }
    int8_t *da, *db; int* dout;
    cudaMalloc(&da, 4096); cudaMalloc(&db, 2048); cudaMalloc(&dout, sizeof(got));
    cudaMemcpy(da, ai, 4096, cudaMemcpyHostToDevice); cudaMemcpy(db, bi, 2048, cudaMemcpyHostToDevice);
    struct V { const char* name; int lbo, sbo; uint32_t idesc; } vs[] = {
        {"lbo128 sbo256 m@24", 128, 256, (2u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24)},
        {"lbo256 sbo128 m@24", 256, 128, (2u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24)},
        {"lbo128 sbo256 m@23", 128, 256, (2u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 23)},
        {"lbo256 sbo128 m@23", 256, 128, (2u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 23)},
    };
    for (auto& v : vs) {
        cudaMemset(dout, 0, sizeof(got));
        k<<<1, 128>>>(da, db, v.lbo, v.sbo, v.idesc, dout);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(got, dout, sizeof(got), cudaMemcpyDeviceToHost);
        int bad = 0; long long maxd = 0;
        for (int i = 0; i < 128; ++i) for (int j = 0; j < 64; ++j) { long long dd = llabs((long long)got[i * 64 + j] - ref[i][j]); if (dd) ++bad; if (dd > maxd) maxd = dd; }
        printf("%-22s err=%s mismatches=%d maxdiff=%lld  got[0..3]=%d %d %d %d ref=%d %d %d %d\n", v.name, cudaGetErrorString(e), bad, maxd,
               got[0], got[1], got[2], got[3], ref[0][0], ref[0][1], ref[0][2], ref[0][3]);
        if (e != cudaSuccess) return 1;
    }
    for (int sw = 0; sw < 2; ++sw) {
        int lbo = sw ? 256 : 128, sbo = sw ? 128 : 256;
        cudaMemset(dout, 0, sizeof(got));
        kts<<<1, 128>>>(da, db, lbo, sbo, vs[0].idesc, dout);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(got, dout, sizeof(got), cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 128; ++i) for (int j = 0; j < 64; ++j) if (got[i * 64 + j] != ref[i][j]) ++bad;
        printf("TS (A via tcgen05.cp) lbo%d sbo%d: err=%s mismatches=%d\n", lbo, sbo, cudaGetErrorString(e), bad);
    }
    long long* dc; cudaMalloc(&dc, 148 * 8);
    cudaFuncSetAttribute(krate, cudaFuncAttributeMaxDynamicSharedMemorySize, 7 * 6144 + 1024);
    for (int ts = 0; ts < 9; ++ts) {
        const int iters = 2000;
        krate<<<148, 128, 7 * 6144 + 1024>>>(ts, iters, dc);
        cudaError_t e = cudaDeviceSynchronize();
        long long c[148]; cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
        if (ts >= 6) { printf("calib %s N=256 M=128: %.1f cycles per MMA (ideal at nominal dense peak: bf16 131, e4m3/i8 128)\n", ts == 6 ? "bf16 K=16" : ts == 7 ? "e4m3 K=32" : "i8 K=32", c[0] / (double)(iters * 7)); continue; }
        printf("rate %s: err=%s  %.1f cycles per MMA (128x64x32 int8) on 148 SMs; ideal 32\n", ts == 0 ? "SS" : ts == 1 ? "TS" : ts == 2 ? "stack1" : ts == 3 ? "stack2" : ts == 4 ? "stack3" : "stack4", cudaGetErrorString(e), c[0] / (double)(iters * 28));
    }
    return 0;
}
