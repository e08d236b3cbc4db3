// dgemm.cu -- stage 2 for large m x d: Z = G . (S.X) as G super-chunks + a pipelined
// FP64 tensor-core GEMM.
//
// When Z is large (config 3: 128 x 256, config 5: 256 x 512) a CTA cannot hold a full
// row of Z tiles, so generating G inside the GEMM would regenerate every G(r, c) once per
// column tile.  Instead G is produced in super-chunks of S bucket-columns (m x S fp64,
// sized to stay resident in L2, ~48 MB) by the high-occupancy generator (53 G normals/s
// on B200), and each chunk is consumed right away by a cp.async-pipelined DMMA GEMM
// (mma.sync.m8n8k4.f64 -- the only FP64 tensor-core path on sm_100a, 37.2 TFLOP/s
// measured by tools/microbench/fp64_peak.cu).  G never exists in full anywhere: at most
// one chunk, in L2.
//
// GEMM: CTA tile BM x BN, BK = 16, 3-stage cp.async pipeline; 8 warps, 32 x 32 warp tiles
// (4 x 4 m8n8 fragments, 32 fp64 accumulators per thread).  Split-K across CTAs; each CTA
// accumulates its partial tile across super-chunks (kernel launches are stream-ordered,
// so the read-modify-write is race-free and the order is fixed) and reduce_splits sums
// the partials in split order: Z is deterministic.
#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

constexpr int BK = 16, STAGES = 3;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
    const unsigned dst = smem_addr(smem);
    const int sz = pred ? 8 : 0;  // src-size 0 zero-fills
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(pred ? gmem : nullptr), "r"(sz));
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, bool pred) {
    const unsigned dst = smem_addr(smem);
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(pred ? gmem : nullptr), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// C[split] (+)= A . Bm over k in [split*kps, min(K, (split+1)*kps)).
// A: m x K column-major (element (r,k) at k*m + r); Bm: K x d row-major; C: col-major d x m.
// V2: m, d even and A, Bm 16 B aligned -> tiles move as 16 B cp.async pairs.
// KG k-groups: KG sets of WGM x WGN warps share the CTA tile and split each BK slice
// (group g takes k4-steps g, g+KG, ...); their accumulators are summed in group order at
// the end, so a small Z tile still gets 8 warps per CTA without more split-K partials.
// FM x FN m8n8 fragments per warp (warp tile 8FM x 8FN): 4 x 4 by default; 8 x 4 halves the
// fragment loads per DMMA for large Z at one CTA per SM.
template <int WGM, int WGN, int KG, bool V2, int FM = 4, int FN = 4>  // CTA tile 8FM*WGM x 8FN*WGN
__global__ void __launch_bounds__(32 * WGM * WGN * KG,
                                  FM * FN > 16 ? 1 : ((32 * WGM * WGN * KG) <= 256 ? 512 / (32 * WGM * WGN * KG) : 1))
    gemm_dmma(const double* __restrict__ A, int64_t m, const double* __restrict__ Bm, int64_t d, int64_t K, int64_t kps,
              double* __restrict__ C, int accumulate) {
    constexpr int BM = 8 * FM * WGM, BN = 8 * FN * WGN, NT = 32 * WGM * WGN * KG;
    constexpr int LDA = BM + 4, LDB = BN + 4;  // padding: 2-wavefront fragment loads
    pdl_trigger();
    pdl_wait();  // S.X (and the partials) of the kernel before are complete
    static_assert(KG == 1 || KG == 2 || KG == 4, "BK = 16 has 4 k4-steps");
    extern __shared__ double dsm[];
    double* As = dsm;                          // [STAGES][BK][LDA]
    double* Bs = dsm + STAGES * BK * LDA;      // [STAGES][BK][LDB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wg = warp % (WGM * WGN), grp = warp / (WGM * WGN);
    const int wm = wg % WGM, wn = wg / WGM;
    const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
    const int64_t split = blockIdx.z;
    const int64_t kb = split * kps, ke = min(K, kb + kps);
    const int ntiles = (int)((ke - kb + BK - 1) / BK);

    // V2: this thread's 16 B pieces of every tile sit at fixed (k, row/col) offsets, so their
    // global pointers are set up once and advance by BK rows per issued tile (tiles are
    // issued in order) -- no per-tile index arithmetic next to the DMMAs.
    constexpr int PA = (BK * BM / 2 + NT - 1) / NT, PB = (BK * BN / 2 + NT - 1) / NT;
    const double* ga[PA];
    const double* gb[PB];
    int sa_off[PA], sb_off[PB], ka[PA], kb_[PB];
    bool oka[PA], okb[PB];
    if constexpr (V2) {
#pragma unroll
        for (int q = 0; q < PA; ++q) {
            const int e = tid + q * NT, kk = e / (BM / 2), r = 2 * (e - kk * (BM / 2));
            ka[q] = kk;
            oka[q] = e < BK * BM / 2 && m0 + r < m;
            sa_off[q] = kk * LDA + r;
            ga[q] = A + (kb + kk) * m + m0 + r;
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            const int e = tid + q * NT, kk = e / (BN / 2), c = 2 * (e - kk * (BN / 2));
            kb_[q] = kk;
            okb[q] = e < BK * BN / 2 && n0 + c < d;
            sb_off[q] = kk * LDB + c;
            gb[q] = Bm + (kb + kk) * d + n0 + c;
        }
    }
    auto load_tile = [&](int stage, int t) {
        const int64_t k0 = kb + (int64_t)t * BK;
        double* as = As + stage * BK * LDA;
        double* bs = Bs + stage * BK * LDB;
        if constexpr (V2) {
#pragma unroll
            for (int q = 0; q < PA; ++q) {
                if (tid + q * NT < BK * BM / 2) cp_async16(as + sa_off[q], ga[q], oka[q] && k0 + ka[q] < ke);
                ga[q] += BK * m;
            }
#pragma unroll
            for (int q = 0; q < PB; ++q) {
                if (tid + q * NT < BK * BN / 2) cp_async16(bs + sb_off[q], gb[q], okb[q] && k0 + kb_[q] < ke);
                gb[q] += BK * d;
            }
        } else {
            for (int e = tid; e < BK * BM; e += NT) {
                const int kk = e / BM, r = e - kk * BM;
                const int64_t gk = k0 + kk, gr = m0 + r;
                cp_async8(as + kk * LDA + r, A + gk * m + gr, gk < ke && gr < m);
            }
            for (int e = tid; e < BK * BN; e += NT) {
                const int kk = e / BN, c = e - kk * BN;
                const int64_t gk = k0 + kk, gc = n0 + c;
                cp_async8(bs + kk * LDB + c, Bm + gk * d + gc, gk < ke && gc < d);
            }
        }
    };

    double acc[FM][FN][2];
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ntiles) load_tile(s, s);
        cp_commit();
    }
    for (int t = 0; t < ntiles; ++t) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const int stage = t % STAGES;
        const double* as = As + stage * BK * LDA + wm * 8 * FM + (lane >> 2);
        const double* bs = Bs + stage * BK * LDB + wn * 8 * FN + (lane >> 2);
#pragma unroll
        for (int k4 = 4 * grp; k4 < BK; k4 += 4 * KG) {
            double a[FM], b[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) a[i] = as[(k4 + (lane & 3)) * LDA + i * 8];
#pragma unroll
            for (int j = 0; j < FN; ++j) b[j] = bs[(k4 + (lane & 3)) * LDB + j * 8];
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        const int nt = t + STAGES - 1;
        if (nt < ntiles) load_tile(nt % STAGES, nt);
        cp_commit();
    }
    cp_wait<0>();
    if constexpr (KG > 1) {  // fold groups 1..KG-1 into group 0, in group order
        __syncthreads();     // pipeline buffers are free now
        constexpr int G0 = 32 * WGM * WGN;
        if (grp > 0) {
            double* dst = dsm + ((size_t)(grp - 1) * G0 + wg * 32 + lane) * (2 * FM * FN);
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) {
                    dst[(i * FN + j) * 2] = acc[i][j][0];
                    dst[(i * FN + j) * 2 + 1] = acc[i][j][1];
                }
        }
        __syncthreads();
        if (grp > 0) return;
#pragma unroll
        for (int g = 1; g < KG; ++g) {
            const double* src = dsm + ((size_t)(g - 1) * G0 + wg * 32 + lane) * (2 * FM * FN);
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
                for (int j = 0; j < FN; ++j) {
                    acc[i][j][0] += src[(i * FN + j) * 2];
                    acc[i][j][1] += src[(i * FN + j) * 2 + 1];
                }
        }
    }
    double* cp = C + split * m * d;
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t r = m0 + wm * 8 * FM + i * 8 + (lane >> 2);
                const int64_t c = n0 + wn * 8 * FN + j * 8 + (lane & 3) * 2 + h;
                if (r < m && c < d) {
                    double* p = cp + c * m + r;
                    *p = accumulate ? *p + acc[i][j][h] : acc[i][j][h];
                }
            }
}

// G columns [c0, c0 + cols) -> out (m x cols, column-major).
__global__ void gen_gauss_cols(uint64_t g_seed, int64_t m, int64_t c0, int64_t cols, double* __restrict__ out) {
    const int64_t total = m * cols;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / m, r = e - c * m;
        out[e] = gauss_entry(g_seed, (uint64_t)m, (uint64_t)r, (uint64_t)(c0 + c));
    }
}

// Rows [r0, r0+rows) of G over all B columns -> out (rows x B, column-major).
__global__ void gen_gauss_rows(uint64_t g_seed, int64_t m, int64_t r0, int64_t rows, int64_t B,
                               double* __restrict__ out) {
    const int64_t total = rows * B;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / rows, r = e - c * rows;
        out[e] = gauss_entry(g_seed, (uint64_t)m, (uint64_t)(r0 + r), (uint64_t)c);
    }
}

// gready: all of G[:, b0:b1) already materialized (m x K column-major), or nullptr.
template <int WGM, int WGN, int KG = 1, int FM = 4, int FN = 4>
void run_chunks(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t b0, int64_t b1, int64_t d, double* z,
                cudaStream_t s, const double* gready = nullptr) {
    constexpr int BM = 8 * FM * WGM, BN = 8 * FN * WGN, NT = 32 * WGM * WGN * KG;
    const int64_t m = xf->m, K = b1 - b0;
    // super-chunk of S bucket-columns: m x S fp64 <= 48 MB (L2-resident), multiple of BK.
    // (Sizing it so the chunk's S.X rows fit L2 too measured slower: every chunk costs each
    // split-K CTA a read-modify-write of its partial tile.)
    int64_t S = (48ll << 20) / (8 * m);
    S = S < BK ? BK : S / BK * BK;
    // G already in memory: one pass over all of K (no per-chunk ramp, tail and partial
    // read-modify-write; the tiles of a split run concurrently, so their G and S.X slices
    // are shared through L2)
    if ((gready || xf->g_dev) && ctx->opt_gemm_chunks == 0) S = K;
    if (S > K) S = (K + BK - 1) / BK * BK;
    const int64_t tm = (m + BM - 1) / BM, tn = (d + BN - 1) / BN;
    const int64_t resident = (int64_t)ctx->num_sms * (FM * FN > 16 ? 1 : (NT <= 256 ? 512 / NT : 1));  // CTAs per wave
    // (the warp-specialized variant also fits two CTAs per SM)
    int64_t splits = resident / (tm * tn);  // one wave: a second, mostly idle wave would double the time
    const int64_t max_splits = (S + 4 * BK - 1) / (4 * BK);  // >= 4 K-tiles per split per chunk
    splits = splits < 1 ? 1 : (splits > max_splits ? max_splits : splits);
    const int64_t kps = ((S + splits - 1) / splits + BK - 1) / BK * BK;
    splits = (S + kps - 1) / kps;
    // own buffer: xstage may hold the (transposed) X this GEMM is about to read
    double* gbuf = gready ? nullptr : (double*)ctx->gchunk.get(sizeof(double) * (size_t)(m * S));
    double* zpart = (double*)ctx->zpart.get(sizeof(double) * (size_t)(splits * m * d));
    const bool v2 = m % 2 == 0 && d % 2 == 0 && ((uintptr_t)sx % 16) == 0 &&
                    (gready ? (uintptr_t)gready % 16 == 0 : !xf->g_dev || (uintptr_t)xf->g_dev % 16 == 0);
    auto kern = v2 ? gemm_dmma<WGM, WGN, KG, true, FM, FN> : gemm_dmma<WGM, WGN, KG, false, FM, FN>;
    const size_t pipe = sizeof(double) * (size_t)(STAGES * BK * ((BM + 4) + (BN + 4)));
    const size_t fold = sizeof(double) * (size_t)((KG - 1) * BM * BN);  // KG > 1 only with FM = FN = 4
    const size_t smem = pipe > fold ? pipe : fold;
    const int nthreads = NT;
    CGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bool first = true;
    for (int64_t c0 = 0; c0 < K; c0 += S) {
        const int64_t cols = K - c0 < S ? K - c0 : S;
        const double* Ach;
        if (gready) {
            Ach = gready + c0 * m;
        } else if (xf->g_dev) {
            Ach = xf->g_dev + (b0 + c0) * m;  // G in memory is already m x B column-major
        } else {
            int64_t blocks = (m * cols + 255) / 256;
            if (blocks > ctx->num_sms * 32) blocks = ctx->num_sms * 32;
            gen_gauss_cols<<<(unsigned)blocks, 256, 0, s>>>(xf->g_seed, m, b0 + c0, cols, gbuf);
            count_launch(ctx);
            check_launch("gen_gauss_cols");
            Ach = gbuf;
        }
        const int64_t sp = (cols + kps - 1) / kps;  // splits that have work in this chunk
        launch_pdl(ctx, kern, dim3((unsigned)tm, (unsigned)tn, (unsigned)sp), dim3(nthreads), smem, s, Ach, m,
                   sx + c0 * d, d, cols, kps, zpart, first ? 0 : 1);
        count_launch(ctx);
        check_launch("gemm_dmma");
        if (first && sp < splits)  // splits without work in the first chunk start at zero
            CGX_CUDA(cudaMemsetAsync(zpart + sp * m * d, 0, sizeof(double) * (size_t)((splits - sp) * m * d), s));
        first = false;
    }
    launch_reduce_splits(ctx, zpart, splits, m * d, z, s);
}

} // namespace

bool launch_gauss_gemm_chunked(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t b0, int64_t b1,
                               int64_t d, double* z, cudaStream_t s, bool force) {
    const int64_t m = xf->m;
    if (!force && m * d <= 64 * 128) return false;  // small Z: the wide in-kernel-generation GEMM is better
    // 128 x 128 CTA tiles of 32 x 64 warp tiles (one CTA per SM) when Z covers them: half the
    // shared-memory fragment traffic per DMMA of 64 x 128 tiles -- c5 8.52 -> 8.32 ms, c3
    // 0.542 -> 0.530 ms -- in the one-pass GEMM over G in memory.  Over generated L2 chunks
    // the 8-warp tiles stay faster (c5 13.3 vs 13.7 ms); option gemm_tile = 1 keeps them always.
    if (ctx->opt_gemm_tile == 0 && xf->g_dev && ctx->opt_gemm_chunks == 0 && m >= 128 && d >= 128)
        run_chunks<4, 2, 1, 4, 8>(ctx, xf, sx, b0, b1, d, z, s);
    else if (m >= 2 * d)
        run_chunks<4, 2>(ctx, xf, sx, b0, b1, d, z, s);  // 128 x 64 tiles
    else
        run_chunks<2, 4>(ctx, xf, sx, b0, b1, d, z, s);  // 64 x 128 tiles
    return true;
}

namespace {
__global__ void widen_f32_kernel(const float* __restrict__ src, int64_t ld, int64_t n, int64_t d,
                                 double* __restrict__ dst) {
    const int64_t total = n * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / d, j = e - i * d;
        dst[e] = (double)src[i * ld + j];
    }
}
} // namespace

void launch_widen_f32(cgx_ctx* ctx, const float* src, int64_t ld, int64_t n, int64_t d, double* dst, cudaStream_t s) {
    widen_f32_kernel<<<ctx->num_sms * 16, 256, 0, s>>>(src, ld, n, d, dst);
    count_launch(ctx);
    check_launch("widen_f32");
}

void launch_gen_gauss(cgx_ctx* ctx, const cgx_xform* xf, int64_t c0, int64_t cols, double* out, cudaStream_t s) {
    int64_t blocks = (xf->m * cols + 255) / 256;
    if (blocks > ctx->num_sms * 32) blocks = ctx->num_sms * 32;
    gen_gauss_cols<<<(unsigned)blocks, 256, 0, s>>>(xf->g_seed, xf->m, c0, cols, out);
    count_launch(ctx);
    check_launch("gen_gauss_cols");
}

bool launch_gemm_small_g_ready(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t b0, int64_t b1,
                               int64_t d, double* z, cudaStream_t s) {
    // Z covered by one CTA tile of <= 8 warps (32 x 32 each): CTAs of exactly the Z tile,
    // many split-K CTAs per SM -- the contraction is a bandwidth-bound stream of G (in
    // memory, or generated into L2-resident chunks) and S.X.
    const int64_t m = xf->m;
    auto p2 = [](int64_t v) { int64_t p = 1; while (p < v) p <<= 1; return p; };
    const int64_t wm = p2((m + 31) / 32), wn = p2((d + 31) / 32);
    if (wm * wn > 8) return false;
    // G in memory: read it; otherwise run_chunks generates L2-resident column chunks first
    const double* g = xf->g_dev ? xf->g_dev + b0 * m : nullptr;
#define CGX_SMALL(A, B_, KG_)                                           \
    if (wm == A && wn == B_) {                                          \
        run_chunks<A, B_, KG_>(ctx, xf, sx, b0, b1, d, z, s, g);        \
        return true;                                                    \
    }
    CGX_SMALL(1, 1, 4) CGX_SMALL(1, 2, 4) CGX_SMALL(1, 4, 2) CGX_SMALL(1, 8, 1) CGX_SMALL(2, 1, 4)
    CGX_SMALL(2, 2, 2) CGX_SMALL(2, 4, 1) CGX_SMALL(4, 1, 2) CGX_SMALL(4, 2, 1) CGX_SMALL(8, 1, 1)
#undef CGX_SMALL
    return false;
}

void launch_gauss_gemm_rows(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t d, int64_t r0, int64_t r1,
                            double* z, cudaStream_t s) {
    // G rows [r0, r1) as their own (r1-r0) x B column-major matrix, then the ordinary stage 2
    const int64_t rows = r1 - r0, B = xf->B;
    double* gsub = (double*)ctx->gfull.get(sizeof(double) * (size_t)(rows * B));
    if (xf->g_dev) {
        CGX_CUDA(cudaMemcpy2DAsync(gsub, sizeof(double) * (size_t)rows, xf->g_dev + r0, sizeof(double) * (size_t)xf->m,
                                   sizeof(double) * (size_t)rows, (size_t)B, cudaMemcpyDeviceToDevice, s));
    } else {
        int64_t blocks = (rows * B + 255) / 256;
        if (blocks > ctx->num_sms * 32) blocks = ctx->num_sms * 32;
        gen_gauss_rows<<<(unsigned)blocks, 256, 0, s>>>(xf->g_seed, xf->m, r0, rows, B, gsub);
        count_launch(ctx);
        check_launch("gen_gauss_rows");
    }
    cgx_xform gx = *xf;  // a view: rows of G, explicit; nothing owned
    gx.m = rows;
    gx.g_dev = gsub;
    gx.g_pool = false;
    gx.g_explicit = true;
    gx.view = true;
    gx.oz_gimg = nullptr;
    gx.oz_gmax = nullptr;
    gx.oz_gS = 0;
    launch_gauss_gemm(ctx, &gx, sx, 0, B, d, z, s);
}

} // namespace cgx
