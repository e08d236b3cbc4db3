// gauss_gemm.cu -- stage 2, Z = G . (S.X), with G generated inside the GEMM.
//
// Replaces gemm(t.g, SX) (reference src/matrix.cpp:111-129) and the materialized
// t.g = gaussian_matrix(m, B, g_rng) (matrix.cpp:199-207, rng.cpp:13-59).  G(r, c) is a
// pure function of (g_seed, c*m + r) -- SplitMix64 draw, 53-bit uniform, Acklam quantile,
// one Halley step -- so each CTA generates exactly the m-tile x K-chunk of G it consumes,
// in shared memory, and G never exists in HBM.
//
// The contraction is FP64 on the tensor pipe: warp-level DMMA (mma.sync m8n8k4 f64;
// tcgen05 has no f64 kind on sm_100a).  3xTF32 would miss the reference's 1e-8
// composite tolerance, so the fp64 drop-in stays fp64.
//
// Work split: CTA tile 64 (rows of Z) x 32 (columns of Z) x a K-range of buckets
// (split-K).  Each split writes its partial tile; a second kernel sums the partials in
// ascending split order, so Z is deterministic run to run.
#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

constexpr int MT = 64, NT = 32, KC = 32;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// sx holds buckets [gcol0, gcol0 + B) (row-major, row k = bucket gcol0 + k).
__global__ void __launch_bounds__(256) gauss_gemm_kernel(const double* __restrict__ sx, int64_t B, int64_t d,
                                                         int64_t m, uint64_t g_seed,
                                                         const double* __restrict__ g_explicit, int64_t gcol0,
                                                         int64_t k_per_split, double* __restrict__ zpart) {
    __shared__ double Gs[MT][KC + 1];
    __shared__ double Ss[KC][NT + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 3, wn = warp >> 2;  // 4 x 2 warps, 16 x 16 each
    const int64_t m0 = (int64_t)blockIdx.x * MT, n0 = (int64_t)blockIdx.y * NT;
    const int64_t split = blockIdx.z;
    const int64_t kb = split * k_per_split;
    const int64_t ke = min(B, kb + k_per_split);

    double acc[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int64_t k0 = kb; k0 < ke; k0 += KC) {
        // G tile: rows m0.., columns k0..  (column-major draw order c*m + r)
#pragma unroll
        for (int i = 0; i < (MT * KC) / 256; ++i) {
            const int e = tid + 256 * i;
            const int r = e % MT, c = e / MT;
            const int64_t gr = m0 + r, gc = k0 + c;
            double g = 0.0;
            if (gr < m && gc < ke) {
                const int64_t col = gcol0 + gc;
                g = g_explicit ? g_explicit[col * m + gr] : gauss_entry(g_seed, (uint64_t)m, (uint64_t)gr, (uint64_t)col);
            }
            Gs[r][c] = g;
        }
        // SX tile: rows k0.., columns n0..   (row-major B x d)
#pragma unroll
        for (int i = 0; i < (KC * NT) / 256; ++i) {
            const int e = tid + 256 * i;
            const int c = e % NT, r = e / NT;
            const int64_t gk = k0 + r, gn = n0 + c;
            Ss[r][c] = (gk < ke && gn < d) ? sx[gk * d + gn] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KC; kk += 4) {
            double a[2], b[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) a[i] = Gs[wm * 16 + i * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < 2; ++j) b[j] = Ss[kk + (lane & 3)][wn * 16 + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
        __syncthreads();
    }
    // partial tile -> zpart[split] (column-major m x d)
    double* zp = zpart + split * m * d;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t r = m0 + wm * 16 + i * 8 + (lane >> 2);
                const int64_t c = n0 + wn * 16 + j * 8 + (lane & 3) * 2 + h;
                if (r < m && c < d) zp[c * m + r] = acc[i][j][h];
            }
}

// z[e] = sum_k zpart[k][e].  Block = 32 entries x 16 split groups: group g sums splits
// g, g+16, ... in order, then the 16 group sums are added in group order -- a fixed
// association, so Z is bit-reproducible; loads stay coalesced along e.
constexpr int kRedGroups = 16;
__global__ void __launch_bounds__(32 * kRedGroups) reduce_splits(const double* __restrict__ zpart, int64_t splits,
                                                                 int64_t md, double* __restrict__ z) {
    pdl_wait();  // the partials of the kernel before are complete
    __shared__ double part[kRedGroups][33];
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int64_t e = (int64_t)blockIdx.x * 32 + lane;
    double s = 0.0;
    if (e < md)
        for (int64_t k = g; k < splits; k += kRedGroups) s += zpart[k * md + e];
    part[g][lane] = s;
    __syncthreads();
    if (g == 0 && e < md) {
        double t = part[0][lane];
#pragma unroll
        for (int q = 1; q < kRedGroups; ++q) t += part[q][lane];
        z[e] = t;
    }
}

// Wide tile: a CTA owns WM rows of Z and ALL d (<= 1024) columns for a K-range, so each
// G(r, c) is generated exactly once over the whole grid (the narrow kernel above
// regenerates G once per 32-column tile -- 8x for d = 256).  The WM x d tile is
// (WM/8) x (dp/8) m8n8k4 fragments spread over the 8 warps (<= 16 per warp, 2 fp64
// accumulators each).  Per K-chunk: 256 threads generate WM x KW normals into smem, the
// KW x d slab of S.X is staged in smem, then every warp issues its DMMAs.
template <int WM, int KW>
__global__ void __launch_bounds__(256, 2) gauss_gemm_wide(const double* __restrict__ sx, int64_t B, int64_t d, int64_t m,
                                                       uint64_t g_seed, const double* __restrict__ g_explicit,
                                                       int64_t gcol0, int64_t k_per_split, double* __restrict__ zpart) {
    extern __shared__ double wsm[];
    const int dp = (int)((d + 7) & ~7);
    double* Gs = wsm;                      // [WM][KW + 1]
    double* Ss = wsm + WM * (KW + 1);      // [KW][dp + 1]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int RF = WM / 8, F = RF * (dp / 8);
    const int64_t m0 = (int64_t)blockIdx.x * WM;
    const int64_t split = blockIdx.y;
    const int64_t kb = split * k_per_split, ke = min(B, kb + k_per_split);
    double acc[16][2];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q][0] = acc[q][1] = 0.0;

    for (int64_t k0 = kb; k0 < ke; k0 += KW) {
#pragma unroll 1
        for (int e = tid; e < WM * KW; e += 256) {
            const int r = e % WM, c = e / WM;
            const int64_t gr = m0 + r, gc = k0 + c;
            double g = 0.0;
            if (gr < m && gc < ke) {
                const int64_t col = gcol0 + gc;
                g = g_explicit ? g_explicit[col * m + gr] : gauss_entry(g_seed, (uint64_t)m, (uint64_t)gr, (uint64_t)col);
            }
            Gs[r * (KW + 1) + c] = g;
        }
        for (int e = tid; e < KW * dp; e += 256) {
            const int c = e % dp, r = e / dp;
            const int64_t gk = k0 + r;
            Ss[r * (dp + 1) + c] = (gk < ke && c < d) ? sx[gk * d + c] : 0.0;
        }
        __syncthreads();
#pragma unroll 1
        for (int kk = 0; kk < KW; kk += 4) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int f = warp + 8 * q;
                if (f < F) {
                    const int rf = f % RF, cf = f / RF;
                    const double a = Gs[(rf * 8 + (lane >> 2)) * (KW + 1) + kk + (lane & 3)];
                    const double b = Ss[(kk + (lane & 3)) * (dp + 1) + cf * 8 + (lane >> 2)];
                    dmma884(acc[q][0], acc[q][1], a, b);
                }
            }
        }
        __syncthreads();
    }
    double* zp = zpart + split * m * d;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int f = warp + 8 * q;
        if (f < F) {
            const int rf = f % RF, cf = f / RF;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t r = m0 + rf * 8 + (lane >> 2);
                const int64_t c = (int64_t)cf * 8 + (lane & 3) * 2 + h;
                if (r < m && c < d) zp[c * m + r] = acc[q][h];
            }
        }
    }
}

// T = G . S (m x n, column-major): the projection svm-check materializes as
// gemm(t.g, reference::materialize(t.cs)) (tools/countgauss_main.cpp:660-668).  gemm skips
// the zero entries of S, so column i is exactly sign_i * G(:, hash_i).  Warp per bucket:
// G(:, b) is read (or generated) once and written, sign-flipped, to each of b's columns.
__global__ void materialize_t_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ offsets, int64_t B,
                                     int64_t m, uint64_t g_seed, const double* __restrict__ g_dev,
                                     double* __restrict__ t) {
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (b >= B) return;
    const uint32_t p0 = offsets[b], p1 = offsets[b + 1];
    if (p0 == p1) return;
    for (int64_t r0 = 0; r0 < m; r0 += 32) {
        const int64_t r = r0 + lane;
        double g = 0.0;
        if (r < m) g = g_dev ? g_dev[b * m + r] : gauss_entry(g_seed, (uint64_t)m, (uint64_t)r, (uint64_t)b);
        for (uint32_t p = p0; p < p1; ++p) {
            const uint32_t e = __ldg(perm + p);
            if (r < m) t[(int64_t)(e & kRowMask) * m + r] = (e & kNegBit) ? -g : g;
        }
    }
}

__global__ void fill_gaussian_kernel(uint64_t g_seed, int64_t m, int64_t total, double* g) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = e / m, r = e - c * m;
        g[e] = gauss_entry(g_seed, (uint64_t)m, (uint64_t)r, (uint64_t)c);
    }
}

__global__ void inverse_normal_cdf_kernel(const double* p, double* out, int64_t count, int* bad) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
        const double v = p[e];
        if (!(v > 0.0 && v < 1.0)) {
            atomicExch(bad, 1);
            out[e] = __longlong_as_double(0x7ff8000000000000LL);
        } else {
            out[e] = inverse_normal_cdf(v);
        }
    }
}

} // namespace

void launch_gauss_gemm(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t b0, int64_t b1, int64_t d,
                       double* z, cudaStream_t s) {
    const int64_t m = xf->m, B = b1 - b0;
    if (B <= 0) {
        CGX_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * (size_t)(m * d), s));
        return;
    }
    if (launch_gemm_ozaki(ctx, xf, b0, b1, sx, d, z, s)) return;  // tcgen05 (opt-in)
    if (launch_gemm_small_g_ready(ctx, xf, sx, b0, b1, d, z, s)) return;  // small Z, G in memory
    if (launch_gauss_gemm_chunked(ctx, xf, sx, b0, b1, d, z, s)) return;  // large Z (dgemm.cu)
    if (d <= 1024) {
        // wide tile: WM rows x all columns, WM * dp <= 8192 (<= 16 fragments per warp)
        const int64_t dp = (d + 7) & ~int64_t(7);
        const int WM = dp <= 128 ? 64 : dp <= 256 ? 32 : dp <= 512 ? 16 : 8;
        // K-chunk sized so the S.X slab stays <= ~34 KB: two CTAs per SM fit in smem
        const int KW = dp <= 128 ? 32 : dp <= 256 ? 16 : 8;
        const int64_t tm = (m + WM - 1) / WM;
        const int64_t kchunks = (B + KW - 1) / KW;
        int64_t want = (2 * (int64_t)ctx->num_sms + tm - 1) / tm;
        want = want < 1 ? 1 : (want > kchunks ? kchunks : (want > 65535 ? 65535 : want));
        const int64_t k_per_split = (kchunks + want - 1) / want * KW;
        const int64_t splits = (B + k_per_split - 1) / k_per_split;
        const size_t smem = sizeof(double) * (size_t)(WM * (KW + 1) + KW * (dp + 1));
        double* zpart = (double*)ctx->zpart.get(sizeof(double) * (size_t)(splits * m * d));
        const double* gex = xf->g_dev;
        const dim3 grid((unsigned)tm, (unsigned)splits);
#define CGX_WIDE(WM_, KW_)                                                                                       \
    do {                                                                                                         \
        auto kern = gauss_gemm_wide<WM_, KW_>;                                                                   \
        CGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));          \
        kern<<<grid, 256, smem, s>>>(sx, B, d, m, xf->g_seed, gex, b0, k_per_split, zpart);                     \
    } while (0)
        if (WM == 64) CGX_WIDE(64, 32);
        else if (WM == 32) CGX_WIDE(32, 16);
        else if (WM == 16) CGX_WIDE(16, 8);
        else CGX_WIDE(8, 8);
#undef CGX_WIDE
        count_launch(ctx);
        check_launch("gauss_gemm_wide");
        launch_reduce_splits(ctx, zpart, splits, m * d, z, s);
        return;
    }
    const int64_t tm = (m + MT - 1) / MT, tn = (d + NT - 1) / NT;
    const int64_t kchunks = (B + KC - 1) / KC;
    int64_t want = (2 * (int64_t)ctx->num_sms + tm * tn - 1) / (tm * tn);
    if (want < 1) want = 1;
    if (want > kchunks) want = kchunks;
    if (want > 65535) want = 65535;
    const int64_t chunks_per_split = (kchunks + want - 1) / want;
    const int64_t k_per_split = chunks_per_split * KC;
    const int64_t splits = (B + k_per_split - 1) / k_per_split;
    double* zpart = (double*)ctx->zpart.get(sizeof(double) * (size_t)(splits * m * d));
    gauss_gemm_kernel<<<dim3((unsigned)tm, (unsigned)tn, (unsigned)splits), 256, 0, s>>>(
        sx, B, d, m, xf->g_seed, xf->g_dev, b0, k_per_split, zpart);
    count_launch(ctx);
    check_launch("gauss_gemm");
    launch_reduce_splits(ctx, zpart, splits, m * d, z, s);
}

void launch_materialize_t(cgx_ctx* ctx, const cgx_xform* xf, double* t, cudaStream_t s) {
    const int64_t threads = xf->B * 32;
    materialize_t_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(xf->perm, xf->offsets, xf->B, xf->m,
                                                                           xf->g_seed, xf->g_dev, t);
    count_launch(ctx);
    check_launch("materialize_t");
}

void launch_reduce_splits(cgx_ctx* ctx, const double* zpart, int64_t splits, int64_t md, double* z, cudaStream_t s) {
    const int64_t blocks = (md + 31) / 32;
    launch_pdl(ctx, reduce_splits, dim3((unsigned)blocks), dim3(32 * kRedGroups), 0, s, zpart, splits, md, z);
    count_launch(ctx);
    check_launch("reduce_splits");
}

void launch_fill_gaussian(cgx_ctx* ctx, const cgx_xform* xf, double* g, cudaStream_t s) {
    const int64_t total = xf->m * xf->B;
    if (xf->g_dev) {
        CGX_CUDA(cudaMemcpyAsync(g, xf->g_dev, sizeof(double) * (size_t)total, cudaMemcpyDeviceToDevice, s));
        return;
    }
    int64_t blocks = (total + 255) / 256;
    if (blocks > ctx->num_sms * 16) blocks = ctx->num_sms * 16;
    fill_gaussian_kernel<<<(unsigned)blocks, 256, 0, s>>>(xf->g_seed, xf->m, total, g);
    count_launch(ctx);
    check_launch("fill_gaussian");
}

void launch_inverse_normal_cdf(cgx_ctx* ctx, const double* p, double* out, int64_t count, int* bad, cudaStream_t s) {
    int64_t blocks = (count + 255) / 256;
    if (blocks > ctx->num_sms * 16) blocks = ctx->num_sms * 16;
    if (blocks < 1) blocks = 1;
    inverse_normal_cdf_kernel<<<(unsigned)blocks, 256, 0, s>>>(p, out, count, bad);
    count_launch(ctx);
    check_launch("inverse_normal_cdf");
}

} // namespace cgx
