// gproject.cu -- the dense-Gaussian baseline G~.X for CSR X (the config-5
// ablation).  Replaces the reference bench's naive O(nnz * m) loop
// (tools/countgauss_main.cpp:535-547, tests/acceptance.cpp:365-377):
//
//   G~ = gaussian_matrix(m, n, g_rng);            // matrix.cpp:199-207, m x n, never stored here
//   for i, for (j, v) in row i:  Z(:, j) += v * G~(:, i)
//
// B200 design: Z is split into 32-row blocks; CTA (rb, p) owns rows [32 rb, 32 rb + 32) of Z
// over (up to 640) columns in shared memory and a contiguous range p of X's rows.  Its 8
// warps take rows in turn: lane r generates G~(32 rb + r, i) (the SplitMix64 draw i*m + r
// of the rng's state, Acklam + Halley: exactly gaussian_matrix's value), then for each
// nonzero of the row every lane adds v * G~(., i) into its own Z row -- 32 consecutive
// shared-memory words.  Each G~ entry is generated once over the grid (n * m normals) and
// never touches HBM.  Warps of a CTA and CTAs of a row block meet in fp64 atomics (shared,
// then global), so Z matches the reference to rounding (a timing baseline, not on the
// product path).  A column-owned variant without shared atomics (binary search for each
// warp's column stretch per row) measured 2.5x slower: its per-row global-load chains
// serialize.
#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

template <typename TV, typename TI>
__global__ void __launch_bounds__(256) gproject_csr_kernel(uint64_t g_seed, int64_t m, const int64_t* __restrict__ rowptr,
                                                           const TI* __restrict__ cols, const TV* __restrict__ vals,
                                                           int64_t n, int64_t d, int64_t c0, int64_t ncol,
                                                           int64_t rows_per_part, double* __restrict__ z) {
    extern __shared__ double zb[];  // [ncol][32]: Z rows 32 rb .. 32 rb + 31, columns c0 .. c0 + ncol
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t rb = blockIdx.x, part = blockIdx.y;
    const int64_t r = 32 * rb + lane;
    for (int64_t e = threadIdx.x; e < 32 * ncol; e += blockDim.x) zb[e] = 0.0;
    __syncthreads();
    const int64_t i0 = part * rows_per_part, i1 = min(n, i0 + rows_per_part);
    for (int64_t i = i0 + wid; i < i1; i += blockDim.x >> 5) {
        const int64_t p0 = rowptr[i], p1 = rowptr[i + 1];
        if (p0 == p1) continue;
        const double g = r < m ? gauss_entry(g_seed, (uint64_t)m, (uint64_t)r, (uint64_t)i) : 0.0;
        for (int64_t p = p0; p < p1; ++p) {
            const int64_t j = (int64_t)cols[p] - c0;
            if (j < 0 || j >= ncol) continue;
            atomicAdd(&zb[j * 32 + lane], (double)vals[p] * g);
        }
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < 32 * ncol; e += blockDim.x) {
        const int64_t j = e >> 5, rr = 32 * rb + (e & 31);
        if (rr < m && zb[e] != 0.0) red_add(&z[(c0 + j) * m + rr], zb[e]);
    }
}

template <typename TV, typename TI>
void run_gp(cgx_ctx* ctx, uint64_t g_seed, int64_t m, const int64_t* rowptr, const TI* cols, const TV* vals, int64_t n,
            int64_t d, double* z, cudaStream_t s) {
    CGX_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * (size_t)(m * d), s));
    const int64_t nrb = (m + 31) / 32;
    const int64_t max_cols = (160 * 1024) / (32 * sizeof(double));  // Z block columns per CTA pass
    for (int64_t c0 = 0; c0 < d; c0 += max_cols) {
        const int64_t ncol = d - c0 < max_cols ? d - c0 : max_cols;
        const size_t smem = sizeof(double) * 32 * (size_t)ncol;
        auto kern = gproject_csr_kernel<TV, TI>;
        CGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
        int64_t parts = ((int64_t)ctx->num_sms * (per_sm < 1 ? 1 : per_sm) * 4 + nrb - 1) / nrb;
        if (parts > n) parts = n;
        if (parts > 65535) parts = 65535;
        const int64_t rpp = (n + parts - 1) / parts;
        parts = (n + rpp - 1) / rpp;
        kern<<<dim3((unsigned)nrb, (unsigned)parts), 256, smem, s>>>(g_seed, m, rowptr, cols, vals, n, d, c0, ncol, rpp,
                                                                     z);
        count_launch(ctx);
        check_launch("gproject_csr");
    }
}

} // namespace

void launch_gproject_csr(cgx_ctx* ctx, uint64_t g_seed, int64_t m, const int64_t* rowptr, const void* cols,
                         int idx_type, const void* vals, int dtype, int64_t n, int64_t d, double* z, cudaStream_t s) {
    if (dtype == CGX_F32) {
        if (idx_type == CGX_I32)
            run_gp<float, int32_t>(ctx, g_seed, m, rowptr, (const int32_t*)cols, (const float*)vals, n, d, z, s);
        else
            run_gp<float, int64_t>(ctx, g_seed, m, rowptr, (const int64_t*)cols, (const float*)vals, n, d, z, s);
    } else {
        if (idx_type == CGX_I32)
            run_gp<double, int32_t>(ctx, g_seed, m, rowptr, (const int32_t*)cols, (const double*)vals, n, d, z, s);
        else
            run_gp<double, int64_t>(ctx, g_seed, m, rowptr, (const int64_t*)cols, (const double*)vals, n, d, z, s);
    }
}

} // namespace cgx
