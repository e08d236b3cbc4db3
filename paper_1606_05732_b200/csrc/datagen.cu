// datagen.cu -- seeded synthetic inputs for the BASELINE configs, generated in HBM.
//
// The reference benchmarks no public dataset (BASELINE.json "published": {}); these
// counter-based generators stand in for it with the configs' shapes and value
// distributions.  Entry e of a stream with seed s is the fp32 N(0,1) quantile of draw e
// of SeededRng(s) (oracle/cgoracle.c cgo_normal_f32 is the CPU twin).
//   dense  : entry (i, j) = stream entry i*d + j
//   CSR    : entry (i, j) present iff uniform(draw i*d+j of mix64(seed,1)) < density;
//            its value is entry i*d + j of stream mix64(seed,2).  Columns come out sorted
//            and distinct per row (the CSR invariant, reference matrix.cpp:92-109).
#include <cmath>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

template <typename T>
__global__ void gen_dense_kernel(uint64_t seed, int64_t row0, const int64_t* __restrict__ rows, int64_t n, int64_t d,
                                 int layout, T* x) {
    const int64_t total = n * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        // e enumerates the destination in its own layout for coalesced stores
        int64_t i, j;
        if (layout == CGX_ROW_MAJOR) {
            i = e / d;
            j = e - i * d;
        } else {
            j = e / n;
            i = e - j * n;
        }
        const int64_t gi = rows ? rows[i] : row0 + i;  // global row: the value is a function of (row, column)
        x[e] = (T)datagen_normal(seed, (uint64_t)(gi * d + j));
    }
}

// Inclusion rule of entry (row, j).  Bernoulli: probability `density`.  Zipf (config 5):
// the row draws a target length L from Zipf(s_len) on [1, cap] (inverse CDF table), and
// column j is kept with probability min(1, c_L * w_j), w_j ~ (j+1)^-s_col normalized and
// c_L solved on the host so that sum_j min(1, c_L * w_j) = L: a row's expected length is
// exactly L (mean nnz/row = E[L], 17.36 at s_len = 1.5, cap 512), rows are heavy-tailed,
// columns skewed toward small indices, sorted and distinct by construction.
struct CsrRule {
    double density;          // Bernoulli mode when len_cdf == nullptr
    const double* len_cdf;   // cap entries, CDF of the target length
    int cap;
    const double* colw;      // d entries, normalized column weights
    const double* scale;     // cap entries: c_L for L = 1..cap
    uint64_t lseed;
};

__device__ __forceinline__ double row_scale(const CsrRule& rule, int64_t row) {
    if (!rule.len_cdf) return 0.0;
    const double u = uniform53(rng_draw(rule.lseed, (uint64_t)row));
    int lo = 0, hi = rule.cap - 1;  // first k with cdf[k] >= u
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (rule.len_cdf[mid] >= u) hi = mid; else lo = mid + 1;
    }
    return rule.scale[lo];
}

__device__ __forceinline__ bool included(const CsrRule& rule, double L, uint64_t mseed, int64_t row, int64_t d,
                                         int64_t j) {
    const double u = uniform53(rng_draw(mseed, (uint64_t)(row * d + j)));
    const double p = rule.len_cdf ? fmin(1.0, L * rule.colw[j]) : rule.density;  // L: the row's c_L
    return u < p;
}

__global__ void gen_csr_counts_kernel(uint64_t mseed, int64_t n, int64_t d, CsrRule rule, int64_t* counts) {
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (row >= n) return;
    const double L = row_scale(rule, row);
    int64_t c = 0;
    for (int64_t j = lane; j < d; j += 32) c += included(rule, L, mseed, row, d, j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[row] = c;
}

__global__ void gen_csr_fill_kernel(uint64_t mseed, uint64_t vseed, int64_t n, int64_t d, CsrRule rule,
                                    const int64_t* rowptr, int32_t* cols, float* vals) {
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (row >= n) return;
    const double L = row_scale(rule, row);
    int64_t pos = rowptr[row];
    for (int64_t j0 = 0; j0 < d; j0 += 32) {
        const int64_t j = j0 + lane;
        const bool in = j < d && included(rule, L, mseed, row, d, j);
        const unsigned mask = __ballot_sync(0xffffffffu, in);
        if (in) {
            const int64_t p = pos + __popc(mask & ((1u << lane) - 1u));
            cols[p] = (int32_t)j;
            vals[p] = datagen_normal(vseed, (uint64_t)(row * d + j));
        }
        pos += __popc(mask);
    }
}

} // namespace

void launch_gen_dense(cgx_ctx* ctx, uint64_t seed, int64_t row0, const int64_t* rows, int64_t n, int64_t d, int dtype,
                      int layout, void* x, cudaStream_t s) {
    const int blocks = ctx->num_sms * 16;
    if (dtype == CGX_F32)
        gen_dense_kernel<float><<<blocks, 256, 0, s>>>(seed, row0, rows, n, d, layout, (float*)x);
    else
        gen_dense_kernel<double><<<blocks, 256, 0, s>>>(seed, row0, rows, n, d, layout, (double*)x);
    count_launch(ctx);
    check_launch("gen_dense");
}

namespace {
// Device copies of the Zipf tables (identical on every call for the same spec).
CsrRule make_rule(cgx_ctx* ctx, uint64_t seed, int64_t d, const CsrGenSpec& spec, cudaStream_t s) {
    CsrRule r{spec.density, nullptr, 0, nullptr, nullptr, mix64(seed, 4)};
    if (!spec.zipf) return r;
    std::vector<double> tab((size_t)(2 * spec.cap + d));
    double acc = 0.0;
    for (int k = 1; k <= spec.cap; ++k) acc += std::pow((double)k, -spec.s_len);
    double run = 0.0;
    for (int k = 1; k <= spec.cap; ++k) {
        run += std::pow((double)k, -spec.s_len);
        tab[(size_t)(k - 1)] = run / acc;
    }
    tab[(size_t)(spec.cap - 1)] = 1.0;
    double wsum = 0.0;
    for (int64_t j = 0; j < d; ++j) wsum += std::pow((double)(j + 1), -spec.s_col);
    for (int64_t j = 0; j < d; ++j) tab[(size_t)(spec.cap + j)] = std::pow((double)(j + 1), -spec.s_col) / wsum;
    // c_L: bisection on the monotone f(c) = sum_j min(1, c w_j) (f(c) -> d; L >= d keeps all)
    const double* w = tab.data() + spec.cap;
    for (int L = 1; L <= spec.cap; ++L) {
        double c;
        if (L >= d) {
            c = 1e300;
        } else {
            double lo = 0.0, hi = 1.0;
            auto f = [&](double cc) {
                double t = 0.0;
                for (int64_t j = 0; j < d; ++j) t += std::min(1.0, cc * w[j]);
                return t;
            };
            while (f(hi) < L) hi *= 2.0;
            for (int it = 0; it < 100; ++it) {
                const double mid = 0.5 * (lo + hi);
                (f(mid) < L ? lo : hi) = mid;
            }
            c = hi;
        }
        tab[(size_t)(spec.cap + d + L - 1)] = c;
    }
    double* dev = (double*)ctx->gen_tables.get(sizeof(double) * tab.size());
    CGX_CUDA(cudaMemcpyAsync(dev, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice, s));
    CGX_CUDA(cudaStreamSynchronize(s));  // tab is a host temporary
    r.len_cdf = dev;
    r.cap = spec.cap;
    r.colw = dev + spec.cap;
    r.scale = dev + spec.cap + d;
    return r;
}
} // namespace

void launch_gen_csr_counts(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, const CsrGenSpec& spec,
                           int64_t* rowptr, cudaStream_t s) {
    const CsrRule rule = make_rule(ctx, seed, d, spec, s);
    const int64_t threads = n * 32;
    gen_csr_counts_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(mix64(seed, 1), n, d, rule, rowptr);
    count_launch(ctx);
    check_launch("gen_csr_counts");
    CGX_CUDA(cudaMemsetAsync(rowptr + n, 0, sizeof(int64_t), s));
    exclusive_scan_i64(ctx, rowptr, rowptr, n + 1, s);
}

void launch_gen_csr_fill(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, const CsrGenSpec& spec,
                         const int64_t* rowptr, int32_t* cols, float* vals, cudaStream_t s) {
    const CsrRule rule = make_rule(ctx, seed, d, spec, s);
    const int64_t threads = n * 32;
    gen_csr_fill_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(mix64(seed, 1), mix64(seed, 2), n, d,
                                                                         rule, rowptr, cols, vals);
    count_launch(ctx);
    check_launch("gen_csr_fill");
}

} // namespace cgx
