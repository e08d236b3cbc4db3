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
#include <algorithm>
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

// Config 4 (near-separable NMF input, BASELINE configs[3]): X = max(A.[I_r | H] + sigma*N, 0).
// Entry (i, j), fp32 with every product and sum rounded separately (no FMA) in ascending
// k, so the CPU twin (oracle/cgoracle.c cgo_gen_separable_f32) reproduces it:
//   a_k   = top 24 bits of draw i*r + k of aseed, times 2^-24      (A uniform on [0, 1))
//   base  = a_j for j < r, else sum_k a_k * H[k, j-r]              (H fp32, r x (d-r) row-major)
//   x     = max(base + sigma * datagen_normal(nseed, i*d + j), 0)
__device__ __forceinline__ float sep_uniform(uint64_t aseed, uint64_t e) {
    return (float)(rng_draw(aseed, e) >> 40) * 0x1.0p-24f;
}

template <typename T>
__global__ void gen_separable_kernel(uint64_t aseed, uint64_t nseed, const float* __restrict__ h, int64_t row0,
                                     int64_t n, int64_t d, int r, float sigma, int layout, T* x) {
    const int64_t total = n * d;
    const int64_t hc = d - r;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t i, j;
        if (layout == CGX_ROW_MAJOR) {
            i = e / d;
            j = e - i * d;
        } else {
            j = e / n;
            i = e - j * n;
        }
        const uint64_t gi = (uint64_t)(row0 + i);
        float base;
        if (j < r) {
            base = sep_uniform(aseed, gi * (uint64_t)r + (uint64_t)j);
        } else {
            base = 0.0f;
            for (int k = 0; k < r; ++k)
                base = __fadd_rn(base, __fmul_rn(sep_uniform(aseed, gi * (uint64_t)r + (uint64_t)k), h[k * hc + (j - r)]));
        }
        const float v = __fadd_rn(base, __fmul_rn(sigma, datagen_normal(nseed, gi * (uint64_t)d + (uint64_t)j)));
        x[e] = (T)(v > 0.0f ? v : 0.0f);
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
// Host restatement of Acklam's rational (rng.cpp:13-41, the reference's evaluation order)
// for the mixing-weight sampler below.
double host_acklam(double p) {
    static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                               1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                               6.680131188771972e+01,  -1.328068155288572e+01};
    static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                               -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
    static const double dd[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                                3.754408661907416e+00};
    const double p_low = 0.02425;
    if (p < p_low || p > 1.0 - p_low) {
        const bool upper = p > 1.0 - p_low;
        const double q = std::sqrt(-2.0 * std::log(upper ? 1.0 - p : p));
        const double x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
                         ((((dd[0] * q + dd[1]) * q + dd[2]) * q + dd[3]) * q + 1.0);
        return upper ? -x : x;
    }
    const double q = p - 0.5, r = q * q;
    return (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
           (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
}

// Gamma(alpha, 1) by Marsaglia-Tsang on a sequential SeededRng stream (draw counter *k);
// alpha < 1 through Gamma(alpha + 1) * U^(1/alpha).
double host_gamma(uint64_t seed, uint64_t* k, double alpha) {
    if (alpha < 1.0) {
        const double g = host_gamma(seed, k, alpha + 1.0);
        const double u = uniform53(rng_draw(seed, (*k)++));
        return g * std::pow(u, 1.0 / alpha);
    }
    const double dm = alpha - 1.0 / 3.0, c = 1.0 / std::sqrt(9.0 * dm);
    for (;;) {
        const double z = host_acklam(uniform53(rng_draw(seed, (*k)++)));
        double v = 1.0 + c * z;
        if (v <= 0.0) continue;
        v = v * v * v;
        const double u = uniform53(rng_draw(seed, (*k)++));
        if (std::log(u) < 0.5 * z * z + dm - dm * v + dm * std::log(v)) return dm * v;
    }
}
} // namespace

// H (r x cols, column-major): column c ~ Dirichlet(alpha, ..., alpha), the normalized
// Gamma(alpha) draws of stream mix64(seed, 13) taken column by column, component by
// component.  The mixing weights of config 4 (oracle twin: cgo_separable_mixing).
void separable_mixing(uint64_t seed, int64_t r, int64_t cols, double alpha, double* h) {
    const uint64_t hseed = mix64(seed, 13);
    uint64_t k = 0;
    for (int64_t c = 0; c < cols; ++c) {
        double* hc = h + c * r;
        double sum = 0.0;
        for (int64_t q = 0; q < r; ++q) {
            hc[q] = host_gamma(hseed, &k, alpha);
            sum += hc[q];
        }
        for (int64_t q = 0; q < r; ++q) hc[q] = sum > 0.0 ? hc[q] / sum : 1.0 / (double)r;
    }
}

void launch_gen_separable(cgx_ctx* ctx, uint64_t seed, int64_t row0, int64_t n, int64_t d, int64_t r, double alpha,
                          double sigma, int dtype, int layout, void* x, cudaStream_t s) {
    const int64_t hc = d - r;
    std::vector<double> h((size_t)(r * hc));
    separable_mixing(seed, r, hc, alpha, h.data());
    std::vector<float> hf((size_t)(r * hc));  // fp32, row-major r x (d - r) for the kernel
    for (int64_t k = 0; k < r; ++k)
        for (int64_t c = 0; c < hc; ++c) hf[(size_t)(k * hc + c)] = (float)h[(size_t)(c * r + k)];
    float* hd = (float*)ctx->gen_tables.get(sizeof(float) * std::max<size_t>(hf.size(), 1));
    if (!hf.empty()) CGX_CUDA(cudaMemcpyAsync(hd, hf.data(), sizeof(float) * hf.size(), cudaMemcpyHostToDevice, s));
    const int blocks = ctx->num_sms * 16;
    const uint64_t aseed = mix64(seed, 11), nseed = mix64(seed, 12);
    if (dtype == CGX_F32)
        gen_separable_kernel<float><<<blocks, 256, 0, s>>>(aseed, nseed, hd, row0, n, d, (int)r, (float)sigma, layout,
                                                           (float*)x);
    else
        gen_separable_kernel<double><<<blocks, 256, 0, s>>>(aseed, nseed, hd, row0, n, d, (int)r, (float)sigma,
                                                            layout, (double*)x);
    count_launch(ctx);
    check_launch("gen_separable");
    CGX_CUDA(cudaStreamSynchronize(s));  // hf is a host temporary
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
