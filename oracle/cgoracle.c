/* oracle/cgoracle.c -- TEST INFRASTRUCTURE ONLY: the CPU restatement of the reference
 * CountGauss path used as the parity checker.  Nothing in the product
 * (paper_1606_05732_b200/) links, loads or calls this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg do.
 *
 * Each function restates the reference algorithm it cites (paths relative to
 * /root/reference/proj).  It is pinned two ways (tests/test_oracle.py):
 *   - against golden vectors produced by the compiled reference
 *     (tests/golden/make_golden.py -> tests/golden/*.npz), and
 *   - directly against oracle/_ref/libcgref.so (the reference itself, built
 *     by oracle/Makefile) on seeded random cases, bit-for-bit.
 *
 * Build with -ffp-contract=off: the reference Release objects contain no FMA
 * (SURVEY.md 8c), and the oracle must round exactly as they do.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9E3779B97F4A7C15ULL

/* SplitMix64 finalizer F(z)  (include/countgauss/rng.hpp:31-37). */
static inline uint64_t fin(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* mix64(a, b)  (include/countgauss/rng.hpp:12-17). */
uint64_t cgo_mix64(uint64_t a, uint64_t b) { return fin(a + GAMMA + b * 0xBF58476D1CE4E5B9ULL); }

/* Draw k (0-based) of SeededRng(seed): state advances by GAMMA before each draw
 * (rng.hpp:31-37), so draw k is F(seed + (k+1)*GAMMA). */
uint64_t cgo_draw(uint64_t seed, uint64_t k) { return fin(seed + (k + 1) * GAMMA); }

/* next_uniform: ((u >> 11) + 0.5) * 2^-53  (rng.hpp:40-42). */
static inline double uniform53(uint64_t u) { return ((double)(u >> 11) + 0.5) * 0x1.0p-53; }

/* Acklam's rational approximation (src/rng.cpp:13-41). */
static double acklam(double p) {
    static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                               1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                               6.680131188771972e+01,  -1.328068155288572e+01};
    static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                               -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
    static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                               3.754408661907416e+00};
    const double p_low = 0.02425;
    if (p < p_low) {
        double q = sqrt(-2.0 * log(p));
        return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
               ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
    }
    if (p <= 1.0 - p_low) {
        double q = p - 0.5, r = q * q;
        return (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
               (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
    }
    double q = sqrt(-2.0 * log(1.0 - p));
    return -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
           ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
}

/* inverse_normal_cdf: Acklam + one Halley step against erfc (src/rng.cpp:45-55).
 * Returns NAN outside (0,1) where the reference throws std::invalid_argument. */
double cgo_inverse_normal_cdf(double p) {
    if (!(p > 0.0 && p < 1.0)) return NAN;
    double x = acklam(p);
    const double sqrt2pi = 2.5066282746310005024;
    const double sqrt2 = 1.41421356237309504880; /* std::numbers::sqrt2 */
    double e = 0.5 * erfc(-x / sqrt2) - p;
    double u = e * sqrt2pi * exp(0.5 * x * x);
    x -= u / (1.0 + 0.5 * x * u);
    return x;
}

/* Seed plumbing of countgauss_new (src/sketch.cpp:115-126) for caller rng
 * SeededRng(caller_seed): t.seed = draw 0; cs_rng = SeededRng(mix64(t.seed,1)),
 * map.seed = cs_rng.next_u64() (sketch.cpp:18); g_rng = SeededRng(mix64(t.seed,2)). */
void cgo_countgauss_seeds(uint64_t caller_seed, uint64_t* t_seed, uint64_t* cs_seed, uint64_t* g_seed) {
    uint64_t t = cgo_draw(caller_seed, 0);
    *t_seed = t;
    *cs_seed = cgo_draw(cgo_mix64(t, 1), 0);
    *g_seed = cgo_mix64(t, 2);
}

/* countsketch_new body (src/sketch.cpp:21-26): per row i, hash = draw 2i mod B,
 * sign = +1 iff draw 2i+1 is odd.  Rows [i0, i0+count). */
void cgo_hash_sign(uint64_t cs_seed, int64_t B, int64_t i0, int64_t count, int64_t* hash, double* sign) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < count; ++k) {
        uint64_t i = (uint64_t)(i0 + k);
        hash[k] = (int64_t)(cgo_draw(cs_seed, 2 * i) % (uint64_t)B);
        sign[k] = (cgo_draw(cs_seed, 2 * i + 1) & 1ULL) ? 1.0 : -1.0;
    }
}

/* gaussian_matrix(m, B, g_rng) (src/matrix.cpp:199-207): column-major draw order,
 * G[r + c*m] = inverse_normal_cdf(uniform(draw c*m + r)).  Columns [c0, c0+nc). */
void cgo_gaussian(uint64_t g_seed, int64_t m, int64_t c0, int64_t nc, double* g) {
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nc; ++c)
        for (int64_t r = 0; r < m; ++r) {
            uint64_t k = (uint64_t)((c0 + c) * m + r);
            g[c * m + r] = cgo_inverse_normal_cdf(uniform53(cgo_draw(g_seed, k)));
        }
}

/* countsketch_apply(map, DenseMatrix) (src/sketch.cpp:52-66): out(B x d, col-major) starts
 * at +0.0 and, per column, adds sign[i]*x(i,j) over ascending i.  x is addressed as
 * x[i*rs + j*cs] so col-major (rs=1, cs=ld) and row-major (rs=ld, cs=1) share one loop;
 * xf32 != 0 reads float entries widened exactly to double. */
void cgo_sketch_dense(const int64_t* hash, const double* sign, int64_t B, const void* x, int xf32,
                      int64_t n, int64_t d, int64_t rs, int64_t cs, double* out) {
    memset(out, 0, sizeof(double) * (size_t)(B * d));
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < d; ++j) {
        double* oj = out + j * B;
        for (int64_t i = 0; i < n; ++i) {
            double v = xf32 ? (double)((const float*)x)[i * rs + j * cs] : ((const double*)x)[i * rs + j * cs];
            oj[hash[i]] += sign[i] * v;
        }
    }
}

/* countsketch_apply(map, SparseMatrix) (src/sketch.cpp:68-113), both branches: the serial
 * row loop when !chunked, and 8192-row chunks with per-chunk partial buffers reduced in
 * ascending chunk order when n_chunks > 1 && B*d <= 2^16 && n_chunks*B*d <= 2^25.
 * col index type: cols64 != 0 -> int64, else int32; vals: vf32 != 0 -> float. */
void cgo_sketch_csr(const int64_t* hash, const double* sign, int64_t B, const int64_t* rowptr,
                    const void* cols, int cols64, const void* vals, int vf32, int64_t n, int64_t d,
                    double* out) {
    const int64_t chunk_rows = 8192;
    const int64_t n_chunks = (n + chunk_rows - 1) / chunk_rows;
    const int64_t out_size = B * d;
    const int chunked = n_chunks > 1 && out_size <= (1LL << 16) && n_chunks * out_size <= (1LL << 25);
    memset(out, 0, sizeof(double) * (size_t)out_size);
#define COL(q) (cols64 ? ((const int64_t*)cols)[q] : (int64_t)((const int32_t*)cols)[q])
#define VAL(q) (vf32 ? (double)((const float*)vals)[q] : ((const double*)vals)[q])
    if (!chunked) {
        for (int64_t i = 0; i < n; ++i) {
            const int64_t b = hash[i];
            const double s = sign[i];
            for (int64_t q = rowptr[i]; q < rowptr[i + 1]; ++q) out[COL(q) * B + b] += s * VAL(q);
        }
        return;
    }
    double* partial = (double*)calloc((size_t)(n_chunks * out_size), sizeof(double));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n_chunks; ++c) {
        double* buf = partial + c * out_size;
        const int64_t lo = c * chunk_rows, hi = lo + chunk_rows < n ? lo + chunk_rows : n;
        for (int64_t i = lo; i < hi; ++i) {
            const int64_t b = hash[i];
            const double s = sign[i];
            for (int64_t q = rowptr[i]; q < rowptr[i + 1]; ++q) buf[COL(q) * B + b] += s * VAL(q);
        }
    }
    for (int64_t c = 0; c < n_chunks; ++c) {
        const double* buf = partial + c * out_size;
        for (int64_t e = 0; e < out_size; ++e) out[e] += buf[e];
    }
    free(partial);
#undef COL
#undef VAL
}

/* gemm(A, B) (src/matrix.cpp:111-129): col-major; per output column, ascending inner
 * index, zero B entries skipped, separate multiply and add (no FMA). */
void cgo_gemm(const double* a, int64_t ar, int64_t ac, const double* b, int64_t bc, double* c) {
    memset(c, 0, sizeof(double) * (size_t)(ar * bc));
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < bc; ++j) {
        double* cj = c + j * ar;
        const double* bj = b + j * ac;
        for (int64_t l = 0; l < ac; ++l) {
            const double blj = bj[l];
            if (blj == 0.0) continue;
            const double* al = a + l * ar;
            for (int64_t i = 0; i < ar; ++i) cj[i] += al[i] * blj;
        }
    }
}

/* select_extremes(Z) per row (src/nmf.cpp:99-118): strict compares so ties go to the
 * lowest column index; a row is a tie row if its max or its min is attained more than
 * once.  z is col-major m x d.  Returns tie_rows; i_max/i_min are the raw per-row
 * indices (the sorted-unique union is taken by the caller, nmf.cpp:119-131). */
int64_t cgo_select_extremes(const double* z, int64_t m, int64_t d, int64_t* amax_out, int64_t* amin_out) {
    int64_t tie_rows = 0;
    for (int64_t r = 0; r < m; ++r) {
        int64_t amax = 0, amin = 0, max_hits = 1, min_hits = 1;
        double vmax = z[r], vmin = z[r];
        for (int64_t j = 1; j < d; ++j) {
            const double v = z[j * m + r];
            if (v > vmax) { vmax = v; amax = j; max_hits = 1; }
            else if (v == vmax) ++max_hits;
            if (v < vmin) { vmin = v; amin = j; min_hits = 1; }
            else if (v == vmin) ++min_hits;
        }
        if (max_hits > 1 || min_hits > 1) ++tie_rows;
        amax_out[r] = amax;
        amin_out[r] = amin;
    }
    return tie_rows;
}

/* ---- synthetic inputs (shared definition with the GPU generator, csrc/datagen.cu) ----
 * Entry e of stream `seed` uses u = uniform53(draw(seed, e)).  Normal entries are the
 * fp64 Acklam quantile of u rounded to fp32 (the Halley step is below fp32 resolution).
 * CUDA's log differs from glibc's by <= 1 ulp in the tails, so a CPU-regenerated entry
 * can (rarely) differ by 1 fp32 ulp from the GPU's: parity tests therefore copy the GPU
 * bytes instead of regenerating them here. */
float cgo_normal_f32(uint64_t seed, uint64_t e) { return (float)acklam(uniform53(cgo_draw(seed, e))); }

/* Dense n x d fp32, element (i,j) = stream entry i*d + j; written row-major. */
void cgo_gen_dense_f32(uint64_t seed, int64_t n, int64_t d, float* x) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < d; ++j) x[i * d + j] = cgo_normal_f32(seed, (uint64_t)(i * d + j));
}

/* Same values, written column-major fp64 (the reference DenseMatrix layout). */
void cgo_gen_dense_f64_colmajor(uint64_t seed, int64_t n, int64_t d, double* x) {
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < d; ++j)
        for (int64_t i = 0; i < n; ++i) x[j * n + i] = (double)cgo_normal_f32(seed, (uint64_t)(i * d + j));
}

/* ---- config 4: near-separable X (twin of csrc/datagen.cu gen_separable_kernel and
 * separable_mixing; BASELINE configs[3]) ---------------------------------------------
 * Mixing weights: column c of H (r x cols, column-major) is Dirichlet(alpha), the
 * normalized Marsaglia-Tsang Gamma(alpha) draws of the sequential stream
 * SeededRng(mix64(seed, 13)); normals there are Acklam's rational (src/rng.cpp:13-41). */
static double sep_gamma(uint64_t seed, uint64_t* k, double alpha) {
    if (alpha < 1.0) {
        double g = sep_gamma(seed, k, alpha + 1.0);
        double u = uniform53(cgo_draw(seed, (*k)++));
        return g * pow(u, 1.0 / alpha);
    }
    double dm = alpha - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * dm);
    for (;;) {
        double z = acklam(uniform53(cgo_draw(seed, (*k)++)));
        double v = 1.0 + c * z;
        if (v <= 0.0) continue;
        v = v * v * v;
        double u = uniform53(cgo_draw(seed, (*k)++));
        if (log(u) < 0.5 * z * z + dm - dm * v + dm * log(v)) return dm * v;
    }
}

void cgo_separable_mixing(uint64_t seed, int64_t r, int64_t cols, double alpha, double* h) {
    uint64_t hseed = cgo_mix64(seed, 13), k = 0;
    for (int64_t c = 0; c < cols; ++c) {
        double* hc = h + c * r;
        double sum = 0.0;
        for (int64_t q = 0; q < r; ++q) {
            hc[q] = sep_gamma(hseed, &k, alpha);
            sum += hc[q];
        }
        for (int64_t q = 0; q < r; ++q) hc[q] = sum > 0.0 ? hc[q] / sum : 1.0 / (double)r;
    }
}

/* X = max(A.[I_r | H] + sigma*N, 0), rows [row0, row0+n) written row-major fp32; every
 * product and sum rounded in fp32 (this file is built with -ffp-contract=off), ascending k.
 * The noise term is cgo_normal_f32, so entries can differ from the GPU's where that
 * normal does (a 1-ulp libm difference in the far tails; see above). */
static void sep_rows(uint64_t seed, int64_t row0, int64_t i, int64_t d, int64_t r, float sg, const float* hf,
                     float* xi) {
    int64_t hc = d - r;
    uint64_t aseed = cgo_mix64(seed, 11), nseed = cgo_mix64(seed, 12);
    uint64_t gi = (uint64_t)(row0 + i);
    float a[64];
    for (int64_t k = 0; k < r && k < 64; ++k) a[k] = (float)(cgo_draw(aseed, gi * (uint64_t)r + (uint64_t)k) >> 40) * 0x1.0p-24f;
    for (int64_t j = 0; j < d; ++j) {
        float base;
        if (j < r) {
            base = a[j];
        } else {
            base = 0.0f;
            for (int64_t k = 0; k < r; ++k) base = base + a[k] * hf[k * hc + (j - r)];
        }
        float v = base + sg * cgo_normal_f32(nseed, gi * (uint64_t)d + (uint64_t)j);
        xi[j] = v > 0.0f ? v : 0.0f;
    }
}

static float* sep_hf(uint64_t seed, int64_t d, int64_t r, double alpha) {
    int64_t hc = d - r;
    double* h = (double*)malloc(sizeof(double) * (size_t)(r * (hc > 0 ? hc : 1)));
    float* hf = (float*)malloc(sizeof(float) * (size_t)(r * (hc > 0 ? hc : 1)));
    cgo_separable_mixing(seed, r, hc, alpha, h);
    for (int64_t k = 0; k < r; ++k)
        for (int64_t c = 0; c < hc; ++c) hf[k * hc + c] = (float)h[c * r + k];
    free(h);
    return hf;
}

/* X = max(A.[I_r | H] + sigma*N, 0), rows [row0, row0+n) written row-major fp32; every
 * product and sum rounded in fp32 (this file is built with -ffp-contract=off), ascending k
 * (r <= 64).  The noise term is cgo_normal_f32, so entries can differ from the GPU's where
 * that normal does (a 1-ulp libm difference in the far tails; see above). */
void cgo_gen_separable_f32(uint64_t seed, int64_t row0, int64_t n, int64_t d, int64_t r, double alpha, double sigma,
                           float* x) {
    float* hf = sep_hf(seed, d, r, alpha);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) sep_rows(seed, row0, i, d, r, (float)sigma, hf, x + i * d);
    free(hf);
}

/* Rows [b0, b1) of countsketch_apply(map, SparseMatrix)'s serial branch
 * (src/sketch.cpp:84-91): out ((b1-b0) x d, column-major) starts at +0.0 and takes every
 * row i with hash in [b0, b1), in ascending i -- the exact per-(bucket, column) order of
 * the full serial loop, so these rows are bit-identical to the full result's.  A
 * full-size parity check that touches only the rows of a bucket range. */
void cgo_sketch_csr_buckets(const int64_t* hash, const double* sign, int64_t b0, int64_t b1, const int64_t* rowptr,
                            const void* cols, int cols64, const void* vals, int vf32, int64_t n, int64_t d,
                            double* out) {
    const int64_t nb = b1 - b0;
    memset(out, 0, sizeof(double) * (size_t)(nb * d));
    for (int64_t i = 0; i < n; ++i) {
        const int64_t b = hash[i];
        if (b < b0 || b >= b1) continue;
        const double s = sign[i];
        for (int64_t q = rowptr[i]; q < rowptr[i + 1]; ++q) {
            const int64_t c = cols64 ? ((const int64_t*)cols)[q] : (int64_t)((const int32_t*)cols)[q];
            const double v = vf32 ? (double)((const float*)vals)[q] : ((const double*)vals)[q];
            out[c * nb + (b - b0)] += s * v;
        }
    }
}

/* The same matrix written column-major fp64 (the reference DenseMatrix layout), rows
 * [0, n): the CPU input of the config-4 reference arm.  Row blocks keep the writes to
 * each column contiguous. */
void cgo_gen_separable_f64_colmajor(uint64_t seed, int64_t n, int64_t d, int64_t r, double alpha, double sigma,
                                    double* x) {
    const int64_t blk = 2048;
    float* hf = sep_hf(seed, d, r, alpha);
#pragma omp parallel
    {
        float* tmp = (float*)malloc(sizeof(float) * (size_t)(blk * d));
#pragma omp for schedule(dynamic, 4)
        for (int64_t b = 0; b < (n + blk - 1) / blk; ++b) {
            int64_t i0 = b * blk, cnt = n - i0 < blk ? n - i0 : blk;
            for (int64_t i = 0; i < cnt; ++i) sep_rows(seed, 0, i0 + i, d, r, (float)sigma, hf, tmp + i * d);
            for (int64_t j = 0; j < d; ++j)
                for (int64_t i = 0; i < cnt; ++i) x[j * n + i0 + i] = (double)tmp[i * d + j];
        }
        free(tmp);
    }
    free(hf);
}
