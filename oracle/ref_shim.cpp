// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" wrapper around the *unmodified* reference library
// (/root/reference/proj/src/{rng,matrix,linalg,sketch,reference,nmf}.cpp), compiled
// by oracle/Makefile into oracle/_ref/libcgref.so.  Only tests/, bench.py's
// cpu_baseline / --impl reference arm and __graft_entry__.smoke() may load it.
//
// Every entry point forwards to the reference symbol it names; nothing here
// re-implements the algorithm (that is oracle/cgoracle.c's job).  Exceptions are
// caught at the boundary and turned into status codes: 0 ok, 1 invalid_argument,
// 2 other exception.
#include "countgauss/matrix.hpp"
#include "countgauss/nmf.hpp"
#include "countgauss/reference.hpp"
#include "countgauss/rng.hpp"
#include "countgauss/sketch.hpp"

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace cg;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

DenseMatrix from_colmajor(const double* x, index_t rows, index_t cols) {
    DenseMatrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data(), x, sizeof(double) * static_cast<std::size_t>(rows * cols));
    return m;
}

void to_colmajor(const DenseMatrix& m, double* out) {
    if (m.size()) std::memcpy(out, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
}

SparseMatrix from_csr(const int64_t* rowptr, const int64_t* cols, const double* vals, index_t n,
                      index_t d) {
    SparseMatrix s;
    s.rows = n;
    s.cols = d;
    s.row_offsets.assign(rowptr, rowptr + n + 1);
    const index_t nnz = rowptr[n];
    s.col_indices.assign(cols, cols + nnz);
    s.values.assign(vals, vals + nnz);
    return s;
}

double now_ms() {
    using clock = std::chrono::steady_clock;
    return std::chrono::duration<double, std::milli>(clock::now().time_since_epoch()).count();
}
} // namespace

extern "C" {

const char* cgref_last_error(void) { return g_err.c_str(); }

void cgref_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

int cgref_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

uint64_t cgref_mix64(uint64_t a, uint64_t b) { return mix64(a, b); }

// First `count` next_u64 draws of SeededRng(seed)  (rng.hpp:31-37).
void cgref_rng_u64(uint64_t seed, int64_t count, uint64_t* out) {
    SeededRng r(seed);
    for (int64_t k = 0; k < count; ++k) out[k] = r.next_u64();
}

// First `count` next_normal draws of SeededRng(seed)  (rng.cpp:57-59).
void cgref_rng_normal(uint64_t seed, int64_t count, double* out) {
    SeededRng r(seed);
    for (int64_t k = 0; k < count; ++k) out[k] = r.next_normal();
}

int cgref_inverse_normal_cdf(double p, double* out) {
    return guard([&] { *out = inverse_normal_cdf(p); });
}

// ---- transforms -------------------------------------------------------------------

struct cgref_xform {
    CountGaussTransform t;
    bool has_g = false;
};

// countgauss_new(m, B, n, SeededRng(caller_seed))  (sketch.cpp:115-126).  B < 1 selects
// the two-argument overload's default B = 5m (sketch.cpp:128-130).
int cgref_countgauss_new(int64_t m, int64_t B, int64_t n, uint64_t caller_seed, void** out) {
    return guard([&] {
        SeededRng rng(caller_seed);
        auto* x = new cgref_xform;
        try {
            x->t = B < 1 ? countgauss_new(m, n, rng) : countgauss_new(m, B, n, rng);
        } catch (...) {
            delete x;
            throw;
        }
        x->has_g = true;
        *out = x;
    });
}

// countsketch_new(B, n, SeededRng(caller_seed))  (sketch.cpp:12-28).
int cgref_countsketch_new(int64_t B, int64_t n, uint64_t caller_seed, void** out) {
    return guard([&] {
        SeededRng rng(caller_seed);
        auto* x = new cgref_xform;
        try {
            x->t.cs = countsketch_new(B, n, rng);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

// countsketch_injective(B, n, SeededRng(caller_seed))  (sketch.cpp:30-50).
int cgref_countsketch_injective(int64_t B, int64_t n, uint64_t caller_seed, void** out) {
    return guard([&] {
        SeededRng rng(caller_seed);
        auto* x = new cgref_xform;
        try {
            x->t.cs = countsketch_injective(B, n, rng);
        } catch (...) {
            delete x;
            throw;
        }
        *out = x;
    });
}

// Hand-built map (test_sketch.cpp:72-92 style): explicit hash/sign, optional G (m x B col-major).
int cgref_xform_explicit(int64_t B, int64_t n, const int64_t* hash, const double* sign, int64_t m,
                         const double* g, void** out) {
    return guard([&] {
        auto* x = new cgref_xform;
        x->t.cs.buckets = B;
        x->t.cs.input_dim = n;
        x->t.cs.hash.assign(hash, hash + n);
        x->t.cs.sign.assign(sign, sign + n);
        if (g && m > 0) {
            x->t.g = from_colmajor(g, m, B);
            x->t.m = m;
            x->has_g = true;
        }
        *out = x;
    });
}

void cgref_xform_free(void* h) { delete static_cast<cgref_xform*>(h); }

void cgref_xform_info(void* h, uint64_t* t_seed, uint64_t* cs_seed, int64_t* m, int64_t* B, int64_t* n) {
    auto* x = static_cast<cgref_xform*>(h);
    *t_seed = x->t.seed;
    *cs_seed = x->t.cs.seed;
    *m = x->t.m;
    *B = x->t.cs.buckets;
    *n = x->t.cs.input_dim;
}

void cgref_xform_hash_sign(void* h, int64_t* hash, double* sign) {
    auto* x = static_cast<cgref_xform*>(h);
    std::copy(x->t.cs.hash.begin(), x->t.cs.hash.end(), hash);
    std::copy(x->t.cs.sign.begin(), x->t.cs.sign.end(), sign);
}

void cgref_xform_g(void* h, double* g) { to_colmajor(static_cast<cgref_xform*>(h)->t.g, g); }

// ---- matrices held on the reference side (so timing excludes the copy-in) ----------

int cgref_dense_new(const double* x_colmajor, int64_t n, int64_t d, void** out) {
    return guard([&] { *out = new DenseMatrix(from_colmajor(x_colmajor, n, d)); });
}
void cgref_dense_free(void* h) { delete static_cast<DenseMatrix*>(h); }

// A zero-filled n x d DenseMatrix whose storage the caller fills in place (so multi-GB
// bench inputs are not held twice).
int cgref_dense_alloc(int64_t n, int64_t d, void** out, double** data) {
    return guard([&] {
        auto* m = new DenseMatrix(n, d);
        *out = m;
        *data = m->data();
    });
}

int cgref_csr_new(const int64_t* rowptr, const int64_t* cols, const double* vals, int64_t n, int64_t d,
                  void** out) {
    return guard([&] {
        auto* s = new SparseMatrix(from_csr(rowptr, cols, vals, n, d));
        *out = s;
    });
}
void cgref_csr_free(void* h) { delete static_cast<SparseMatrix*>(h); }

// kind: 0 countsketch_apply (sketch.cpp:52-113), 1 countgauss_apply (sketch.cpp:132-138),
//       2 reference::countsketch_apply serial (reference.cpp:44-67).
// sparse: 0 -> xh is a DenseMatrix*, 1 -> SparseMatrix*.
int cgref_apply(void* xf, void* xh, int sparse, int kind, double* out) {
    return guard([&] {
        const auto& t = static_cast<cgref_xform*>(xf)->t;
        DenseMatrix r;
        if (sparse) {
            const auto& x = *static_cast<SparseMatrix*>(xh);
            r = kind == 0 ? countsketch_apply(t.cs, x)
                : kind == 1 ? countgauss_apply(t, x)
                            : reference::countsketch_apply(t.cs, x);
        } else {
            const auto& x = *static_cast<DenseMatrix*>(xh);
            r = kind == 0 ? countsketch_apply(t.cs, x)
                : kind == 1 ? countgauss_apply(t, x)
                            : reference::countsketch_apply(t.cs, x);
        }
        to_colmajor(r, out);
    });
}

// distcheck's trial loop body (distcheck.cpp:107-113) for trials [t0, t0+trials):
// SeededRng(mix64(master, t)) -> countsketch_new -> countsketch_apply(map, U) -> gram.
// su (trials x B x d) and gram (trials x d x d), each column-major; either may be null.
int cgref_sketch_gram_trials(uint64_t master, int64_t t0, int64_t trials, int64_t B, const double* u_colmajor,
                             int64_t n, int64_t d, double* su, double* gm) {
    return guard([&] {
        DenseMatrix u(n, d);
        std::memcpy(u.data(), u_colmajor, sizeof(double) * (size_t)(n * d));
#pragma omp parallel for schedule(static)  // as the reference's trial loop
        for (int64_t t = 0; t < trials; ++t) {
            SeededRng trial_rng(mix64(master, static_cast<std::uint64_t>(t0 + t)));
            CountSketchMap s = countsketch_new(B, n, trial_rng);
            DenseMatrix r = countsketch_apply(s, u);
            if (su) to_colmajor(r, su + t * B * d);
            if (gm) to_colmajor(gram(r), gm + t * d * d);
        }
    });
}

// Times `reps` calls of cgref_apply after one warm-up, like timed_median_ms
// (countgauss_main.cpp:96-108); writes every sample (ms).
int cgref_time_apply(void* xf, void* xh, int sparse, int kind, int reps, double* ms_out, double* out) {
    int rc = cgref_apply(xf, xh, sparse, kind, out);
    for (int i = 0; i < reps && rc == 0; ++i) {
        const double t0 = now_ms();
        rc = cgref_apply(xf, xh, sparse, kind, out);
        ms_out[i] = now_ms() - t0;
    }
    return rc;
}

// gemm(A, B)  (matrix.cpp:111-129), col-major in/out.
int cgref_gemm(const double* a, int64_t ar, int64_t ac, const double* b, int64_t br, int64_t bc, double* c) {
    return guard([&] { to_colmajor(gemm(from_colmajor(a, ar, ac), from_colmajor(b, br, bc)), c); });
}

// reference::matmul(reference::materialize(S), X)  (reference.cpp:13-42): the dense oracle
// the reference's own exactness tests compare against (test_sketch.cpp:94-109).
int cgref_materialized_sketch(void* xf, const double* x, int64_t n, int64_t d, double* out) {
    return guard([&] {
        const auto& t = static_cast<cgref_xform*>(xf)->t;
        to_colmajor(reference::matmul(reference::materialize(t.cs), from_colmajor(x, n, d)), out);
    });
}

// cg_nmf(X, m, B, SeededRng(caller_seed))  (nmf.cpp:141-153).  Outputs are written into
// caller arrays of capacity >= m (i_max, i_min) and >= 2m (unioned).
int cgref_cg_nmf(void* xh, int sparse, int64_t m, int64_t B, uint64_t caller_seed, int64_t* i_max,
                 int64_t* n_max, int64_t* i_min, int64_t* n_min, int64_t* unioned, int64_t* n_union,
                 int64_t* tie_rows) {
    return guard([&] {
        SeededRng rng(caller_seed);
        AnchorSet a = sparse ? cg_nmf(*static_cast<SparseMatrix*>(xh), m, B, rng)
                             : cg_nmf(*static_cast<DenseMatrix*>(xh), m, B, rng);
        std::copy(a.i_max.begin(), a.i_max.end(), i_max);
        std::copy(a.i_min.begin(), a.i_min.end(), i_min);
        std::copy(a.unioned.begin(), a.unioned.end(), unioned);
        *n_max = static_cast<int64_t>(a.i_max.size());
        *n_min = static_cast<int64_t>(a.i_min.size());
        *n_union = static_cast<int64_t>(a.unioned.size());
        *tie_rows = a.tie_rows;
    });
}

// gp_nmf(X, m, SeededRng(caller_seed))  (nmf.cpp:155-159), dense X only; same outputs as
// cgref_cg_nmf.
int cgref_gp_nmf(void* xh, int64_t m, uint64_t caller_seed, int64_t* i_max, int64_t* n_max, int64_t* i_min,
                 int64_t* n_min, int64_t* unioned, int64_t* n_union, int64_t* tie_rows) {
    return guard([&] {
        SeededRng rng(caller_seed);
        AnchorSet a = gp_nmf(*static_cast<DenseMatrix*>(xh), m, rng);
        std::copy(a.i_max.begin(), a.i_max.end(), i_max);
        std::copy(a.i_min.begin(), a.i_min.end(), i_min);
        std::copy(a.unioned.begin(), a.unioned.end(), unioned);
        *n_max = static_cast<int64_t>(a.i_max.size());
        *n_min = static_cast<int64_t>(a.i_min.size());
        *n_union = static_cast<int64_t>(a.unioned.size());
        *tie_rows = a.tie_rows;
    });
}

// random_sparse(rows, cols, per_row, SeededRng(seed))  (matrix.cpp:209-233): the reference's own
// bench input generator; output sized rows*per_row.
int cgref_random_sparse(int64_t rows, int64_t cols, int64_t per_row, uint64_t seed, int64_t* rowptr,
                        int64_t* col_idx, double* vals) {
    return guard([&] {
        SeededRng rng(seed);
        SparseMatrix s = random_sparse(rows, cols, per_row, rng);
        std::copy(s.row_offsets.begin(), s.row_offsets.end(), rowptr);
        std::copy(s.col_indices.begin(), s.col_indices.end(), col_idx);
        std::copy(s.values.begin(), s.values.end(), vals);
    });
}

// generate_separable(d, n, k, SeededRng(seed)).x  (nmf.cpp:12-44), col-major d x n.
int cgref_generate_separable(int64_t d, int64_t n, int64_t k, uint64_t seed, double* x) {
    return guard([&] {
        SeededRng rng(seed);
        auto inst = generate_separable(d, n, k, rng);
        to_colmajor(inst.x, x);
    });
}

} // extern "C"
