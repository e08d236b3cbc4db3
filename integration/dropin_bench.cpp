// integration/dropin_bench.cpp -- times the reference's own public API,
// cg::countgauss_apply(t, DenseMatrix / SparseMatrix) (sketch.cpp:132-138), exactly as a
// reference caller uses it: fp64 column-major DenseMatrix or int64/fp64 CSR in pageable
// std::vector storage, transform from cg::countgauss_new.  Linked twice by oracle/Makefile:
// against integration/countgauss_gpu.cpp + libcgx.so (the drop-in, "gpu") and against the
// reference's sketch.cpp (the CPU library, "cpu"), so both numbers come from one program.
//
//   dropin_bench <c1|c2|c3|c3s|c4> <reps> [fp64]
//
// Inputs: c2/c4 dense N(0,1) values rounded to fp32 and widened (BASELINE's configs hold
// fp32 entries) -- or, with "fp64", full-precision doubles; c3 is CSR 1% with
// random_sparse-style rows (sorted distinct columns).  Prints one JSON line: median ms of
// `reps` applies after one warm-up, nnz/s, and a checksum of Z.
#include "countgauss/matrix.hpp"
#include "countgauss/rng.hpp"
#include "countgauss/sketch.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

using namespace cg;

static double now_ms() {
    using clock = std::chrono::steady_clock;
    return std::chrono::duration<double, std::milli>(clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
    const std::string cfg = argc > 1 ? argv[1] : "c2";
    const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
    const bool full64 = argc > 3 && std::string(argv[3]) == "fp64";
    index_t n, d, B, m;
    if (cfg == "c1") {
        n = 65536, d = 8, B = 2048, m = 16;
    } else if (cfg == "c2") {
        n = (index_t)1 << 24, d = 32, B = 65536, m = 64;
    } else if (cfg == "c4") {
        n = (index_t)1 << 25, d = 128, B = 131072, m = 32;
    } else if (cfg == "c3") {
        n = (index_t)1 << 26, d = 256, B = 262144, m = 128;
    } else if (cfg == "c3s") {  // c3's shape at 1/64 of the rows (test-sized CSR)
        n = (index_t)1 << 20, d = 256, B = 16384, m = 128;
    } else {
        std::fprintf(stderr, "unknown config %s\n", cfg.c_str());
        return 2;
    }
    SeededRng t_rng(12345);
    const double t0 = now_ms();
    CountGaussTransform t = countgauss_new(m, B, n, t_rng);
    const double construct_ms = now_ms() - t0;
    DenseMatrix z;
    std::vector<double> ms;
    double units = 0, in_bytes = 0;
    if (cfg == "c3" || cfg == "c3s") {
        SparseMatrix x;
        x.rows = n;
        x.cols = d;
        x.row_offsets.assign((std::size_t)n + 1, 0);
        // Bernoulli(0.01) entries per row, values N(0,1) (fp64), one counter stream per row
        std::vector<index_t> len((std::size_t)n);
#pragma omp parallel for schedule(static)
        for (index_t i = 0; i < n; ++i) {
            SeededRng r(mix64(777, (std::uint64_t)i));
            index_t c = 0;
            for (index_t j = 0; j < d; ++j) c += r.next_uniform() < 0.01;
            len[(std::size_t)i] = c;
        }
        for (index_t i = 0; i < n; ++i) x.row_offsets[(std::size_t)i + 1] = x.row_offsets[(std::size_t)i] + len[(std::size_t)i];
        x.col_indices.resize((std::size_t)x.row_offsets.back());
        x.values.resize((std::size_t)x.row_offsets.back());
#pragma omp parallel for schedule(static)
        for (index_t i = 0; i < n; ++i) {
            SeededRng r(mix64(777, (std::uint64_t)i));
            index_t p = x.row_offsets[(std::size_t)i];
            for (index_t j = 0; j < d; ++j)
                if (r.next_uniform() < 0.01) x.col_indices[(std::size_t)p++] = j;
            SeededRng v(mix64(778, (std::uint64_t)i));
            for (index_t q = x.row_offsets[(std::size_t)i]; q < p; ++q) {
                const double g = v.next_normal();
                x.values[(std::size_t)q] = full64 ? g : (double)(float)g;
            }
        }
        units = (double)x.nnz();
        in_bytes = 16.0 * x.nnz() + 8.0 * (n + 1);
        z = countgauss_apply(t, x);
        for (int k = 0; k < reps; ++k) {
            const double a = now_ms();
            z = countgauss_apply(t, x);
            ms.push_back(now_ms() - a);
        }
    } else {
        DenseMatrix x(n, d);
        double* p = x.data();
#pragma omp parallel for schedule(static)
        for (index_t j = 0; j < d; ++j) {
            SeededRng r(mix64(779, (std::uint64_t)j));
            for (index_t i = 0; i < n; ++i) {
                const double g = r.next_normal();
                p[j * n + i] = full64 ? g : (double)(float)g;
            }
        }
        units = (double)n * d;
        in_bytes = 8.0 * n * d;
        z = countgauss_apply(t, x);
        for (int k = 0; k < reps; ++k) {
            const double a = now_ms();
            z = countgauss_apply(t, x);
            ms.push_back(now_ms() - a);
        }
    }
    std::sort(ms.begin(), ms.end());
    const double med = ms[ms.size() / 2];
    double zsum = 0.0;
    for (index_t k = 0; k < z.size(); ++k) zsum += std::abs(z.data()[k]);
    std::printf("{\"config\": \"%s\", \"values\": \"%s\", \"ms\": %.4f, \"min_ms\": %.4f, \"reps\": %d, "
                "\"nnz_per_s\": %.6e, \"input_bytes\": %.0f, \"construct_ms\": %.2f, \"z_abs_sum\": %.17g}\n",
                cfg.c_str(), full64 ? "fp64" : "fp32-valued fp64", med, ms.front(), reps, units / (med / 1e3), in_bytes,
                construct_ms, zsum);
    return 0;
}
