// integration/countgauss_gpu.cpp -- the reference-side binding: a drop-in replacement for
// the CountSketch / CountGauss functions of the reference's proj/src/sketch.cpp
// (declared in proj/include/countgauss/sketch.hpp:25-54), implemented on the B200
// through the cgx C-ABI (include/cgx.h, libcgx.so).
//
// A maintainer adds this file to countgauss_core in place of those functions (SRHT stays
// in sketch.cpp) and links libcgx.so; every caller -- cg_nmf (nmf.cpp:141-153), distcheck,
// the CLI bench, the tests -- then runs on the GPU unchanged.  oracle/Makefile builds the
// reference's own acceptance binary against it (oracle/_ref/acceptance_gpu) as the
// drop-in regression test.
//
// Semantics kept from the reference:
//  * each constructor consumes exactly one caller-rng draw (sketch.cpp:17,36,120);
//  * the public struct fields (cs.hash, cs.sign, g) are materialized, so code that reads
//    or hand-edits them keeps working; apply uses whatever the fields hold (they are
//    shipped to the GPU as an explicit map / explicit G on each call);
//  * std::invalid_argument with the reference's messages; CGX_ERANGE -> length_error;
//  * thread safety: one process-wide context, calls serialized inside libcgx (the
//    reference calls these from OpenMP regions, distcheck.cpp:107-111).
#include "countgauss/sketch.hpp"

#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "cgx.h"

namespace cg {
namespace {

void check(int rc) {
    if (rc == CGX_OK) return;
    const std::string msg = cgx_last_error();
    if (rc == CGX_EINVAL) throw std::invalid_argument(msg);
    if (rc == CGX_ERANGE) throw std::length_error(msg);
    if (rc == CGX_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error("cgx: " + msg);
}

cgx_ctx* context() {
    static std::once_flag once;
    static cgx_ctx* ctx = nullptr;
    std::call_once(once, [] {
        const char* dev = std::getenv("CGX_DEVICE");
        check(cgx_init(dev ? std::atoi(dev) : 0, &ctx));
    });
    return ctx;
}

struct Xform {
    cgx_xform* h = nullptr;
    ~Xform() {
        if (h) cgx_xform_free(h);
    }
};

// The map exactly as its public fields hold it (hand-built maps included).
void explicit_map(const CountSketchMap& map, Xform& xf) {
    if (static_cast<index_t>(map.hash.size()) != map.input_dim ||
        static_cast<index_t>(map.sign.size()) != map.input_dim)
        throw std::invalid_argument("countsketch_apply: map hash/sign length differs from input_dim");
    check(cgx_countsketch_explicit(context(), map.buckets, map.input_dim, map.hash.data(), map.sign.data(),
                                   CGX_MEM_HOST, &xf.h));
}

} // namespace

CountSketchMap countsketch_new(index_t buckets, index_t input_dim, SeededRng& rng) {
    if (buckets < 1 || input_dim < 1)
        throw std::invalid_argument("countsketch_new: buckets and input_dim must be >= 1");
    CountSketchMap map;
    map.buckets = buckets;
    map.input_dim = input_dim;
    map.seed = rng.next_u64();
    Xform xf;
    check(cgx_countsketch_new(context(), map.seed, buckets, input_dim, &xf.h));
    map.hash.resize(static_cast<std::size_t>(input_dim));
    map.sign.resize(static_cast<std::size_t>(input_dim));
    check(cgx_fill_hash_sign(context(), xf.h, map.hash.data(), map.sign.data(), CGX_MEM_HOST, nullptr));
    return map;
}

CountSketchMap countsketch_injective(index_t buckets, index_t input_dim, SeededRng& rng) {
    if (buckets < input_dim)
        throw std::invalid_argument("countsketch_injective: needs buckets >= input_dim");
    CountSketchMap map;
    map.buckets = buckets;
    map.input_dim = input_dim;
    map.seed = rng.next_u64();
    if (input_dim == 0) return map;
    Xform xf;
    check(cgx_countsketch_injective(context(), map.seed, buckets, input_dim, &xf.h));
    map.hash.resize(static_cast<std::size_t>(input_dim));
    map.sign.resize(static_cast<std::size_t>(input_dim));
    check(cgx_fill_hash_sign(context(), xf.h, map.hash.data(), map.sign.data(), CGX_MEM_HOST, nullptr));
    return map;
}

DenseMatrix countsketch_apply(const CountSketchMap& map, const DenseMatrix& x) {
    if (x.rows() != map.input_dim)
        throw std::invalid_argument("countsketch_apply: X has " + std::to_string(x.rows()) +
                                    " rows, sketch expects " + std::to_string(map.input_dim));
    DenseMatrix out(map.buckets, x.cols());
    if (x.cols() == 0 || x.rows() == 0) return out;
    Xform xf;
    explicit_map(map, xf);
    check(cgx_countsketch_apply_dense(context(), xf.h, x.data(), CGX_F64, CGX_COL_MAJOR, std::max<index_t>(x.rows(), 1),
                                      x.rows(), x.cols(), CGX_MEM_HOST, out.data(), CGX_COL_MAJOR, CGX_MEM_HOST,
                                      nullptr));
    return out;
}

DenseMatrix countsketch_apply(const CountSketchMap& map, const SparseMatrix& x) {
    if (x.rows != map.input_dim)
        throw std::invalid_argument("countsketch_apply: X has " + std::to_string(x.rows) +
                                    " rows, sketch expects " + std::to_string(map.input_dim));
    DenseMatrix out(map.buckets, x.cols);
    if (x.cols == 0 || x.rows == 0) return out;
    Xform xf;
    explicit_map(map, xf);
    check(cgx_countsketch_apply_csr(context(), xf.h, x.row_offsets.data(), x.col_indices.data(), CGX_I64,
                                    x.values.data(), CGX_F64, x.rows, x.cols, x.nnz(), CGX_MEM_HOST, out.data(),
                                    CGX_COL_MAJOR, CGX_MEM_HOST, nullptr));
    return out;
}

CountGaussTransform countgauss_new(index_t m, index_t buckets, index_t input_dim, SeededRng& rng) {
    if (m < 1 || buckets < 1 || input_dim < 1)
        throw std::invalid_argument("countgauss_new: m, buckets and input_dim must be >= 1");
    CountGaussTransform t;
    t.m = m;
    t.seed = rng.next_u64();
    Xform xf;
    check(cgx_countgauss_new(context(), t.seed, m, buckets, input_dim, &xf.h));
    uint64_t map_seed = 0;
    check(cgx_xform_info(xf.h, nullptr, &map_seed, nullptr, nullptr, nullptr, nullptr));
    t.cs.buckets = buckets;
    t.cs.input_dim = input_dim;
    t.cs.seed = map_seed;
    t.cs.hash.resize(static_cast<std::size_t>(input_dim));
    t.cs.sign.resize(static_cast<std::size_t>(input_dim));
    check(cgx_fill_hash_sign(context(), xf.h, t.cs.hash.data(), t.cs.sign.data(), CGX_MEM_HOST, nullptr));
    t.g = DenseMatrix(m, buckets);
    check(cgx_fill_gaussian(context(), xf.h, t.g.data(), CGX_MEM_HOST, nullptr));
    return t;
}

CountGaussTransform countgauss_new(index_t m, index_t input_dim, SeededRng& rng) {
    return countgauss_new(m, 5 * m, input_dim, rng);
}

namespace {
template <class Apply>
DenseMatrix countgauss_apply_impl(const CountGaussTransform& t, index_t rows, index_t cols, Apply&& apply) {
    if (rows != t.cs.input_dim)
        throw std::invalid_argument("countsketch_apply: X has " + std::to_string(rows) + " rows, sketch expects " +
                                    std::to_string(t.cs.input_dim));
    if (t.g.cols() != t.cs.buckets)
        throw std::invalid_argument("gemm: inner dimensions mismatch (" + std::to_string(t.g.cols()) + " vs " +
                                    std::to_string(t.cs.buckets) + ")");
    DenseMatrix z(t.g.rows(), cols);
    if (cols == 0 || t.g.rows() == 0) return z;
    Xform xf;
    explicit_map(t.cs, xf);
    check(cgx_xform_set_gaussian_explicit(context(), xf.h, t.g.rows(), t.g.data(), CGX_MEM_HOST));
    apply(xf.h, z.data());
    return z;
}
} // namespace

DenseMatrix countgauss_apply(const CountGaussTransform& t, const DenseMatrix& x) {
    return countgauss_apply_impl(t, x.rows(), x.cols(), [&](cgx_xform* h, double* z) {
        check(cgx_countgauss_apply_dense(context(), h, x.data(), CGX_F64, CGX_COL_MAJOR, std::max<index_t>(x.rows(), 1),
                                         x.rows(), x.cols(), CGX_MEM_HOST, z, CGX_MEM_HOST, nullptr));
    });
}

DenseMatrix countgauss_apply(const CountGaussTransform& t, const SparseMatrix& x) {
    return countgauss_apply_impl(t, x.rows, x.cols, [&](cgx_xform* h, double* z) {
        check(cgx_countgauss_apply_csr(context(), h, x.row_offsets.data(), x.col_indices.data(), CGX_I64,
                                       x.values.data(), CGX_F64, x.rows, x.cols, x.nnz(), CGX_MEM_HOST, z,
                                       CGX_MEM_HOST, nullptr));
    });
}

} // namespace cg
