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
//    or hand-edits them keeps working, and apply uses whatever the fields hold;
//  * seeded fast path (SURVEY 8b dispatch rule): the device transform a constructor built
//    stays cached, keyed by its seeds and sizes, together with 64-bit checksums of the
//    fields it wrote.  An apply whose argument matches a cached key AND whose fields still
//    have those checksums (recomputed over the whole arrays on every call, with the
//    library's host threads) runs on the cached transform -- no re-validation, re-sort or
//    re-upload of the map and G.  Anything else (hand-built or edited maps) takes the
//    explicit path, which ships the fields as they are.  Cached device memory is capped
//    (CGX_SHIM_CACHE_MB, default 8192) and evicted least-recently-used;
//  * std::invalid_argument with the reference's messages; CGX_ERANGE -> length_error;
//  * thread safety: one process-wide context, calls serialized inside libcgx (the
//    reference calls these from OpenMP regions, distcheck.cpp:107-111).
// Beyond the reference: CGX_DEVICES="0,1,2,3" makes countgauss_apply on a constructor-built
// (seeded) transform span those GPUs -- rows of X split across them, each GPU staging its own
// row block over its own PCIe link, the partial sketches combined over NVLink (cgx_group_*,
// INTEGRATION.md).  CGX_COMBINE = p2p | g | sx | z picks the combine (default: the sketch
// kernels' peer-memory stores when the devices can map each other, else NCCL).
#include "countgauss/sketch.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

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

// ---- CGX_DEVICES: the device group and its row-sharded transforms --------------------
cgx_group* group() {
    static std::once_flag once;
    static cgx_group* g = nullptr;
    std::call_once(once, [] {
        const char* list = std::getenv("CGX_DEVICES");
        if (!list) return;
        std::vector<int> devs;
        for (const char* p = list; *p;) {
            char* end = nullptr;
            const long v = std::strtol(p, &end, 10);
            if (end == p) break;
            devs.push_back((int)v);
            p = *end == ',' ? end + 1 : end;
        }
        if (devs.size() < 2) return;  // one device: the single-context path (CGX_DEVICE)
        check(cgx_group_init((int)devs.size(), devs.data(), &g));
    });
    return g;
}

int group_combine(cgx_group* g, bool dense) {
    const char* c = std::getenv("CGX_COMBINE");
    const std::string want = c ? c : "";
    if (want == "z") return CGX_COMBINE_Z;
    if (want == "g") return CGX_COMBINE_G;
    if (want == "sx") return CGX_COMBINE_SX;
    if (want == "p2p" || cgx_group_supports(g, CGX_COMBINE_P2P)) return CGX_COMBINE_P2P;
    return dense ? CGX_COMBINE_G : CGX_COMBINE_SX;  // the north star's NCCL schemes
}

// Group transforms are pure functions of (seed, m, B, n): built on first use, a few kept.
std::shared_ptr<cgx_gxform> group_xform(cgx_group* g, uint64_t t_seed, index_t m, index_t B, index_t n) {
    using Key = std::tuple<uint64_t, index_t, index_t, index_t>;
    static std::mutex mu;
    static std::list<std::pair<Key, std::shared_ptr<cgx_gxform>>> lru;
    std::lock_guard<std::mutex> lk(mu);
    const Key k{t_seed, m, B, n};
    for (auto it = lru.begin(); it != lru.end(); ++it)
        if (it->first == k) {
            lru.splice(lru.begin(), lru, it);
            return lru.front().second;
        }
    cgx_gxform* t = nullptr;
    check(cgx_group_countgauss_new(g, t_seed, m, B, n, &t));
    lru.emplace_front(k, std::shared_ptr<cgx_gxform>(t, cgx_gxform_free));
    while (lru.size() > 4) lru.pop_back();
    return lru.front().second;
}

struct Xform {
    cgx_xform* h = nullptr;
    ~Xform() {
        if (h) cgx_xform_free(h);
    }
};

uint64_t checksum(const void* p, std::size_t bytes) {
    uint64_t h = 0;
    check(cgx_host_checksum(context(), p, bytes, &h));
    return h;
}

// ---- seeded fast path: constructor-built device transforms, keyed and checksummed ----
struct Entry {
    bool gauss = false;                  // has G (countgauss_new) or map only
    uint64_t t_seed = 0, cs_seed = 0;
    index_t m = 0, B = 0, n = 0;
    uint64_t sum_hash = 0, sum_sign = 0, sum_g = 0;
    std::shared_ptr<cgx_xform> h;  // freed when the last user (entry or running apply) drops it
    std::size_t bytes = 0;
};

class Cache {
    std::mutex mu_;
    std::list<Entry> lru_;  // front = most recent
    std::size_t bytes_ = 0, cap_;

  public:
    Cache() {
        const char* mb = std::getenv("CGX_SHIM_CACHE_MB");
        cap_ = (std::size_t)(mb ? std::atoll(mb) : 8192) << 20;
    }
    void insert(Entry e) {
        std::lock_guard<std::mutex> lk(mu_);
        if (e.bytes > cap_) return;
        bytes_ += e.bytes;
        lru_.push_front(std::move(e));
        while (bytes_ > cap_ || lru_.size() > 256) {
            bytes_ -= lru_.back().bytes;
            lru_.pop_back();
        }
    }
    // The cached transform for a map (any entry holding it) or a CountGauss transform
    // (gauss entries only), verified against the fields' checksums; null if none.
    std::shared_ptr<cgx_xform> find(const CountSketchMap& cs, const CountGaussTransform* t) {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = lru_.begin(); it != lru_.end(); ++it) {
            const Entry& e = *it;
            if (e.cs_seed != cs.seed || e.B != cs.buckets || e.n != cs.input_dim) continue;
            if (t && (!e.gauss || e.t_seed != t->seed || e.m != t->g.rows() || t->g.cols() != e.B)) continue;
            if (static_cast<index_t>(cs.hash.size()) != e.n || static_cast<index_t>(cs.sign.size()) != e.n) continue;
            if (checksum(cs.hash.data(), cs.hash.size() * sizeof(index_t)) != e.sum_hash ||
                checksum(cs.sign.data(), cs.sign.size() * sizeof(double)) != e.sum_sign)
                continue;
            if (t && checksum(t->g.data(), (std::size_t)t->g.size() * sizeof(double)) != e.sum_g) continue;
            lru_.splice(lru_.begin(), lru_, it);
            return lru_.front().h;
        }
        return {};
    }
};

// Never destroyed: freeing device transforms from a static destructor would run after the
// CUDA runtime's own teardown at process exit.
Cache& cache() {
    static Cache* c = new Cache;
    return *c;
}

void remember_map(const CountSketchMap& map, cgx_xform*& h) {
    Entry e;
    e.cs_seed = map.seed;
    e.B = map.buckets;
    e.n = map.input_dim;
    e.sum_hash = checksum(map.hash.data(), map.hash.size() * sizeof(index_t));
    e.sum_sign = checksum(map.sign.data(), map.sign.size() * sizeof(double));
    e.h = std::shared_ptr<cgx_xform>(h, cgx_xform_free);
    e.bytes = (std::size_t)(4 * (e.n + e.B + 1));
    h = nullptr;  // the cache owns it now
    cache().insert(std::move(e));
}

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
    remember_map(map, xf.h);
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
    remember_map(map, xf.h);
    return map;
}

DenseMatrix countsketch_apply(const CountSketchMap& map, const DenseMatrix& x) {
    if (x.rows() != map.input_dim)
        throw std::invalid_argument("countsketch_apply: X has " + std::to_string(x.rows()) +
                                    " rows, sketch expects " + std::to_string(map.input_dim));
    DenseMatrix out(map.buckets, x.cols());
    if (x.cols() == 0 || x.rows() == 0) return out;
    Xform xf;
    std::shared_ptr<cgx_xform> hit = cache().find(map, nullptr);
    cgx_xform* h = hit.get();
    if (!h) {
        explicit_map(map, xf);
        h = xf.h;
    }
    check(cgx_countsketch_apply_dense(context(), h, x.data(), CGX_F64, CGX_COL_MAJOR, std::max<index_t>(x.rows(), 1),
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
    std::shared_ptr<cgx_xform> hit = cache().find(map, nullptr);
    cgx_xform* h = hit.get();
    if (!h) {
        explicit_map(map, xf);
        h = xf.h;
    }
    check(cgx_countsketch_apply_csr(context(), h, x.row_offsets.data(), x.col_indices.data(), CGX_I64,
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
    Entry e;
    e.gauss = true;
    e.t_seed = t.seed;
    e.cs_seed = map_seed;
    e.m = m;
    e.B = buckets;
    e.n = input_dim;
    e.sum_hash = checksum(t.cs.hash.data(), t.cs.hash.size() * sizeof(index_t));
    e.sum_sign = checksum(t.cs.sign.data(), t.cs.sign.size() * sizeof(double));
    e.sum_g = checksum(t.g.data(), (std::size_t)t.g.size() * sizeof(double));
    e.h = std::shared_ptr<cgx_xform>(xf.h, cgx_xform_free);
    e.bytes = (std::size_t)(4 * (input_dim + buckets + 1) + 8 * m * buckets);
    xf.h = nullptr;
    cache().insert(std::move(e));
    return t;
}

CountGaussTransform countgauss_new(index_t m, index_t input_dim, SeededRng& rng) {
    return countgauss_new(m, 5 * m, input_dim, rng);
}

namespace {
template <class Apply, class GroupApply>
DenseMatrix countgauss_apply_impl(const CountGaussTransform& t, index_t rows, index_t cols, Apply&& apply,
                                  GroupApply&& group_apply) {
    if (rows != t.cs.input_dim)
        throw std::invalid_argument("countsketch_apply: X has " + std::to_string(rows) + " rows, sketch expects " +
                                    std::to_string(t.cs.input_dim));
    if (t.g.cols() != t.cs.buckets)
        throw std::invalid_argument("gemm: inner dimensions mismatch (" + std::to_string(t.g.cols()) + " vs " +
                                    std::to_string(t.cs.buckets) + ")");
    DenseMatrix z(t.g.rows(), cols);
    if (cols == 0 || t.g.rows() == 0) return z;
    if (std::shared_ptr<cgx_xform> hit = cache().find(t.cs, &t)) {  // seeded fast path
        cgx_group* g = group();  // CGX_DEVICES: the same transform, row-sharded over the group
        // (small inputs stay on one GPU: the shards' fixed costs would exceed the work)
        if (g && rows >= (index_t)4096 * cgx_group_size(g)) {
            std::shared_ptr<cgx_gxform> gt = group_xform(g, t.seed, t.g.rows(), t.cs.buckets, t.cs.input_dim);
            group_apply(g, gt.get(), z.data());
            if (std::getenv("CGX_SHIM_TRACE"))
                std::fprintf(stderr, "cgx shim: countgauss_apply over %d ranks (CGX_DEVICES)\n", cgx_group_size(g));
            return z;
        }
        apply(hit.get(), z.data());
        return z;
    }
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
    }, [&](cgx_group* g, cgx_gxform* gt, double* z) {
        check(cgx_group_countgauss_apply_dense(g, gt, x.data(), CGX_F64, CGX_COL_MAJOR, std::max<index_t>(x.rows(), 1),
                                               x.rows(), x.cols(), CGX_MEM_HOST, z, CGX_MEM_HOST,
                                               group_combine(g, true)));
    });
}

DenseMatrix countgauss_apply(const CountGaussTransform& t, const SparseMatrix& x) {
    return countgauss_apply_impl(t, x.rows, x.cols, [&](cgx_xform* h, double* z) {
        check(cgx_countgauss_apply_csr(context(), h, x.row_offsets.data(), x.col_indices.data(), CGX_I64,
                                       x.values.data(), CGX_F64, x.rows, x.cols, x.nnz(), CGX_MEM_HOST, z,
                                       CGX_MEM_HOST, nullptr));
    }, [&](cgx_group* g, cgx_gxform* gt, double* z) {
        check(cgx_group_countgauss_apply_csr(g, gt, x.row_offsets.data(), x.col_indices.data(), CGX_I64,
                                             x.values.data(), CGX_F64, x.rows, x.cols, x.nnz(), z, CGX_MEM_HOST,
                                             group_combine(g, false)));
    });
}

} // namespace cg
