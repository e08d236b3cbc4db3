// capi.cu -- the cgx C-ABI (include/cgx.h): contexts, transforms, argument checking that
// mirrors the reference's std::invalid_argument cases, host<->device staging, and the
// stage-1 / stage-2 dispatch.  No exception crosses the extern "C" boundary.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <initializer_list>
#include <new>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

namespace cgx {

namespace {
thread_local std::string g_err;
}

void fail(int code, const std::string& msg) { throw Error{code, msg}; }
void set_last_error(const std::string& msg) { g_err = msg; }

void check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        fail(CGX_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
    }
    fail(CGX_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void check_launch(const char* what) { check_cuda(cudaGetLastError(), what); }

void* DevBuf::get(size_t need) {
    if (need == 0) need = 1;
    if (need <= bytes) return p;
    if (p) CGX_CUDA(cudaFree(p));  // synchronizes: no in-flight user of the old buffer
    p = nullptr;
    bytes = 0;
    const size_t want = need + need / 8;
    CGX_CUDA(cudaMalloc(&p, want));
    bytes = want;
    return p;
}

// Size classes: powers of two up to 1 MiB, then eighths of the enclosing power of two
// (at most 12.5% over the request: a 2.15 GB G or a 268 MB perm no longer rounds up to 4 GB
// or 512 MB).
size_t pool_class_of(size_t bytes) {
    size_t cls = 256;
    while (cls < bytes) cls <<= 1;
    if (cls <= ((size_t)1 << 20)) return cls;
    const size_t q = cls >> 3;
    return (bytes + q - 1) / q * q;
}

void* pool_alloc(cgx_ctx* ctx, size_t bytes) {
    const size_t cls = pool_class_of(bytes);
    auto& fl = ctx->pool_free[cls];
    if (!fl.empty()) {
        void* p = fl.back();
        fl.pop_back();
        return p;
    }
    void* p = nullptr;
    CGX_CUDA(cudaMalloc(&p, cls));
    ctx->pool_class[p] = cls;
    return p;
}

void pool_free(cgx_ctx* ctx, void* p) {
    if (!p) return;
    auto it = ctx->pool_class.find(p);
    if (it == ctx->pool_class.end()) {
        cudaFree(p);
        return;
    }
    ctx->pool_free[it->second].push_back(p);
}

void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

void Profile::begin(int stage, cudaStream_t s) {
    if (!on) return;
    auto& v = ev[stage];
    if (used[stage] == v.size()) {
        cudaEvent_t a, b;
        CGX_CUDA(cudaEventCreate(&a));
        CGX_CUDA(cudaEventCreate(&b));
        v.push_back({a, b});
    }
    CGX_CUDA(cudaEventRecord(v[used[stage]].first, s));
}

void Profile::end(int stage, cudaStream_t s) {
    if (!on) return;
    CGX_CUDA(cudaEventRecord(ev[stage][used[stage]].second, s));
    ++used[stage];
}

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return CGX_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return CGX_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return CGX_ECUDA;
    }
}

// Serializes a call on its context, binds the device and orders the call's stream after
// the previous call (which may have used the same scratch on another stream).
struct CallScope {
    cgx_ctx* ctx;
    cudaStream_t st;
    std::lock_guard<std::recursive_mutex> lock;
    CallScope(cgx_ctx* c, void* stream) : ctx(c), st(stream ? (cudaStream_t)stream : c->stream), lock(c->mu) {
        ctx->oz_colmax_for = nullptr;  // column maxima left by a sketch are valid within one call only
        CGX_CUDA(cudaSetDevice(ctx->device));
        CGX_CUDA(cudaStreamWaitEvent(st, ctx->done, 0));
    }
    ~CallScope() { cudaEventRecord(ctx->done, st); }
    void sync() { CGX_CUDA(cudaStreamSynchronize(st)); }
};

// Small results the host reads back (Z, a small S.X, the hash/sign fields of a small map): a
// cudaMemcpyAsync into pageable memory goes through the driver's own staging and costs ~12 us
// a call -- a third of a tiny apply -- so up to kSmallPin bytes come back through a pinned
// bounce buffer instead: one async copy, the stream sync the call needs anyway, a memcpy.
// `pieces`: consecutive device ranges -> their host destinations.
constexpr size_t kSmallPin = (size_t)256 << 10;
struct HostPiece {
    void* dst;
    size_t bytes;
};
void d2h_sync(cgx_ctx* ctx, const void* src_dev, std::initializer_list<HostPiece> pieces, CallScope& sc) {
    size_t total = 0;
    for (const HostPiece& p : pieces) total += p.bytes;
    if (total <= kSmallPin && !ctx->small_pin) {
        if (cudaMallocHost((void**)&ctx->small_pin, kSmallPin) != cudaSuccess) {
            cudaGetLastError();
            ctx->small_pin = nullptr;
        }
    }
    if (total <= kSmallPin && ctx->small_pin) {
        CGX_CUDA(cudaMemcpyAsync(ctx->small_pin, src_dev, total, cudaMemcpyDeviceToHost, sc.st));
        sc.sync();
        size_t off = 0;
        for (const HostPiece& p : pieces) {
            if (p.dst) std::memcpy(p.dst, ctx->small_pin + off, p.bytes);
            off += p.bytes;
        }
        return;
    }
    size_t off = 0;
    for (const HostPiece& p : pieces) {
        if (p.dst) CGX_CUDA(cudaMemcpyAsync(p.dst, (const char*)src_dev + off, p.bytes, cudaMemcpyDeviceToHost, sc.st));
        off += p.bytes;
    }
    sc.sync();
}

void need_ctx(cgx_ctx* ctx) {
    if (!ctx) fail(CGX_EINVAL, "cgx: null context");
}
void need_xf(const cgx_xform* xf) {
    if (!xf) fail(CGX_EINVAL, "cgx: null transform");
}
void need_mem(int mem) {
    if (mem != CGX_MEM_HOST && mem != CGX_MEM_DEVICE) fail(CGX_EINVAL, "cgx: mem must be CGX_MEM_HOST or CGX_MEM_DEVICE");
}
size_t dsize(int dtype) {
    if (dtype == CGX_F32) return 4;
    if (dtype == CGX_F64) return 8;
    fail(CGX_EINVAL, "cgx: dtype must be CGX_F32 or CGX_F64");
}

// A device view of a (possibly host) input array; host arrays land in `buf`.
const void* to_device(cgx_ctx* ctx, DevBuf& buf, const void* p, size_t bytes, int mem, cudaStream_t s) {
    if (mem == CGX_MEM_DEVICE || bytes == 0) return p;
    void* d = buf.get(bytes);
    CGX_CUDA(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, s));
    return d;
}

cgx_xform* new_xform(cgx_ctx* ctx, int64_t B, int64_t n) {
    if (n >= ((int64_t)1 << 31))
        fail(CGX_EINVAL, "cgx: input_dim must be < 2^31 on the GPU path (perm entries are 31-bit row indices)");
    if (B >= ((int64_t)1 << 31)) fail(CGX_EINVAL, "cgx: buckets must be < 2^31 on the GPU path");
    auto* xf = new cgx_xform;
    xf->ctx = ctx;
    xf->B = B;
    xf->n = n;
    try {
        xf->perm = (uint32_t*)pool_alloc(ctx, sizeof(uint32_t) * (size_t)n);
        xf->offsets = (uint32_t*)pool_alloc(ctx, sizeof(uint32_t) * (size_t)(B + 1));
    } catch (...) {
        pool_free(ctx, xf->perm);
        delete xf;
        throw;
    }
    return xf;
}

void drop_g(cgx_xform* xf) {
    oz_drop_image(xf);
    if (!xf->g_dev) return;
    if (xf->g_pool)
        pool_free(xf->ctx, xf->g_dev);
    else
        cudaFree(xf->g_dev);
    xf->g_dev = nullptr;
    xf->g_pool = false;
}

// Seeded G, materialized once per transform the way the reference's countgauss_new fills
// CountGaussTransform::g (sketch.cpp:115-130): every apply then reads G (m*B*8 bytes)
// instead of regenerating ~170 FP64 instructions per entry.  Skipped above 4 GiB or
// when option g_resident = 0 (the apply kernels then generate G where they use it).
void make_g_resident(cgx_ctx* ctx, cgx_xform* xf, cudaStream_t s) {
    const int64_t bytes = (int64_t)sizeof(double) * xf->m * xf->B;
    if (!ctx->opt_g_resident || xf->g_explicit || bytes > ((int64_t)4 << 30)) return;
    xf->g_dev = (double*)pool_alloc(ctx, (size_t)bytes);
    xf->g_pool = true;
    launch_gen_gauss(ctx, xf, 0, xf->B, xf->g_dev, s);
}

// Caller holds ctx->mu.  The device is drained first: kernels of this (or a failed)
// call may still read xf's arrays, and pooled blocks are reused immediately.
void free_xform(cgx_xform* xf) {
    if (!xf) return;
    cudaSetDevice(xf->ctx->device);
    cudaDeviceSynchronize();
    pool_free(xf->ctx, xf->perm);
    pool_free(xf->ctx, xf->offsets);
    pool_free(xf->ctx, xf->grows);
    drop_g(xf);
    delete xf;
}

// The reference's chunked-CSR branch condition (sketch.cpp:74-82).
int64_t csr_chunk_rows(int64_t n, int64_t B, int64_t d) {
    const int64_t chunk_rows = 8192;
    const int64_t n_chunks = (n + chunk_rows - 1) / chunk_rows;
    const int64_t out_size = B * d;
    const bool chunked = n_chunks > 1 && out_size <= ((int64_t)1 << 16) && n_chunks * out_size <= ((int64_t)1 << 25);
    return chunked ? chunk_rows : 0;
}

// Host dense X -> device (hoststage.cu): fp64 values that all round-trip through fp32
// arrive as fp32 and *dtype switches to CGX_F32.  A padded layout (ld beyond the rows of a
// column-major X, or the columns of a row-major one -- e.g. a row block of a larger
// matrix) is staged as its segments only and lands dense: *ld becomes n or d.
const void* stage_dense(cgx_ctx* ctx, const void* x, int* dtype, int layout, int64_t* ld, int64_t n, int64_t d,
                        int x_mem, cudaStream_t s) {
    if (x_mem == CGX_MEM_DEVICE || n == 0 || d == 0) return x;
    const size_t es = dsize(*dtype);
    const int64_t seg = layout == CGX_COL_MAJOR ? n : d, nseg = layout == CGX_COL_MAJOR ? d : n;
    bool narrowed = false;
    const void* p = stage_in(ctx, ctx->hin[0], ctx->hin[1], x, (size_t)(seg * nseg), es, *dtype == CGX_F64 ? 1 : 0,
                             &narrowed, s, (size_t)seg, (size_t)*ld);
    *ld = seg;
    if (narrowed) *dtype = CGX_F32;
    return p;
}

// Dense input -> device-resident row-major view (stages host X, transposes column-major X).
const void* dense_rowmajor(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int* dtype_io, int layout, int64_t ld,
                           int64_t n, int64_t d, int x_mem, int64_t* rld_out, cudaStream_t s) {
    int& dtype = *dtype_io;
    size_t es = dsize(dtype);
    if (layout != CGX_COL_MAJOR && layout != CGX_ROW_MAJOR) fail(CGX_EINVAL, "cgx: bad layout");
    if (n != xf->n)
        fail(CGX_EINVAL, "countsketch_apply: X has " + std::to_string(n) + " rows, sketch expects " +
                             std::to_string(xf->n));
    if (d < 0) fail(CGX_EINVAL, "cgx: negative column count");
    const int64_t minld = layout == CGX_COL_MAJOR ? n : d;
    if (ld < std::max<int64_t>(minld, 1)) fail(CGX_EINVAL, "cgx: leading dimension too small");
    if (d == 0) return x;
    const void* xd = stage_dense(ctx, x, &dtype, layout, &ld, n, d, x_mem, s);
    es = dsize(dtype);
    *rld_out = ld;
    if (layout == CGX_COL_MAJOR) {
        void* rm = ctx->xstage.get(es * (size_t)(n * d));
        launch_transpose_x(ctx, xd, dtype, ld, n, d, rm, s);
        xd = rm;
        *rld_out = d;
    }
    return xd;
}

// A stage-1 call of a device group in CGX_COMBINE_P2P mode (ctx->out_segs set): when the
// sketch kernel that will run cannot store into the peers' landing slots itself, it writes a
// local S.X (ctx->seg_local) and the bucket ranges are copied out afterwards.
struct SegsFallback {
    cgx_ctx* ctx;
    const cgx_xform* xf;
    int64_t d;
    const OutSegs* held = nullptr;
    double* local = nullptr;
    SegsFallback(cgx_ctx* c, const cgx_xform* x, int64_t dd, bool fused, double** sx) : ctx(c), xf(x), d(dd) {
        if (!ctx->out_segs) return;
        ++(fused ? ctx->seg_fused : ctx->seg_copied);
        if (fused) return;
        held = ctx->out_segs;
        ctx->out_segs = nullptr;
        local = (double*)ctx->seg_local.get(sizeof(double) * (size_t)(xf->B * d));
        *sx = local;
    }
    void finish(cudaStream_t s) {
        if (!held) return;
        ctx->out_segs = held;
        push_segs(ctx, local, xf->B, d, *held, s);
        held = nullptr;
    }
    ~SegsFallback() {
        if (held) ctx->out_segs = held;
    }
};

// Stage 1 (dense): SX row-major (B x d) into `sx_dev`.
void sketch_dense_dev(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int layout, int64_t ld,
                      int64_t n, int64_t d, int x_mem, double* sx_dev, cudaStream_t s) {
    size_t es = dsize(dtype);
    if (layout != CGX_COL_MAJOR && layout != CGX_ROW_MAJOR) fail(CGX_EINVAL, "cgx: bad layout");
    if (n != xf->n)
        fail(CGX_EINVAL, "countsketch_apply: X has " + std::to_string(n) + " rows, sketch expects " +
                             std::to_string(xf->n));
    if (d < 0) fail(CGX_EINVAL, "cgx: negative column count");
    const int64_t minld = layout == CGX_COL_MAJOR ? n : d;
    if (ld < std::max<int64_t>(minld, 1)) fail(CGX_EINVAL, "cgx: leading dimension too small");
    const void* xd = stage_dense(ctx, x, &dtype, layout, &ld, n, d, x_mem, s);
    es = dsize(dtype);
    int64_t rld = ld;
    if (layout == CGX_COL_MAJOR && d > 0) {
        void* rm = ctx->xstage.get(es * (size_t)(n * d));
        launch_transpose_x(ctx, xd, dtype, ld, n, d, rm, s);
        xd = rm;
        rld = d;
    }
    if (d == 0) return;
    ctx->prof.begin(0, s);
    SegsFallback fb(ctx, xf, d, sketch_dense_fuses_segs(ctx, xd, dtype, rld, d), &sx_dev);
    launch_sketch_dense(ctx, xf, xd, dtype, rld, n, d, sx_dev, s);
    fb.finish(s);
    ctx->prof.end(0, s);
}

// Host CSR inputs -> device (hoststage.cu; device inputs pass).  int64 column indices that
// all fit int32 arrive as int32 and fp64 values that all round-trip through fp32 arrive as
// fp32: *idx_type / *dtype switch accordingly (the kernels take both widths natively).
void stage_csr(cgx_ctx* ctx, const void** rp, const void** cp, int* idx_type, const void** vp, int* dtype, int64_t n,
               int64_t nnz, int x_mem, cudaStream_t s) {
    if (x_mem != CGX_MEM_HOST) return;
    bool nr = false;
    *rp = stage_in(ctx, ctx->hin[0], ctx->hin[1], *rp, (size_t)(n + 1), sizeof(int64_t), 0, &nr, s);
    if (nnz == 0) return;
    *cp = stage_in(ctx, ctx->hin[2], ctx->hin[3], *cp, (size_t)nnz, *idx_type == CGX_I32 ? 4 : 8,
                   *idx_type == CGX_I64 ? 2 : 0, &nr, s);
    if (nr) *idx_type = CGX_I32;
    *vp = stage_in(ctx, ctx->hin[4], ctx->hin[5], *vp, (size_t)nnz, dsize(*dtype), *dtype == CGX_F64 ? 1 : 0, &nr, s);
    if (nr) *dtype = CGX_F32;
}

void sketch_csr_dev(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols, int idx_type,
                    const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz, int x_mem, double* sx_dev,
                    cudaStream_t s) {
    const size_t es = dsize(dtype);
    if (idx_type != CGX_I32 && idx_type != CGX_I64) fail(CGX_EINVAL, "cgx: idx_type must be CGX_I32 or CGX_I64");
    if (n != xf->n)
        fail(CGX_EINVAL, "countsketch_apply: X has " + std::to_string(n) + " rows, sketch expects " +
                             std::to_string(xf->n));
    if (d < 0 || nnz < 0) fail(CGX_EINVAL, "cgx: negative size");
    if (d >= ((int64_t)1 << 26)) fail(CGX_EINVAL, "cgx: CSR column count must be < 2^26 on the GPU path");
    if (d == 0) return;
    const void* rp = rowptr;
    const void* cp = cols;
    const void* vp = vals;
    (void)es;
    stage_csr(ctx, &rp, &cp, &idx_type, &vp, &dtype, n, nnz, x_mem, s);
    if (ctx->csr_base) {  // offsets count from the caller's element 0: rebase the array pointers instead
        cp = (const char*)cp - (idx_type == CGX_I32 ? 4 : 8) * ctx->csr_base;
        vp = (const char*)vp - (int64_t)dsize(dtype) * ctx->csr_base;
    }
    ctx->prof.begin(0, s);
    const int64_t chunk_rows = csr_chunk_rows(n, xf->B, d);
    const bool records = chunk_rows == 0 && csr_atomic_applies(ctx, xf, n, d, nnz, dtype);
    SegsFallback fb(ctx, xf, d, !records && sketch_csr_fuses_segs(ctx, d, chunk_rows), &sx_dev);
    if (records)
        launch_sketch_csr_atomic(ctx, xf, (const int64_t*)rp, cp, idx_type, vp, n, d, nnz, sx_dev, s);
    else
        launch_sketch_csr(ctx, xf, (const int64_t*)rp, cp, idx_type, vp, dtype, n, d, sx_dev, chunk_rows, s);
    fb.finish(s);
    ctx->prof.end(0, s);
}

} // namespace
void push_segs(cgx_ctx* ctx, const double* sx, int64_t B, int64_t d, const OutSegs& segs, cudaStream_t s) {
    (void)ctx;
    for (int64_t q = 0, b0 = 0; b0 < B; ++q, b0 += segs.per) {
        const int64_t nb = std::min<int64_t>(segs.per, B - b0);
        CGX_CUDA(cudaMemcpyAsync(segs.base[q], sx + b0 * d, sizeof(double) * (size_t)(nb * d), cudaMemcpyDeviceToDevice, s));
    }
}
namespace {

void need_g(const cgx_xform* xf) {
    if (!xf->has_g) fail(CGX_EINVAL, "countgauss_apply: transform has no Gaussian factor (use countgauss_new)");
}

// Stage 2 + output placement.
void finish_gemm(cgx_ctx* ctx, const cgx_xform* xf, const double* sx_dev, int64_t d, double* z, int z_mem,
                 CallScope& sc, int64_t b0 = 0, int64_t b1 = -1) {
    const size_t zb = sizeof(double) * (size_t)(xf->m * d);
    if (d == 0) return;
    if (b1 < 0) b1 = xf->B;
    double* zd = z;
    if (z_mem == CGX_MEM_HOST) zd = (double*)ctx->tmp.get(zb);  // tmp is free again after the scans
    ctx->prof.begin(1, sc.st);
    launch_gauss_gemm(ctx, xf, sx_dev, b0, b1, d, zd, sc.st);
    ctx->prof.end(1, sc.st);
    if (z_mem == CGX_MEM_HOST) d2h_sync(ctx, zd, {{z, zb}}, sc);
}

void place_sx(cgx_ctx* ctx, const cgx_xform* xf, const double* sx_dev, int64_t d, double* sx, int sx_layout, int sx_mem,
              CallScope& sc) {
    const size_t bytes = sizeof(double) * (size_t)(xf->B * d);
    if (d == 0) return;
    const double* src = sx_dev;
    if (sx_layout == CGX_COL_MAJOR) {
        double* dst = sx_mem == CGX_MEM_DEVICE ? sx : (double*)ctx->zpart.get(bytes);
        launch_transpose_sx(ctx, sx_dev, xf->B, d, dst, sc.st);
        src = dst;
        if (sx_mem == CGX_MEM_DEVICE) return;
    } else if (sx_layout != CGX_ROW_MAJOR) {
        fail(CGX_EINVAL, "cgx: bad sx layout");
    } else if (sx_mem == CGX_MEM_DEVICE) {
        if (src != sx) CGX_CUDA(cudaMemcpyAsync(sx, src, bytes, cudaMemcpyDeviceToDevice, sc.st));
        return;
    }
    d2h_sync(ctx, src, {{sx, bytes}}, sc);
}

void build_explicit(cgx_ctx* ctx, cgx_xform* xf, const int64_t* hash, const double* sign, int mem, CallScope& sc) {
    const int64_t n = xf->n;
    uint32_t* keys = (uint32_t*)ctx->sx.get(sizeof(uint32_t) * (size_t)n * 2);
    uint32_t* vals = keys + n;
    if (mem == CGX_MEM_HOST) {
        // validate and pack on the host: 8 B/row cross the bus instead of 16, no device sync
        std::vector<uint32_t> hk((size_t)(2 * n));
        for (int64_t i = 0; i < n; ++i) {
            const int64_t h = hash[i];
            const double s = sign[i];
            if (h < 0 || h >= xf->B || !(s == 1.0 || s == -1.0))
                fail(CGX_EINVAL, "countsketch map: hash must lie in [0, buckets) and sign in {-1, +1}");
            hk[(size_t)i] = (uint32_t)h;
            hk[(size_t)(n + i)] = (uint32_t)i | (s < 0 ? kNegBit : 0u);
        }
        CGX_CUDA(cudaMemcpyAsync(keys, hk.data(), sizeof(uint32_t) * (size_t)(2 * n), cudaMemcpyHostToDevice, sc.st));
    } else if (!prep_explicit(ctx, hash, sign, n, xf->B, keys, vals, sc.st)) {
        fail(CGX_EINVAL, "countsketch map: hash must lie in [0, buckets) and sign in {-1, +1}");
    }
    xf->seeded_map = false;
    build_perm_explicit(ctx, xf, keys, vals, sc.st);
}

// Two-phase CSR generation: without cols/vals, row offsets + nnz; with them, the fill.
void gen_csr(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, const CsrGenSpec& spec, int64_t* rowptr_dev,
             int32_t* cols_dev, float* vals_dev, int64_t* nnz_out, void* stream) {
    CallScope sc(ctx, stream);
    if (!cols_dev || !vals_dev) {
        launch_gen_csr_counts(ctx, seed, n, d, spec, rowptr_dev, sc.st);
        int64_t nnz = 0;
        CGX_CUDA(cudaMemcpyAsync(&nnz, rowptr_dev + n, sizeof(int64_t), cudaMemcpyDeviceToHost, sc.st));
        sc.sync();
        if (nnz_out) *nnz_out = nnz;
        return;
    }
    launch_gen_csr_fill(ctx, seed, n, d, spec, rowptr_dev, cols_dev, vals_dev, sc.st);
}

} // namespace
} // namespace cgx

using namespace cgx;

extern "C" {

const char* cgx_last_error(void) { return g_err.c_str(); }
const char* cgx_version(void) { return "cgx 0.1 (sm_100a)"; }

int cgx_init(int device, cgx_ctx** out) {
    return guard([&] {
        if (!out) fail(CGX_EINVAL, "cgx_init: null out");
        int count = 0;
        CGX_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) fail(CGX_EINVAL, "cgx_init: no such device");
        CGX_CUDA(cudaSetDevice(device));
        auto* ctx = new cgx_ctx;
        ctx->device = device;
        CGX_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        CGX_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        CGX_CUDA(cudaEventCreateWithFlags(&ctx->done, cudaEventDisableTiming));
        CGX_CUDA(cudaMalloc((void**)&ctx->task_ctr, sizeof(unsigned long long)));
        CGX_CUDA(cudaMemsetAsync(ctx->task_ctr, 0, sizeof(unsigned long long), ctx->stream));
        CGX_CUDA(cudaEventRecord(ctx->done, ctx->stream));
        *out = ctx;
    });
}

int cgx_free(cgx_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        cudaSetDevice(ctx->device);
        cudaDeviceSynchronize();
        for (DevBuf* b : {&ctx->sx, &ctx->zpart, &ctx->xstage, &ctx->tmp, &ctx->sort_k[0], &ctx->sort_k[1],
                          &ctx->sort_v[0], &ctx->sort_v[1], &ctx->sort_hist, &ctx->counts, &ctx->hstage_dev,
                          &ctx->sched, &ctx->gen_tables})
            b->release();
        for (auto& kv : ctx->pool_class) cudaFree(kv.first);
        if (ctx->pinned) cudaFreeHost(ctx->pinned);
        if (ctx->small_pin) cudaFreeHost(ctx->small_pin);
        for (auto& b : ctx->hin) b.release();
        host_pool_free(ctx);
        for (int s = 0; s < 2; ++s)
            for (auto& e : ctx->prof.ev[s]) {
                cudaEventDestroy(e.first);
                cudaEventDestroy(e.second);
            }
        cudaEventDestroy(ctx->done);
        ctx->gfull.release();
        ctx->gchunk.release();
        for (DevBuf& b : ctx->part) b.release();
        for (DevBuf* b : {&ctx->oz_max, &ctx->oz_a, &ctx->oz_b, &ctx->seg_local}) b->release();
        cudaStreamDestroy(ctx->stream);
        cudaFree(ctx->task_ctr);
        delete ctx;
    });
}

int cgx_trim(cgx_ctx* ctx) {
    return guard([&] {
        need_ctx(ctx);
        std::lock_guard<std::recursive_mutex> lk(ctx->mu);
        CGX_CUDA(cudaSetDevice(ctx->device));
        CGX_CUDA(cudaDeviceSynchronize());
        for (DevBuf* b : {&ctx->sx, &ctx->zpart, &ctx->xstage, &ctx->tmp, &ctx->sort_k[0], &ctx->sort_k[1],
                          &ctx->sort_v[0], &ctx->sort_v[1], &ctx->sort_hist, &ctx->counts, &ctx->hstage_dev,
                          &ctx->gfull, &ctx->gchunk, &ctx->oz_max, &ctx->oz_a, &ctx->seg_local})
            b->release();
        for (DevBuf& b : ctx->hin) b.release();
        for (DevBuf& b : ctx->part) b.release();
        for (auto& kv : ctx->pool_free) {
            for (void* p : kv.second) {
                cudaFree(p);
                ctx->pool_class.erase(p);
            }
            kv.second.clear();
        }
        ctx->pool_free.clear();
        ctx->oz_colmax_for = nullptr;
    });
}

int cgx_synchronize(cgx_ctx* ctx, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        CGX_CUDA(cudaSetDevice(ctx->device));
        CGX_CUDA(cudaStreamSynchronize(stream ? (cudaStream_t)stream : ctx->stream));
    });
}

int cgx_device_alloc(cgx_ctx* ctx, size_t bytes, void** out) {
    return guard([&] {
        need_ctx(ctx);
        CGX_CUDA(cudaSetDevice(ctx->device));
        CGX_CUDA(cudaMalloc(out, bytes ? bytes : 1));
    });
}
int cgx_device_free(cgx_ctx* ctx, void* p) {
    return guard([&] {
        need_ctx(ctx);
        CGX_CUDA(cudaSetDevice(ctx->device));
        CGX_CUDA(cudaFree(p));
    });
}
// ---- peer memory across processes (one process per GPU): CUDA IPC ------------------------
int cgx_ipc_export(cgx_ctx* ctx, const void* p, unsigned char* handle) {
    return guard([&] {
        need_ctx(ctx);
        if (!p || !handle) fail(CGX_EINVAL, "cgx_ipc_export: null argument");
        static_assert(sizeof(cudaIpcMemHandle_t) == CGX_IPC_HANDLE_BYTES, "CUDA IPC handle size");
        CGX_CUDA(cudaSetDevice(ctx->device));
        cudaIpcMemHandle_t h;
        CGX_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(p)));
        std::memcpy(handle, &h, sizeof h);
    });
}
int cgx_ipc_open(cgx_ctx* ctx, const unsigned char* handle, void** out) {
    return guard([&] {
        need_ctx(ctx);
        if (!out || !handle) fail(CGX_EINVAL, "cgx_ipc_open: null argument");
        CGX_CUDA(cudaSetDevice(ctx->device));
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        CGX_CUDA(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
    });
}
int cgx_ipc_close(cgx_ctx* ctx, void* p) {
    return guard([&] {
        need_ctx(ctx);
        CGX_CUDA(cudaSetDevice(ctx->device));
        CGX_CUDA(cudaIpcCloseMemHandle(p));
    });
}

int cgx_host_alloc(cgx_ctx* ctx, size_t bytes, void** out) {
    return guard([&] {
        need_ctx(ctx);
        CGX_CUDA(cudaSetDevice(ctx->device));
        CGX_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
    });
}
int cgx_host_free(cgx_ctx* ctx, void* p) {
    return guard([&] {
        need_ctx(ctx);
        CGX_CUDA(cudaFreeHost(p));
    });
}
int cgx_memcpy(cgx_ctx* ctx, void* dst, const void* src, size_t bytes, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        CallScope sc(ctx, stream);
        CGX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, sc.st));
        sc.sync();
    });
}

uint64_t cgx_mix64(uint64_t a, uint64_t b) { return mix64(a, b); }
uint64_t cgx_rng_draw(uint64_t seed, uint64_t k) { return rng_draw(seed, k); }

int cgx_countsketch_new(cgx_ctx* ctx, uint64_t map_seed, int64_t buckets, int64_t input_dim, cgx_xform** out) {
    return guard([&] {
        need_ctx(ctx);
        if (buckets < 1 || input_dim < 1)
            fail(CGX_EINVAL, "countsketch_new: buckets and input_dim must be >= 1");
        CallScope sc(ctx, nullptr);
        cgx_xform* xf = new_xform(ctx, buckets, input_dim);
        try {
            xf->map_seed = map_seed;
            xf->seeded_map = true;
            build_perm_seeded(ctx, xf, sc.st);  // stream-ordered: no host wait
        } catch (...) {
            free_xform(xf);
            throw;
        }
        *out = xf;
    });
}


int cgx_countsketch_explicit(cgx_ctx* ctx, int64_t buckets, int64_t input_dim, const int64_t* hash, const double* sign,
                             int mem, cgx_xform** out) {
    return guard([&] {
        need_ctx(ctx);
        need_mem(mem);
        if (buckets < 1 || input_dim < 1) fail(CGX_EINVAL, "countsketch map: buckets and input_dim must be >= 1");
        if (!hash || !sign) fail(CGX_EINVAL, "countsketch map: null hash/sign");
        CallScope sc(ctx, nullptr);
        cgx_xform* xf = new_xform(ctx, buckets, input_dim);
        try {
            build_explicit(ctx, xf, hash, sign, mem, sc);
        } catch (...) {
            free_xform(xf);
            throw;
        }
        *out = xf;
    });
}

int cgx_countsketch_injective(cgx_ctx* ctx, uint64_t map_seed, int64_t buckets, int64_t input_dim, cgx_xform** out) {
    return guard([&] {
        need_ctx(ctx);
        if (buckets < input_dim) fail(CGX_EINVAL, "countsketch_injective: needs buckets >= input_dim");
        if (input_dim < 1) fail(CGX_EINVAL, "countsketch_injective: input_dim must be >= 1 on the GPU path");
        // Partial Fisher-Yates over [0, buckets) (sketch.cpp:38-48): inherently sequential.
        std::vector<int64_t> pool((size_t)buckets), hash((size_t)input_dim);
        std::vector<double> sign((size_t)input_dim);
        std::iota(pool.begin(), pool.end(), int64_t{0});
        uint64_t k = 0;
        for (int64_t i = 0; i < input_dim; ++i) {
            const int64_t j = i + (int64_t)(rng_draw(map_seed, k++) % (uint64_t)(buckets - i));
            std::swap(pool[(size_t)i], pool[(size_t)j]);
            hash[(size_t)i] = pool[(size_t)i];
            sign[(size_t)i] = (rng_draw(map_seed, k++) & 1ULL) ? 1.0 : -1.0;
        }
        CallScope sc(ctx, nullptr);
        cgx_xform* xf = new_xform(ctx, buckets, input_dim);
        try {
            xf->map_seed = map_seed;
            build_explicit(ctx, xf, hash.data(), sign.data(), CGX_MEM_HOST, sc);
        } catch (...) {
            free_xform(xf);
            throw;
        }
        *out = xf;
    });
}

int cgx_countgauss_new(cgx_ctx* ctx, uint64_t t_seed, int64_t m, int64_t buckets, int64_t input_dim, cgx_xform** out) {
    return cgx_countgauss_new_shard(ctx, t_seed, m, buckets, input_dim, 0, input_dim, out);
}

int cgx_countgauss_new_shard(cgx_ctx* ctx, uint64_t t_seed, int64_t m, int64_t buckets, int64_t input_dim,
                             int64_t row0, int64_t rows, cgx_xform** out) {
    return guard([&] {
        need_ctx(ctx);
        if (m < 1 || buckets < 1 || input_dim < 1)
            fail(CGX_EINVAL, "countgauss_new: m, buckets and input_dim must be >= 1");
        if (row0 < 0 || rows < 1 || row0 + rows > input_dim)
            fail(CGX_EINVAL, "countgauss_new_shard: need 0 <= row0 and 1 <= rows and row0 + rows <= input_dim");
        CallScope sc(ctx, nullptr);
        cgx_xform* xf = new_xform(ctx, buckets, rows);
        try {
            xf->row0 = row0;
            xf->t_seed = t_seed;
            xf->map_seed = rng_draw(mix64(t_seed, 1), 0);  // countsketch_new(..., cs_rng): map.seed
            xf->g_seed = mix64(t_seed, 2);                 // g_rng = SeededRng(mix64(t.seed, 2))
            xf->m = m;
            xf->has_g = true;
            build_perm_seeded(ctx, xf, sc.st);  // stream-ordered: no host wait
            make_g_resident(ctx, xf, sc.st);
        } catch (...) {
            free_xform(xf);
            throw;
        }
        *out = xf;
    });
}

int cgx_countgauss_bucket_shard(cgx_ctx* ctx, uint64_t t_seed, int64_t m, int64_t buckets, int64_t input_dim,
                                int64_t b0, int64_t b1, cgx_xform** out) {
    return guard([&] {
        need_ctx(ctx);
        if (m < 1 || buckets < 1 || input_dim < 1)
            fail(CGX_EINVAL, "countgauss_new: m, buckets and input_dim must be >= 1");
        if (b0 < 0 || b1 <= b0 || b1 > buckets)
            fail(CGX_EINVAL, "countgauss_bucket_shard: need 0 <= b0 < b1 <= buckets");
        CallScope sc(ctx, nullptr);
        // the full map (rows of every bucket, seeded), then its bucket range as a transform
        cgx_xform* full = new_xform(ctx, buckets, input_dim);
        cgx_xform* xf = nullptr;
        try {
            full->t_seed = t_seed;
            full->map_seed = rng_draw(mix64(t_seed, 1), 0);
            full->g_seed = mix64(t_seed, 2);
            full->m = m;
            full->has_g = true;
            build_perm_seeded(ctx, full, sc.st);
            uint32_t o[2];
            CGX_CUDA(cudaMemcpyAsync(&o[0], full->offsets + b0, 4, cudaMemcpyDeviceToHost, sc.st));
            CGX_CUDA(cudaMemcpyAsync(&o[1], full->offsets + b1, 4, cudaMemcpyDeviceToHost, sc.st));
            sc.sync();
            const int64_t count = (int64_t)o[1] - (int64_t)o[0];
            if (count < 1) fail(CGX_EINVAL, "countgauss_bucket_shard: no rows hash into the bucket range");
            xf = new_xform(ctx, b1 - b0, count);
            xf->grows = (uint32_t*)pool_alloc(ctx, sizeof(uint32_t) * (size_t)count);
            xf->t_seed = t_seed;
            xf->map_seed = full->map_seed;
            xf->g_seed = full->g_seed;
            xf->seeded_map = false;
            xf->m = m;
            xf->has_g = true;
            launch_bucket_shard(ctx, full, b0, b1 - b0, o[0], xf, sc.st);
            // G[:, b0:b1) of the full transform, held like an explicit G
            CGX_CUDA(cudaMalloc((void**)&xf->g_dev, sizeof(double) * (size_t)(m * (b1 - b0))));
            xf->g_explicit = true;
            launch_gen_gauss(ctx, full, b0, b1 - b0, xf->g_dev, sc.st);
            sc.sync();
        } catch (...) {
            free_xform(xf);
            free_xform(full);
            throw;
        }
        free_xform(full);
        *out = xf;
    });
}

int cgx_xform_rows(cgx_ctx* ctx, const cgx_xform* xf, int64_t* rows, int mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(mem);
        CallScope sc(ctx, stream);
        const size_t bytes = sizeof(int64_t) * (size_t)xf->n;
        int64_t* rd = mem == CGX_MEM_HOST ? (int64_t*)ctx->xstage.get(bytes) : rows;
        launch_xform_rows(ctx, xf, rd, sc.st);
        if (mem == CGX_MEM_HOST) {
            CGX_CUDA(cudaMemcpyAsync(rows, rd, bytes, cudaMemcpyDeviceToHost, sc.st));
            sc.sync();
        }
    });
}

int cgx_xform_set_gaussian_seeded(cgx_ctx* ctx, cgx_xform* xf, int64_t m, uint64_t g_seed) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        if (m < 1) fail(CGX_EINVAL, "gaussian_matrix: dimensions must be positive");
        CallScope sc(ctx, nullptr);
        drop_g(xf);
        xf->m = m;
        xf->g_seed = g_seed;
        xf->has_g = true;
        xf->g_explicit = false;
        make_g_resident(ctx, xf, sc.st);
    });
}

int cgx_xform_set_gaussian_explicit(cgx_ctx* ctx, cgx_xform* xf, int64_t m, const double* g, int mem) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(mem);
        if (m < 1) fail(CGX_EINVAL, "gaussian_matrix: dimensions must be positive");
        CallScope sc(ctx, nullptr);
        const size_t bytes = sizeof(double) * (size_t)(m * xf->B);
        double* gd = nullptr;
        CGX_CUDA(cudaMalloc((void**)&gd, bytes));
        CGX_CUDA(cudaMemcpyAsync(gd, g, bytes, mem == CGX_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                                 sc.st));
        sc.sync();
        drop_g(xf);
        xf->g_dev = gd;
        xf->m = m;
        xf->has_g = true;
        xf->g_explicit = true;
    });
}

int cgx_xform_info(const cgx_xform* xf, uint64_t* t_seed, uint64_t* map_seed, uint64_t* g_seed, int64_t* m,
                   int64_t* buckets, int64_t* input_dim) {
    return guard([&] {
        need_xf(xf);
        if (t_seed) *t_seed = xf->t_seed;
        if (map_seed) *map_seed = xf->map_seed;
        if (g_seed) *g_seed = xf->g_seed;
        if (m) *m = xf->has_g ? xf->m : 0;
        if (buckets) *buckets = xf->B;
        if (input_dim) *input_dim = xf->n;
    });
}

int cgx_xform_free(cgx_xform* xf) {
    return guard([&] {
        if (!xf) return;
        std::lock_guard<std::recursive_mutex> lk(xf->ctx->mu);
        free_xform(xf);
    });
}

int cgx_fill_hash_sign(cgx_ctx* ctx, const cgx_xform* xf, int64_t* hash, double* sign, int mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(mem);
        CallScope sc(ctx, stream);
        const size_t hb = sizeof(int64_t) * (size_t)xf->n, sb = sizeof(double) * (size_t)xf->n;
        int64_t* hd = hash;
        double* sd = sign;
        char* both = nullptr;
        if (mem == CGX_MEM_HOST) {
            both = (char*)ctx->xstage.get(hb + sb);  // hash | sign, contiguous
            hd = hash ? (int64_t*)both : nullptr;
            sd = sign ? (double*)(both + hb) : nullptr;
        }
        launch_fill_hash_sign(ctx, xf, hd, sd, sc.st);
        if (mem == CGX_MEM_HOST) {
            if (hash && sign)
                d2h_sync(ctx, both, {{hash, hb}, {sign, sb}}, sc);
            else if (hash)
                d2h_sync(ctx, hd, {{hash, hb}}, sc);
            else if (sign)
                d2h_sync(ctx, sd, {{sign, sb}}, sc);
        }
    });
}

int cgx_fill_gaussian(cgx_ctx* ctx, const cgx_xform* xf, double* g, int mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(mem);
        if (!xf->has_g) fail(CGX_EINVAL, "cgx_fill_gaussian: transform has no Gaussian factor");
        CallScope sc(ctx, stream);
        const size_t bytes = sizeof(double) * (size_t)(xf->m * xf->B);
        double* gd = mem == CGX_MEM_HOST ? (double*)ctx->xstage.get(bytes) : g;
        launch_fill_gaussian(ctx, xf, gd, sc.st);
        if (mem == CGX_MEM_HOST) {
            CGX_CUDA(cudaMemcpyAsync(g, gd, bytes, cudaMemcpyDeviceToHost, sc.st));
            sc.sync();
        }
    });
}

int cgx_inverse_normal_cdf(cgx_ctx* ctx, const double* p, double* out, int64_t count, int mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_mem(mem);
        if (count <= 0) return;
        CallScope sc(ctx, stream);
        const size_t bytes = sizeof(double) * (size_t)count;
        const double* pd = (const double*)to_device(ctx, ctx->hstage_dev, p, bytes, mem, sc.st);
        double* od = mem == CGX_MEM_HOST ? (double*)ctx->xstage.get(bytes) : out;
        int* bad = (int*)ctx->counts.get(sizeof(int));
        CGX_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), sc.st));
        launch_inverse_normal_cdf(ctx, pd, od, count, bad, sc.st);
        int hbad = 0;
        CGX_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, sc.st));
        if (mem == CGX_MEM_HOST) CGX_CUDA(cudaMemcpyAsync(out, od, bytes, cudaMemcpyDeviceToHost, sc.st));
        sc.sync();
        if (hbad) fail(CGX_EINVAL, "inverse_normal_cdf: p must lie in (0,1)");
    });
}

int cgx_countsketch_apply_dense(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int layout, int64_t ld,
                                int64_t n, int64_t d, int x_mem, double* sx, int sx_layout, int sx_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(x_mem);
        need_mem(sx_mem);
        CallScope sc(ctx, stream);
        const size_t bytes = sizeof(double) * (size_t)(xf->B * d);
        double* sxd = (sx_mem == CGX_MEM_DEVICE && sx_layout == CGX_ROW_MAJOR) ? sx : (double*)ctx->sx.get(bytes);
        sketch_dense_dev(ctx, xf, x, dtype, layout, ld, n, d, x_mem, sxd, sc.st);
        place_sx(ctx, xf, sxd, d, sx, sx_layout, sx_mem, sc);
        if (x_mem == CGX_MEM_HOST) sc.sync();
    });
}

int cgx_countsketch_apply_csr(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols, int idx_type,
                              const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz, int x_mem, double* sx,
                              int sx_layout, int sx_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(x_mem);
        need_mem(sx_mem);
        CallScope sc(ctx, stream);
        const size_t bytes = sizeof(double) * (size_t)(xf->B * d);
        double* sxd = (sx_mem == CGX_MEM_DEVICE && sx_layout == CGX_ROW_MAJOR) ? sx : (double*)ctx->sx.get(bytes);
        sketch_csr_dev(ctx, xf, rowptr, cols, idx_type, vals, dtype, n, d, nnz, x_mem, sxd, sc.st);
        place_sx(ctx, xf, sxd, d, sx, sx_layout, sx_mem, sc);
        if (x_mem == CGX_MEM_HOST) sc.sync();
    });
}

// countsketch_apply with the finished S.X rows stored by bucket range into caller-supplied
// destinations (peer-mapped landing slots): the stage 1 of CGX_COMBINE_P2P for callers that run
// one process per GPU (distributed.py "p2p").
namespace {
struct SegScope {
    cgx_ctx* ctx;
    OutSegs segs{};
    SegScope(cgx_ctx* c, const cgx_xform* xf, double* const* bases, int nseg, int64_t per) : ctx(c) {
        if (!bases || nseg < 1 || nseg > kMaxSegs || per < 1 || per * nseg < xf->B)
            fail(CGX_EINVAL, "cgx_countsketch_apply_*_to: need 1..8 destinations covering all buckets");
        for (int q = 0; q < nseg; ++q) {
            if (!bases[q]) fail(CGX_EINVAL, "cgx_countsketch_apply_*_to: null destination");
            segs.base[q] = bases[q];
        }
        segs.per = (uint32_t)per;
        ctx->out_segs = &segs;
    }
    ~SegScope() { ctx->out_segs = nullptr; }
};
} // namespace

int cgx_countsketch_apply_dense_to(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int layout, int64_t ld,
                                   int64_t n, int64_t d, int x_mem, double* const* bases, int nseg, int64_t per,
                                   void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(x_mem);
        CallScope sc(ctx, stream);
        SegScope seg(ctx, xf, bases, nseg, per);
        sketch_dense_dev(ctx, xf, x, dtype, layout, ld, n, d, x_mem, seg.segs.base[0], sc.st);
        if (x_mem == CGX_MEM_HOST) sc.sync();
    });
}

int cgx_countsketch_apply_csr_to(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols,
                                 int idx_type, const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz, int x_mem,
                                 double* const* bases, int nseg, int64_t per, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(x_mem);
        CallScope sc(ctx, stream);
        SegScope seg(ctx, xf, bases, nseg, per);
        sketch_csr_dev(ctx, xf, rowptr, cols, idx_type, vals, dtype, n, d, nnz, x_mem, seg.segs.base[0], sc.st);
        if (x_mem == CGX_MEM_HOST) sc.sync();
    });
}

int cgx_sum_slots(cgx_ctx* ctx, const double* slots, int nslots, int64_t stride, int64_t count, double* out,
                  void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (!slots || !out || nslots < 1 || stride < count || count < 0)
            fail(CGX_EINVAL, "cgx_sum_slots: bad arguments");
        CallScope sc(ctx, stream);
        launch_sum_slots(ctx, slots, nslots, stride, count, out, sc.st);
    });
}

int cgx_countgauss_apply_dense(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int layout, int64_t ld,
                               int64_t n, int64_t d, int x_mem, double* z, int z_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(x_mem);
        need_mem(z_mem);
        need_g(xf);
        CallScope sc(ctx, stream);
        int64_t rld = ld;
        const void* xd = dense_rowmajor(ctx, xf, x, &dtype, layout, ld, n, d, x_mem, &rld, sc.st);
        if (d == 0) return;
        // One-pass kernel (sketch + G generation + contraction) when G must be generated and
        // rows are narrow (d <= 64).  With G in memory, or wide rows, the two stages win: the
        // cp.async stream sketch leaves S.X in L2 and the split-K DMMA contraction streams G
        // (measured: resident G c2 0.418 vs 0.427 ms, c4 2.57 vs 3.59 ms; generated G c2
        // one-pass 0.439 ms, c4 two-stage beats one-pass 3.62 ms).
        if (!ctx->no_fuse && ((!xf->g_dev && d <= 64) || ctx->force_fuse)) {
            const size_t zb = sizeof(double) * (size_t)(xf->m * d);
            double* zd = z_mem == CGX_MEM_HOST ? (double*)ctx->tmp.get(zb) : z;
            ctx->prof.begin(0, sc.st);
            const bool fused = launch_countgauss_dense_fused(ctx, xf, xd, dtype, rld, d, zd, sc.st);
            ctx->prof.end(0, sc.st);
            if (fused) {
                if (z_mem == CGX_MEM_HOST) {
                    CGX_CUDA(cudaMemcpyAsync(z, zd, zb, cudaMemcpyDeviceToHost, sc.st));
                    sc.sync();
                }
                return;
            }
        }
        double* sxd = (double*)ctx->sx.get(sizeof(double) * (size_t)(xf->B * d));
        ctx->prof.begin(0, sc.st);
        launch_sketch_dense(ctx, xf, xd, dtype, rld, n, d, sxd, sc.st);
        ctx->prof.end(0, sc.st);
        finish_gemm(ctx, xf, sxd, d, z, z_mem, sc);
        if (x_mem == CGX_MEM_HOST) sc.sync();
    });
}

int cgx_countgauss_apply_csr(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols, int idx_type,
                             const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz, int x_mem, double* z,
                             int z_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(x_mem);
        need_mem(z_mem);
        need_g(xf);
        CallScope sc(ctx, stream);
        double* sxd = (double*)ctx->sx.get(sizeof(double) * (size_t)(xf->B * d));
        sketch_csr_dev(ctx, xf, rowptr, cols, idx_type, vals, dtype, n, d, nnz, x_mem, sxd, sc.st);
        finish_gemm(ctx, xf, sxd, d, z, z_mem, sc);
        if (x_mem == CGX_MEM_HOST) sc.sync();
    });
}

int cgx_gauss_gemm(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int sx_layout, int64_t d, int sx_mem, double* z,
                   int z_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(sx_mem);
        need_mem(z_mem);
        need_g(xf);
        if (d < 0) fail(CGX_EINVAL, "gemm: negative column count");
        CallScope sc(ctx, stream);
        const size_t bytes = sizeof(double) * (size_t)(xf->B * d);
        const double* sd = (const double*)to_device(ctx, ctx->hstage_dev, sx, bytes, sx_mem, sc.st);
        if (sx_layout == CGX_COL_MAJOR && d > 0) {
            // col-major B x d == row-major d x B -> transpose into row-major B x d
            double* rm = (double*)ctx->sx.get(bytes);
            launch_transpose_x(ctx, sd, CGX_F64, xf->B, xf->B, d, rm, sc.st);
            sd = rm;
        }
        finish_gemm(ctx, xf, sd, d, z, z_mem, sc);
    });
}

int cgx_gauss_gemm_range(cgx_ctx* ctx, const cgx_xform* xf, const double* sx_rows, int64_t b0, int64_t b1, int64_t d,
                         int sx_mem, double* z, int z_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(sx_mem);
        need_mem(z_mem);
        need_g(xf);
        if (d < 0 || b0 < 0 || b1 < b0 || b1 > xf->B) fail(CGX_EINVAL, "gemm: bad bucket range");
        CallScope sc(ctx, stream);
        const size_t bytes = sizeof(double) * (size_t)((b1 - b0) * d);
        const double* sd = (const double*)to_device(ctx, ctx->hstage_dev, sx_rows, bytes, sx_mem, sc.st);
        finish_gemm(ctx, xf, sd, d, z, z_mem, sc, b0, b1);
    });
}

int cgx_gauss_gemm_rows(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t d, int64_t r0, int64_t r1,
                        int sx_mem, double* z, int z_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(sx_mem);
        need_mem(z_mem);
        need_g(xf);
        if (d < 1 || r0 < 0 || r1 <= r0 || r1 > xf->m) fail(CGX_EINVAL, "gemm: bad row range of G");
        CallScope sc(ctx, stream);
        const size_t bytes = sizeof(double) * (size_t)(xf->B * d);
        const double* sd = (const double*)to_device(ctx, ctx->hstage_dev, sx, bytes, sx_mem, sc.st);
        const size_t zb = sizeof(double) * (size_t)((r1 - r0) * d);
        double* zd = z_mem == CGX_MEM_HOST ? (double*)ctx->tmp.get(zb) : z;
        ctx->prof.begin(1, sc.st);
        launch_gauss_gemm_rows(ctx, xf, sd, d, r0, r1, zd, sc.st);
        ctx->prof.end(1, sc.st);
        if (z_mem == CGX_MEM_HOST) {
            CGX_CUDA(cudaMemcpyAsync(z, zd, zb, cudaMemcpyDeviceToHost, sc.st));
            sc.sync();
        } else if (sx_mem == CGX_MEM_HOST) {
            sc.sync();
        }
    });
}

int cgx_gaussian_project_dense(cgx_ctx* ctx, uint64_t rng_state, int64_t m, const void* x, int dtype, int layout,
                               int64_t ld, int64_t n, int64_t d, int x_mem, double* z, int z_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_mem(x_mem);
        need_mem(z_mem);
        if (m < 1) fail(CGX_EINVAL, "anchor extraction: m must be >= 1");
        if (n < 1) fail(CGX_EINVAL, "gaussian_matrix: dimensions must be positive");
        if (d < 1) fail(CGX_EINVAL, "anchor extraction: X must have at least one column");
        CallScope sc(ctx, stream);
        // G~(r, i) = draw i*m + r of the caller's stream (gaussian_matrix, matrix.cpp:199-207):
        // the generator seed is the rng's current state.  A stack transform carries (m, n, seed).
        cgx_xform gx;
        gx.ctx = ctx;
        gx.B = n;
        gx.n = n;
        gx.m = m;
        gx.g_seed = rng_state;
        gx.has_g = true;
        gx.view = true;
        int64_t rld = ld;
        const void* xd = dense_rowmajor(ctx, &gx, x, &dtype, layout, ld, n, d, x_mem, &rld, sc.st);
        const double* x64 = (const double*)xd;
        if (dtype == CGX_F32 || rld != d) {
            double* w = (double*)ctx->sx.get(sizeof(double) * (size_t)(n * d));
            if (dtype == CGX_F32)
                launch_widen_f32(ctx, (const float*)xd, rld, n, d, w, sc.st);
            else
                CGX_CUDA(cudaMemcpy2DAsync(w, sizeof(double) * d, xd, sizeof(double) * rld, sizeof(double) * d, n,
                                           cudaMemcpyDeviceToDevice, sc.st));
            x64 = w;
        }
        const size_t zb = sizeof(double) * (size_t)(m * d);
        double* zd = z_mem == CGX_MEM_HOST ? (double*)ctx->tmp.get(zb) : z;
        ctx->prof.begin(1, sc.st);
        launch_gauss_gemm_chunked(ctx, &gx, x64, 0, n, d, zd, sc.st, true);
        ctx->prof.end(1, sc.st);
        if (z_mem == CGX_MEM_HOST) {
            CGX_CUDA(cudaMemcpyAsync(z, zd, zb, cudaMemcpyDeviceToHost, sc.st));
            sc.sync();
        }
    });
}

int cgx_gaussian_project_csr(cgx_ctx* ctx, uint64_t rng_state, int64_t m, const int64_t* rowptr, const void* cols,
                             int idx_type, const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz, int x_mem,
                             double* z, int z_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_mem(x_mem);
        need_mem(z_mem);
        const size_t es = dsize(dtype);
        if (idx_type != CGX_I32 && idx_type != CGX_I64) fail(CGX_EINVAL, "cgx: idx_type must be CGX_I32 or CGX_I64");
        if (m < 1) fail(CGX_EINVAL, "anchor extraction: m must be >= 1");
        if (n < 1) fail(CGX_EINVAL, "gaussian_matrix: dimensions must be positive");
        if (d < 1) fail(CGX_EINVAL, "anchor extraction: X must have at least one column");
        if (nnz < 0) fail(CGX_EINVAL, "cgx: negative size");
        CallScope sc(ctx, stream);
        const void* rp = rowptr;
        const void* cp = cols;
        const void* vp = vals;
        (void)es;
        stage_csr(ctx, &rp, &cp, &idx_type, &vp, &dtype, n, nnz, x_mem, sc.st);
        const size_t zb = sizeof(double) * (size_t)(m * d);
        double* zd = z_mem == CGX_MEM_HOST ? (double*)ctx->tmp.get(zb) : z;
        ctx->prof.begin(1, sc.st);
        launch_gproject_csr(ctx, rng_state, m, (const int64_t*)rp, cp, idx_type, vp, dtype, n, d, zd, sc.st);
        ctx->prof.end(1, sc.st);
        if (z_mem == CGX_MEM_HOST) {
            CGX_CUDA(cudaMemcpyAsync(z, zd, zb, cudaMemcpyDeviceToHost, sc.st));
            sc.sync();
        } else if (x_mem == CGX_MEM_HOST) {
            sc.sync();
        }
    });
}

int cgx_select_extremes(cgx_ctx* ctx, const double* z, int64_t m, int64_t d, int mem, int64_t* amax, int64_t* amin,
                        int64_t* tie_rows, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_mem(mem);
        if (m < 1) fail(CGX_EINVAL, "anchor extraction: m must be >= 1");
        if (d < 1) fail(CGX_EINVAL, "anchor extraction: X must have at least one column");
        CallScope sc(ctx, stream);
        const double* zd = (const double*)to_device(ctx, ctx->hstage_dev, z, sizeof(double) * (size_t)(m * d), mem, sc.st);
        int64_t* outs = (int64_t*)ctx->counts.get(sizeof(int64_t) * (size_t)(3 * m));
        launch_select_extremes(ctx, zd, m, d, outs, outs + m, outs + 2 * m, sc.st);
        std::vector<int64_t> h((size_t)(3 * m));
        CGX_CUDA(cudaMemcpyAsync(h.data(), outs, sizeof(int64_t) * (size_t)(3 * m), cudaMemcpyDeviceToHost, sc.st));
        sc.sync();
        if (mem == CGX_MEM_HOST) {
            std::copy(h.begin(), h.begin() + m, amax);
            std::copy(h.begin() + m, h.begin() + 2 * m, amin);
        } else {
            CGX_CUDA(cudaMemcpyAsync(amax, outs, sizeof(int64_t) * (size_t)m, cudaMemcpyDeviceToDevice, sc.st));
            CGX_CUDA(cudaMemcpyAsync(amin, outs + m, sizeof(int64_t) * (size_t)m, cudaMemcpyDeviceToDevice, sc.st));
            sc.sync();
        }
        int64_t t = 0;
        for (int64_t r = 0; r < m; ++r) t += h[(size_t)(2 * m + r)];
        if (tie_rows) *tie_rows = t;
    });
}

int cgx_csr_save(const char* path, const int64_t* rowptr, const void* cols, int idx_type, const void* vals, int dtype,
                 int64_t n, int64_t d, int64_t nnz) {
    return guard([&] {
        if (!path) fail(CGX_EINVAL, "cgx_csr_save: null path");
        csr_save(path, rowptr, cols, idx_type, vals, dtype, n, d, nnz);
    });
}

int cgx_csr_info(const char* path, int64_t* n, int64_t* d, int64_t* nnz, int* idx_type, int* dtype) {
    return guard([&] {
        if (!path) fail(CGX_EINVAL, "cgx_csr_info: null path");
        csr_info(path, n, d, nnz, idx_type, dtype);
    });
}

int cgx_csr_load(cgx_ctx* ctx, const char* path, int64_t* rowptr, void* cols, void* vals, int mem, void* stream) {
    return guard([&] {
        need_mem(mem);
        if (!path) fail(CGX_EINVAL, "cgx_csr_load: null path");
        if (mem == CGX_MEM_HOST) {  // plain file read, no device involved (ctx may be null)
            csr_load(nullptr, path, rowptr, cols, vals, mem, nullptr);
            return;
        }
        need_ctx(ctx);
        CallScope sc(ctx, stream);
        csr_load(ctx, path, rowptr, cols, vals, mem, sc.st);
    });
}

int cgx_countgauss_materialize(cgx_ctx* ctx, const cgx_xform* xf, double* t, int mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_xf(xf);
        need_mem(mem);
        need_g(xf);
        CallScope sc(ctx, stream);
        const size_t bytes = sizeof(double) * (size_t)(xf->m * xf->n);
        double* td = mem == CGX_MEM_HOST ? (double*)ctx->tmp.get(bytes) : t;
        launch_materialize_t(ctx, xf, td, sc.st);
        if (mem == CGX_MEM_HOST) {
            CGX_CUDA(cudaMemcpyAsync(t, td, bytes, cudaMemcpyDeviceToHost, sc.st));
            sc.sync();
        }
    });
}

int cgx_countsketch_batch_gram(cgx_ctx* ctx, uint64_t master, int64_t t0, int64_t trials, int64_t buckets,
                               const double* u, int64_t ld, int64_t n, int64_t d, int u_mem, double* su,
                               double* gram, int out_mem, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        need_mem(u_mem);
        need_mem(out_mem);
        if (buckets < 1 || n < 1) fail(CGX_EINVAL, "countsketch_new: buckets and input_dim must be >= 1");
        if (trials < 0 || d < 1 || t0 < 0) fail(CGX_EINVAL, "cgx_countsketch_batch_gram: need trials >= 0, d >= 1");
        if (ld < n) fail(CGX_EINVAL, "cgx_countsketch_batch_gram: ld < n");
        if (trials == 0) return;
        CallScope sc(ctx, stream);
        const double* ud = (const double*)to_device(ctx, ctx->hstage_dev, u, sizeof(double) * (size_t)(ld * d), u_mem,
                                                    sc.st);
        const size_t su_b = sizeof(double) * (size_t)(trials * buckets * d), g_b = sizeof(double) * (size_t)(trials * d * d);
        double* sud = su;
        double* gd = gram;
        if (out_mem == CGX_MEM_HOST) {
            char* base = (char*)ctx->tmp.get((su ? su_b : 0) + (gram ? g_b : 0));
            sud = su ? (double*)base : nullptr;
            gd = gram ? (double*)(base + (su ? su_b : 0)) : nullptr;
        }
        launch_batch_sketch_gram(ctx, master, t0, trials, buckets, ud, ld, n, d, sud, gd, sc.st);
        if (out_mem == CGX_MEM_HOST) {
            if (su) CGX_CUDA(cudaMemcpyAsync(su, sud, su_b, cudaMemcpyDeviceToHost, sc.st));
            if (gram) CGX_CUDA(cudaMemcpyAsync(gram, gd, g_b, cudaMemcpyDeviceToHost, sc.st));
            sc.sync();
        } else if (u_mem == CGX_MEM_HOST) {
            sc.sync();  // the staged U must outlive the kernel
        }
    });
}

int cgx_gen_dense_normal(cgx_ctx* ctx, uint64_t seed, int64_t row0, int64_t n, int64_t d, int dtype, int layout,
                         void* x_dev, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        dsize(dtype);
        if (n < 0 || d < 0) fail(CGX_EINVAL, "cgx_gen_dense_normal: negative size");
        if (n * d == 0) return;
        CallScope sc(ctx, stream);
        if (row0 < 0) fail(CGX_EINVAL, "cgx_gen_dense_normal: negative row0");
        launch_gen_dense(ctx, seed, row0, nullptr, n, d, dtype, layout, x_dev, sc.st);
    });
}

int cgx_gen_dense_normal_rows(cgx_ctx* ctx, uint64_t seed, const int64_t* rows_dev, int64_t n, int64_t d, int dtype,
                              int layout, void* x_dev, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        dsize(dtype);
        if (n < 0 || d < 0) fail(CGX_EINVAL, "cgx_gen_dense_normal_rows: negative size");
        if (n * d == 0) return;
        if (!rows_dev) fail(CGX_EINVAL, "cgx_gen_dense_normal_rows: null rows");
        CallScope sc(ctx, stream);
        launch_gen_dense(ctx, seed, 0, rows_dev, n, d, dtype, layout, x_dev, sc.st);
    });
}

int cgx_host_checksum(cgx_ctx* ctx, const void* p, size_t bytes, uint64_t* out) {
    return guard([&] {
        if (!out || (!p && bytes)) fail(CGX_EINVAL, "cgx_host_checksum: null argument");
        if (ctx) {
            std::lock_guard<std::recursive_mutex> lk(ctx->mu);
            *out = host_checksum(ctx, p, bytes);
        } else {
            *out = host_checksum(nullptr, p, bytes);
        }
    });
}

int cgx_separable_mixing(uint64_t seed, int64_t r, int64_t cols, double alpha, double* h) {
    return guard([&] {
        if (r < 1 || cols < 0) fail(CGX_EINVAL, "cgx_separable_mixing: need r >= 1 and cols >= 0");
        if (!(alpha > 0.0) || !std::isfinite(alpha)) fail(CGX_EINVAL, "cgx_separable_mixing: alpha must be > 0");
        if (!h && r * cols > 0) fail(CGX_EINVAL, "cgx_separable_mixing: null output");
        separable_mixing(seed, r, cols, alpha, h);
    });
}

int cgx_gen_separable(cgx_ctx* ctx, uint64_t seed, int64_t row0, int64_t n, int64_t d, int64_t r, double alpha,
                      double sigma, int dtype, int layout, void* x_dev, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        dsize(dtype);
        if (layout != CGX_COL_MAJOR && layout != CGX_ROW_MAJOR) fail(CGX_EINVAL, "cgx_gen_separable: bad layout");
        if (n < 0 || row0 < 0) fail(CGX_EINVAL, "cgx_gen_separable: negative size");
        if (r < 1 || r > d) fail(CGX_EINVAL, "cgx_gen_separable: need 1 <= r <= d");
        if (!(alpha > 0.0) || !std::isfinite(alpha)) fail(CGX_EINVAL, "cgx_gen_separable: alpha must be > 0");
        if (!(sigma >= 0.0) || !std::isfinite(sigma)) fail(CGX_EINVAL, "cgx_gen_separable: sigma must be >= 0");
        if (n == 0) return;
        CallScope sc(ctx, stream);
        launch_gen_separable(ctx, seed, row0, n, d, r, alpha, sigma, dtype, layout, x_dev, sc.st);
    });
}

int cgx_gen_csr_bernoulli(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, double density, int64_t* rowptr_dev,
                          int32_t* cols_dev, float* vals_dev, int64_t* nnz_out, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (n < 1 || d < 1) fail(CGX_EINVAL, "cgx_gen_csr_bernoulli: n and d must be >= 1");
        if (!(density >= 0.0 && density <= 1.0)) fail(CGX_EINVAL, "cgx_gen_csr_bernoulli: density must lie in [0,1]");
        CsrGenSpec spec;
        spec.density = density;
        gen_csr(ctx, seed, n, d, spec, rowptr_dev, cols_dev, vals_dev, nnz_out, stream);
    });
}

int cgx_gen_csr_zipf(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, double s_len, int64_t cap, double s_col,
                     int64_t* rowptr_dev, int32_t* cols_dev, float* vals_dev, int64_t* nnz_out, void* stream) {
    return guard([&] {
        need_ctx(ctx);
        if (n < 1 || d < 1 || cap < 1 || cap > d) fail(CGX_EINVAL, "cgx_gen_csr_zipf: need n, d >= 1 and 1 <= cap <= d");
        if (!(s_len > 0.0) || !(s_col >= 0.0)) fail(CGX_EINVAL, "cgx_gen_csr_zipf: bad exponents");
        CsrGenSpec spec;
        spec.zipf = true;
        spec.s_len = s_len;
        spec.s_col = s_col;
        spec.cap = (int)cap;
        gen_csr(ctx, seed, n, d, spec, rowptr_dev, cols_dev, vals_dev, nnz_out, stream);
    });
}

uint64_t cgx_launch_count(const cgx_ctx* ctx) { return ctx ? ctx->launches : 0; }

int cgx_set_option(cgx_ctx* ctx, const char* key, int64_t value) {
    return guard([&] {
        need_ctx(ctx);
        if (!key) fail(CGX_EINVAL, "cgx_set_option: null key");
        std::lock_guard<std::recursive_mutex> lk(ctx->mu);
        const std::string k(key);
        if (k == "fuse") {
            ctx->no_fuse = value == 0;
            ctx->force_fuse = value == 2;
        } else if (k == "fuse_mode" && (value == 1 || value == 2))
            ctx->fuse_mode = (int)value;
        else if (k == "rows_per_task" && value >= 1)
            ctx->opt_rows_per_task = value;
        else if (k == "tail_tasks" && value >= 0 && value <= 64)
            ctx->opt_tail_tasks = value;
        else if (k == "grid_waves" && value >= 1)
            ctx->opt_grid_waves = value;
        else if (k == "ws_gw" && value >= 0 && value <= 8)
            ctx->opt_ws_gw = value;
        else if (k == "async_stages" && (value == 0 || (value >= 2 && value <= 4)))
            ctx->opt_async = value;
        else if (k == "csr_mode" && (value == 0 || value == 1 || value == 3))
            ctx->opt_csr_mode = value;
        else if (k == "csr_slice_mb" && value >= 1 && value <= 1024)
            ctx->opt_csr_slice_mb = value;
        else if (k == "gather_sms" && value >= 0)
            ctx->opt_gather_sms = value;
        else if (k == "csr_zero" && (value == 0 || value == 1))
            ctx->opt_csr_zero = value;
        else if (k == "g_resident" && (value == 0 || value == 1))
            ctx->opt_g_resident = value;
        else if (k == "gemm_tile" && (value == 0 || value == 1))
            ctx->opt_gemm_tile = value;
        else if (k == "oz_slices" && (value == 0 || (value >= 3 && value <= 7)))
            ctx->opt_oz_slices = value;
        else if (k == "pdl" && (value == 0 || value == 1))
            ctx->opt_pdl = value;
        else if (k == "oz_cluster" && (value == 1 || value == 2 || value == 4 || value == 8))
            ctx->opt_oz_cluster = value;
        else if (k == "oz_st" && value >= 0 && value <= 8)
            ctx->opt_oz_st = value;
        else if (k == "oz_rs" && value >= 0 && value <= 8)
            ctx->opt_oz_rs = value;
        else if (k == "oz_min_z" && value >= 0)
            ctx->opt_oz_min_z = value;
        else if (k == "oz_staged" && (value == 0 || value == 1))
            ctx->opt_oz_staged = value;
        else if (k == "oz_mpair" && (value == 0 || value == 1))
            ctx->opt_oz_mpair = value;
        else if (k == "gemm_chunks" && (value == 0 || value == 1))
            ctx->opt_gemm_chunks = value;
        else
            fail(CGX_EINVAL, "cgx_set_option: unknown key '" + k + "'");
    });
}

int cgx_profile_enable(cgx_ctx* ctx, int on) {
    return guard([&] {
        need_ctx(ctx);
        std::lock_guard<std::recursive_mutex> lk(ctx->mu);
        ctx->prof.on = on != 0;
        ctx->prof.used[0] = ctx->prof.used[1] = 0;
    });
}

int cgx_profile_read(cgx_ctx* ctx, int stage, double* total_ms, int64_t* launches) {
    return guard([&] {
        need_ctx(ctx);
        if (stage < 0 || stage > 1) fail(CGX_EINVAL, "cgx_profile_read: stage must be 0 or 1");
        std::lock_guard<std::recursive_mutex> lk(ctx->mu);
        CGX_CUDA(cudaSetDevice(ctx->device));
        double tot = 0.0;
        auto& v = ctx->prof.ev[stage];
        for (size_t i = 0; i < ctx->prof.used[stage]; ++i) {
            CGX_CUDA(cudaEventSynchronize(v[i].second));
            float ms = 0.f;
            CGX_CUDA(cudaEventElapsedTime(&ms, v[i].first, v[i].second));
            tot += ms;
        }
        if (total_ms) *total_ms = tot;
        if (launches) *launches = (int64_t)ctx->prof.used[stage];
        ctx->prof.used[stage] = 0;
    });
}

} // extern "C"
