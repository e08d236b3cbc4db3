// hoststage.cu -- host-side input staging for the as-is API: the reference's DenseMatrix /
// SparseMatrix live in pageable std::vector storage (matrix.hpp:16-61), and a plain
// cudaMemcpy from pageable memory runs at ~11 GB/s on the B200 box against ~55 GB/s from
// pinned memory (tools/microbench/h2d.cu).  Host arrays therefore go through a ring of
// pinned chunks filled by a persistent pool of host threads while the copy engine drains
// the previous chunks.
//
// Lossless narrowing on the way: a chunk of fp64 values that are all exactly representable
// in fp32 (or of int64 column indices that all fit int32) is sent at half width and
// widened back on the device -- or, when the whole array narrowed, handed to the kernels
// as fp32 / int32, which they take natively.  The device sees exactly the caller's values
// in every case; the check is per chunk, and a chunk that fails it is sent at full width.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <immintrin.h>
#include <thread>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace cgx {

// ---- persistent host thread pool ---------------------------------------------------------
// Workers and the caller spin briefly (60 us by default) before they block: a staging call issues one
// job per chunk a few microseconds apart, and a condition-variable sleep and wake-up per
// worker and job cost ~40 us of every one of them (13 jobs in a 68 MB CSR call).
struct HostPool {
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv, done_cv;
    std::function<void(int)> job;
    std::atomic<uint64_t> gen{0};
    std::atomic<int> pending{0};
    bool quit = false;
    // Spinning pays only where the jobs are short (arrays under 16 MB: c1 through the drop-in
    // 0.46 -> 0.24 ms): on long arrays the spinners slowed the working threads' cores (c2
    // through the drop-in 67 -> 83 ms; 32 MB CSR arrays 2.17 -> 2.38 ms), so the caller sets
    // `spin` per array: stage_in / host_checksum -> set_spin.
    std::atomic<int> spin{0};
    static int spin_default() {  // CGX_POOL_SPIN_US overrides (0: always block at once)
        static const int v = [] {
            const char* e = getenv("CGX_POOL_SPIN_US");
            return e ? atoi(e) : 60;
        }();
        return v;
    }
    void set_spin(bool short_jobs) { spin.store(short_jobs ? spin_default() : 0, std::memory_order_relaxed); }

    template <class Pred>
    bool spin_until(Pred&& pred) {
        const int limit = spin.load(std::memory_order_relaxed);
        if (limit <= 0) return pred();
        const auto t0 = std::chrono::steady_clock::now();
        for (int it = 0;; ++it) {
            if (pred()) return true;
            _mm_pause();
            if ((it & 63) == 63 &&
                std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() > limit)
                return false;
        }
    }

    explicit HostPool(int n) {
        for (int k = 0; k < n; ++k)
            th.emplace_back([this, k] {
                uint64_t seen = 0;
                for (;;) {
                    std::function<void(int)> f;
                    if (!spin_until([&] { return gen.load(std::memory_order_acquire) != seen; })) {
                        std::unique_lock<std::mutex> lk(mu);
                        cv.wait(lk, [&] { return quit || gen.load(std::memory_order_acquire) != seen; });
                    }
                    {
                        std::lock_guard<std::mutex> lk(mu);
                        if (quit) return;
                        seen = gen.load(std::memory_order_acquire);
                        f = job;
                    }
                    f(k + 1);
                    if (pending.fetch_sub(1, std::memory_order_acq_rel) == 1) {
                        std::lock_guard<std::mutex> lk(mu);
                        done_cv.notify_all();
                    }
                }
            });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu);
            quit = true;
            gen.fetch_add(1, std::memory_order_release);
        }
        cv.notify_all();
        for (auto& t : th) t.join();
    }
    int size() const { return (int)th.size() + 1; }
    // f(k) for k = 0 .. size()-1, k = 0 on the calling thread; returns when all are done
    void run(const std::function<void(int)>& f) {
        {
            std::lock_guard<std::mutex> lk(mu);
            job = f;
            pending.store((int)th.size(), std::memory_order_release);
            gen.fetch_add(1, std::memory_order_release);
        }
        cv.notify_all();
        f(0);
        if (spin_until([&] { return pending.load(std::memory_order_acquire) == 0; })) return;
        std::unique_lock<std::mutex> lk(mu);
        done_cv.wait(lk, [&] { return pending.load(std::memory_order_acquire) == 0; });
    }
};

namespace {

constexpr size_t kChunk = (size_t)32 << 20;  // source bytes per pipeline chunk
constexpr int kSlots = 4;

HostPool& pool_of(cgx_ctx* ctx) {
    if (!ctx->hpool) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        ctx->hpool = new HostPool((int)std::min(32u, hw) - 1);
    }
    return *ctx->hpool;
}

void ensure_ring(cgx_ctx* ctx) {
    if (ctx->ring) return;
    CGX_CUDA(cudaMallocHost((void**)&ctx->ring, kChunk * kSlots));
    for (int s = 0; s < kSlots; ++s) CGX_CUDA(cudaEventCreateWithFlags(&ctx->ring_ev[s], cudaEventDisableTiming));
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Narrow len values of src into dst; false as soon as some value does not round-trip.
// Cloned for AVX-512 / AVX2 hosts (the B200 boxes' Xeons have both), with a baseline
// fallback.
#define CGX_HOST_SIMD __attribute__((target_clones("avx512f", "avx2", "default")))
CGX_HOST_SIMD bool narrow_f64(const double* src, float* dst, size_t len) {
    for (size_t i = 0; i < len; i += 4096) {
        const size_t e = std::min(len, i + 4096);
        unsigned bad = 0;
        for (size_t k = i; k < e; ++k) {
            const float f = (float)src[k];
            dst[k] = f;
            bad |= (unsigned)((double)f != src[k]);
        }
        if (bad) return false;
    }
    return true;
}
CGX_HOST_SIMD bool narrow_i64(const int64_t* src, int32_t* dst, size_t len) {
    for (size_t i = 0; i < len; i += 4096) {
        const size_t e = std::min(len, i + 4096);
        unsigned bad = 0;
        for (size_t k = i; k < e; ++k) {
            const int32_t v = (int32_t)src[k];
            dst[k] = v;
            bad |= (unsigned)((int64_t)v != src[k]);
        }
        if (bad) return false;
    }
    return true;
}

// memcpy into the pinned ring with non-temporal stores: the ring is written once and read
// only by the copy engine, so the stores skip the read-for-ownership of every destination
// line that a plain memcpy of these 2 MiB per-thread pieces pays (glibc switches to
// streaming stores only for much larger copies).
__attribute__((target("avx512f"))) static void copy_nt_avx512(char* dst, const char* src, size_t n) {
    while (n && ((uintptr_t)dst & 63)) {
        *dst++ = *src++;
        --n;
    }
    for (; n >= 256; n -= 256, dst += 256, src += 256) {
        const __m512i a = _mm512_loadu_si512(src), b = _mm512_loadu_si512(src + 64);
        const __m512i c = _mm512_loadu_si512(src + 128), d = _mm512_loadu_si512(src + 192);
        _mm512_stream_si512((__m512i*)dst, a);
        _mm512_stream_si512((__m512i*)(dst + 64), b);
        _mm512_stream_si512((__m512i*)(dst + 128), c);
        _mm512_stream_si512((__m512i*)(dst + 192), d);
    }
    _mm_sfence();
    std::memcpy(dst, src, n);
}
static void copy_nt(char* dst, const char* src, size_t n) {
    static const bool avx512 = __builtin_cpu_supports("avx512f");
    if (avx512 && n >= 4096)
        copy_nt_avx512(dst, src, n);
    else
        std::memcpy(dst, src, n);
}

// Elements [e, e_end) of a source made of segments of `seg` elements spaced `sld`
// elements apart (a column-major row block: seg = rows, sld = ld), as contiguous pieces:
// fn(source element offset, destination element offset relative to e, length).
template <class F>
bool for_pieces(size_t e, size_t e_end, size_t seg, size_t sld, F&& fn) {
    const size_t base = e;
    while (e < e_end) {
        const size_t si = e / seg, off = e - si * seg;
        const size_t len = std::min(seg - off, e_end - e);
        if (!fn(si * sld + off, e - base, len)) return false;
        e += len;
    }
    return true;
}

template <typename N, typename W>
__global__ void widen_kernel(const N* __restrict__ src, W* __restrict__ dst, size_t count) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = (W)src[i];
}

} // namespace

void host_pool_free(cgx_ctx* ctx) {
    delete ctx->hpool;
    ctx->hpool = nullptr;
    if (ctx->ring) {
        for (int s = 0; s < kSlots; ++s) cudaEventDestroy(ctx->ring_ev[s]);
        cudaFreeHost(ctx->ring);
        ctx->ring = nullptr;
    }
}

// Copy `count` elements of `esize` bytes from host `src` to the device.  kind: 0 plain,
// 1 fp64 -> fp32 narrowing allowed, 2 int64 -> int32 narrowing allowed.  Returns the device
// pointer and sets *narrowed when the whole array arrived narrowed (then the result holds
// count elements of esize/2 bytes).  `full` / `half` are the device landing buffers.
const void* stage_in(cgx_ctx* ctx, DevBuf& full, DevBuf& half, const void* src, size_t count, size_t esize, int kind,
                     bool* narrowed, cudaStream_t s, size_t seg, size_t sld) {
    *narrowed = false;
    const size_t bytes = count * esize;
    if (bytes == 0) return src;
    // contiguous (no gaps between segments): one piece.  (A dense row-major X arrives as
    // segments of d elements at stride d; as a 2-D copy of 2^24 rows of 128 B the DMA ran at
    // 51 GB/s instead of 55.6, and through the ring every 128 B row was a memcpy of its own.)
    if (seg == 0 || seg >= count || sld == seg) seg = sld = count;
    if (bytes < ((size_t)1 << 20) || is_pinned(src)) {  // small, or already DMA-able: one copy
        void* d = full.get(bytes);
        if (seg == count)
            CGX_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s));  // pageable: returns once consumed
        else
            CGX_CUDA(cudaMemcpy2DAsync(d, seg * esize, src, sld * esize, seg * esize, count / seg,
                                       cudaMemcpyHostToDevice, s));
        return d;
    }
    static const bool trace = getenv("CGX_TRACE_STAGE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    double t_wait = 0, t_narrow = 0, t_copy = 0;
    auto since = [](std::chrono::steady_clock::time_point a) {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count();
    };
    ensure_ring(ctx);
    HostPool& pool = pool_of(ctx);
    pool.set_spin(bytes < ((size_t)16 << 20));
    char* dfull = nullptr;                 // allocated when some chunk goes at full width
    char* dhalf = kind ? (char*)half.get(bytes / 2) : nullptr;
    // elements per chunk: a ring slot's worth for long arrays; a mid-sized array (up to a few
    // slots) goes in ~8 smaller chunks, or its one or two big chunks would be filled and then
    // copied with next to no overlap
    size_t chunk_bytes = kChunk;
    if (bytes < 4 * kChunk) chunk_bytes = std::min(kChunk, std::max<size_t>((size_t)2 << 20, (bytes / 4 + 0xfffff) & ~(size_t)0xfffff));
    const size_t per_chunk = chunk_bytes / esize;
    const size_t nchunks = (count + per_chunk - 1) / per_chunk;
    std::vector<char> chunk_narrow(nchunks, 0);
    bool try_narrow = kind != 0;
    const int T = pool.size();
    for (size_t c = 0; c < nchunks; ++c) {
        const int slot = (int)(ctx->ring_next++ % kSlots);  // rotates across calls: back-to-back arrays overlap
        auto tw = std::chrono::steady_clock::now();
        CGX_CUDA(cudaEventSynchronize(ctx->ring_ev[slot]));  // the slot's previous copy (this call or an earlier one)
        t_wait += since(tw);
        tw = std::chrono::steady_clock::now();
        char* buf = ctx->ring + (size_t)slot * kChunk;
        const size_t e0 = c * per_chunk, ne = std::min(per_chunk, count - e0);
        const char* sp = (const char*)src;
        bool ok = false;
        if (try_narrow) {
            std::atomic<int> bad{0};
            pool.run([&](int k) {
                const size_t a = e0 + ne * k / T, b = e0 + ne * (k + 1) / T;
                const size_t h = esize / 2;
                const bool good = for_pieces(a, b, seg, sld, [&](size_t so, size_t dofs, size_t len) {
                    char* dst = buf + (a - e0 + dofs) * h;
                    return kind == 1 ? narrow_f64((const double*)(sp + so * esize), (float*)dst, len)
                                     : narrow_i64((const int64_t*)(sp + so * esize), (int32_t*)dst, len);
                });
                if (!good) bad.store(1);
            });
            ok = bad.load() == 0;
            if (!ok) try_narrow = false;  // data that does not narrow: stop paying for the check
        }
        t_narrow += since(tw);
        tw = std::chrono::steady_clock::now();
        if (ok) {
            chunk_narrow[c] = 1;
            CGX_CUDA(cudaMemcpyAsync(dhalf + e0 * esize / 2, buf, ne * esize / 2, cudaMemcpyHostToDevice, s));
        } else {
            pool.run([&](int k) {
                const size_t a = e0 + ne * k / T, b = e0 + ne * (k + 1) / T;
                for_pieces(a, b, seg, sld, [&](size_t so, size_t dofs, size_t len) {
                    copy_nt(buf + (a - e0 + dofs) * esize, sp + so * esize, len * esize);
                    return true;
                });
            });
            if (!dfull) dfull = (char*)full.get(bytes);
            CGX_CUDA(cudaMemcpyAsync(dfull + e0 * esize, buf, ne * esize, cudaMemcpyHostToDevice, s));
        }
        CGX_CUDA(cudaEventRecord(ctx->ring_ev[slot], s));
        t_copy += since(tw);
    }
    if (trace)
        fprintf(stderr, "stage_in %zu B x %zu (kind %d, seg %zu): %.1f us total, wait %.1f, narrow %.1f, copy+dma %.1f\n",
                esize, count, kind, seg, since(t_start), t_wait, t_narrow, t_copy);
    if (!dfull) {  // every chunk narrowed
        *narrowed = true;
        return dhalf;
    }
    for (size_t c = 0; c < nchunks; ++c) {  // widen the narrowed chunks into place
        if (!chunk_narrow[c]) continue;
        const size_t e0 = c * per_chunk, ne = std::min(per_chunk, count - e0);
        const unsigned blocks = (unsigned)std::min<size_t>((ne + 255) / 256, (size_t)ctx->num_sms * 8);
        if (kind == 1)
            widen_kernel<float, double><<<blocks, 256, 0, s>>>((const float*)dhalf + e0, (double*)dfull + e0, ne);
        else
            widen_kernel<int32_t, int64_t><<<blocks, 256, 0, s>>>((const int32_t*)dhalf + e0, (int64_t*)dfull + e0, ne);
        count_launch(ctx);
        check_launch("widen");
    }
    return dfull;
}

// 64-bit content checksum of a host array (the drop-in shim's check that a transform's
// public fields still hold what construction put there).  Per 64 KiB block a multiply-mix
// hash of its 8-byte words, combined in block order: independent of the thread count.
uint64_t host_checksum(cgx_ctx* ctx, const void* p, size_t bytes) {
    const size_t blk = (size_t)64 << 10;
    const size_t nb = (bytes + blk - 1) / blk;
    std::vector<uint64_t> part(nb);
    auto body = [&](size_t b) {
        const unsigned char* q = (const unsigned char*)p + b * blk;
        const size_t len = std::min(blk, bytes - b * blk);
        uint64_t h = 0x243F6A8885A308D3ULL ^ (uint64_t)b, h2 = 0x13198A2E03707344ULL;
        size_t i = 0;
        for (; i + 16 <= len; i += 16) {
            uint64_t w0, w1;
            std::memcpy(&w0, q + i, 8);
            std::memcpy(&w1, q + i + 8, 8);
            h = (h ^ w0) * 0x9E3779B97F4A7C15ULL;
            h2 = (h2 ^ w1) * 0xBF58476D1CE4E5B9ULL;
        }
        for (; i < len; ++i) h = (h ^ q[i]) * 0x100000001B3ULL;
        part[b] = fin64(h ^ fin64(h2 + len));
    };
    if (ctx && bytes >= ((size_t)256 << 10)) {
        HostPool& pool = pool_of(ctx);
        pool.set_spin(bytes < ((size_t)16 << 20));
        const int T = pool.size();
        pool.run([&](int k) {
            for (size_t b = (size_t)k; b < nb; b += (size_t)T) body(b);
        });
    } else {
        for (size_t b = 0; b < nb; ++b) body(b);
    }
    uint64_t h = fin64(bytes);
    for (size_t b = 0; b < nb; ++b) h = fin64(h ^ part[b]) + (uint64_t)b;
    return h;
}

} // namespace cgx
