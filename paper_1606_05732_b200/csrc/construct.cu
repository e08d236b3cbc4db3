// construct.cu -- transform construction: the CountSketch hash/sign generator and the
// bucket-sorted row permutation every apply kernel walks.
//
// The reference materializes hash[i], sign[i] for every row (countsketch_new,
// sketch.cpp:12-28; 16 B/row) and re-reads them in every apply.  Here a transform keeps
//   perm[n]      uint32: row | (sign<0)<<31, rows sorted by (bucket, row)
//   offsets[B+1] uint32: bucket b owns perm[offsets[b] .. offsets[b+1])
// (4 B/row).  Sorting by (bucket, row) is what lets every apply kernel sum each
// (bucket, column) in ascending row order -- the reference's order -- without atomics,
// so S.X is bit-identical to the reference and deterministic run to run.
//
// The sort is a stable LSD radix sort over the bucket bits (8 bits per pass).  Its
// first pass computes (bucket, sign) straight from the SplitMix64 index map
// (bucket = draw 2i mod B, sign = parity of draw 2i+1), so no hash array is ever
// stored.  Stability comes from a per-tile rank built with warp lane matching and
// per-warp digit counters, processed in index order.
#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

constexpr int kThreads = 256;
constexpr int kRounds = 16;
constexpr int kTile = kThreads * kRounds;  // 4096 items per CTA
constexpr int kWarps = kThreads / 32;

struct KeySrc {
    // mode 0: seeded (computed from the row index); mode 1: arrays
    const uint32_t* keys;
    const uint32_t* vals;
    uint64_t cs_seed;
    FastMod mod;
    int64_t row0;  // global index of local row 0
};

template <int MODE>
__device__ __forceinline__ void load_item(const KeySrc& src, int64_t idx, uint32_t& key, uint32_t& val) {
    if (MODE == 0) {
        const uint64_t gi = (uint64_t)(src.row0 + idx);
        key = cs_bucket(src.cs_seed, gi, src.mod);
        val = (uint32_t)idx | (cs_negative(src.cs_seed, gi) << 31);
    } else {
        key = src.keys[idx];
        val = src.vals[idx];
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) radix_hist(KeySrc src, int64_t n, int shift, int64_t ntiles,
                                                         uint32_t* hist) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kTile;
    for (int r = 0; r < kRounds; ++r) {
        const int64_t idx = base + r * kThreads + threadIdx.x;
        if (idx < n) {
            uint32_t key, val;
            load_item<MODE>(src, idx, key, val);
            atomicAdd(&h[(key >> shift) & 255u], 1u);
        }
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

template <int MODE>
__global__ void __launch_bounds__(kThreads) radix_scatter(KeySrc src, int64_t n, int shift, int64_t ntiles,
                                                            const uint32_t* offs, uint32_t* kout, uint32_t* vout) {
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_wcnt[kWarps][256];
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    s_base[tid] = offs[(int64_t)tid * ntiles + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s_wcnt[w][tid] = 0;
    __syncthreads();
    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * kTile;
    for (int r = 0; r < kRounds; ++r) {
        if (base + r * kThreads >= n) break;  // uniform across the CTA
        const int64_t idx = base + r * kThreads + tid;
        const bool valid = idx < n;
        uint32_t key = 0, val = 0;
        if (valid) load_item<MODE>(src, idx, key, val);
        const uint32_t digit = valid ? ((key >> shift) & 255u) : 256u;
        const unsigned peers = match_any_bits(digit, 9);  // digit <= 256
        const unsigned rank = __popc(peers & lt_mask);
        if (valid && rank == 0) s_wcnt[warp][digit] = __popc(peers);
        __syncthreads();
        if (valid) {
            uint32_t pos = s_base[digit] + rank;
            for (unsigned w = 0; w < warp; ++w) pos += s_wcnt[w][digit];
            if (kout) kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
        uint32_t sum = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            sum += s_wcnt[w][tid];
            s_wcnt[w][tid] = 0;
        }
        s_base[tid] += sum;
        __syncthreads();
    }
}

template <int MODE>
__global__ void bucket_count(KeySrc src, int64_t n, uint32_t* counts) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        uint32_t key, val;
        load_item<MODE>(src, idx, key, val);
        red_add(&counts[key], 1u);
    }
}

template <int MODE>
__global__ void identity_perm(KeySrc src, int64_t n, uint32_t* perm) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        uint32_t key, val;
        load_item<MODE>(src, idx, key, val);
        perm[idx] = val;
    }
}

// Explicit map (hand-built or injective): validate and pack.
__global__ void explicit_prep(const int64_t* hash, const double* sign, int64_t n, int64_t B, uint32_t* keys,
                              uint32_t* vals, int* bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = hash[i];
        const double s = sign[i];
        if (h < 0 || h >= B || !(s == 1.0 || s == -1.0)) {
            atomicExch(bad, 1);
            keys[i] = 0;
            vals[i] = (uint32_t)i;
            continue;
        }
        keys[i] = (uint32_t)h;
        vals[i] = (uint32_t)i | (s < 0 ? kNegBit : 0u);
    }
}

// Materialize cs.hash / cs.sign from (perm, offsets): warp per bucket.
__global__ void fill_hash_sign_kernel(const uint32_t* perm, const uint32_t* offsets, int64_t B, int64_t* hash,
                                      double* sign) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (warp >= B) return;
    for (uint32_t p = offsets[warp] + lane; p < offsets[warp + 1]; p += 32) {
        const uint32_t e = perm[p];
        const uint32_t row = e & kRowMask;
        if (hash) hash[row] = warp;
        if (sign) sign[row] = (e & kNegBit) ? -1.0 : 1.0;
    }
}

// Tiny maps (n, B <= kTinyMax: distcheck's Monte-Carlo trials build hundreds of thousands of
// them) in ONE launch of one CTA instead of memset + count + scan + histogram + scan + scatter:
// bucket counts by shared-memory atomics, their scan by thread 0, and a stable placement where
// row i's rank inside its bucket is the number of earlier rows with the same bucket.  Same
// perm / offsets as the radix path (rows of a bucket in ascending order).
constexpr int kTinyMax = 1024;
template <int MODE>
__global__ void __launch_bounds__(kTinyMax) tiny_perm(KeySrc src, int n, int B, uint32_t* __restrict__ perm,
                                                       uint32_t* __restrict__ offsets) {
    __shared__ uint32_t s_key[kTinyMax];
    __shared__ uint32_t s_cnt[kTinyMax + 1];
    const int tid = threadIdx.x;
    for (int b = tid; b <= B; b += blockDim.x) s_cnt[b] = 0;
    __syncthreads();
    uint32_t key = 0, val = 0;
    if (tid < n) {
        load_item<MODE>(src, tid, key, val);
        s_key[tid] = key;
        atomicAdd(&s_cnt[key], 1u);
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t run = 0;
        for (int b = 0; b <= B; ++b) {
            const uint32_t c = s_cnt[b];
            s_cnt[b] = run;
            run += c;
        }
    }
    __syncthreads();
    for (int b = tid; b <= B; b += blockDim.x) offsets[b] = s_cnt[b];
    if (tid < n) {
        uint32_t rank = 0;
        for (int j = 0; j < tid; ++j) rank += s_key[j] == key;
        perm[s_cnt[key] + rank] = val;
    }
}

int key_bits(int64_t B) {
    int bits = 0;
    while (bits < 63 && ((int64_t)1 << bits) < B) ++bits;  // bucket values are < B
    return bits;
}

template <int MODE>
void build_perm(cgx_ctx* ctx, cgx_xform* xf, KeySrc src, cudaStream_t s) {
    const int64_t n = xf->n, B = xf->B;
    if (n <= kTinyMax && B <= kTinyMax) {
        tiny_perm<MODE><<<1, kTinyMax, 0, s>>>(src, (int)n, (int)B, xf->perm, xf->offsets);
        count_launch(ctx);
        check_launch("tiny_perm");
        return;
    }
    // bucket offsets
    uint32_t* counts = (uint32_t*)ctx->counts.get(sizeof(uint32_t) * (size_t)(B + 1));
    CGX_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * (size_t)(B + 1), s));
    const int grid = ctx->num_sms * 8;
    bucket_count<MODE><<<grid, 256, 0, s>>>(src, n, counts);
    count_launch(ctx);
    check_launch("bucket_count");
    exclusive_scan_u32(ctx, counts, xf->offsets, B + 1, s);

    const int bits = key_bits(B);
    const int passes = (bits + 7) / 8;
    if (passes == 0) {
        identity_perm<MODE><<<grid, 256, 0, s>>>(src, n, xf->perm);
        count_launch(ctx);
        check_launch("identity_perm");
        return;
    }
    const int64_t ntiles = (n + kTile - 1) / kTile;
    uint32_t* hist = (uint32_t*)ctx->sort_hist.get(sizeof(uint32_t) * (size_t)(256 * ntiles));
    uint32_t* kbuf[2] = {nullptr, nullptr};
    uint32_t* vbuf[2] = {nullptr, nullptr};
    if (passes > 1) {
        for (int i = 0; i < 2; ++i) {
            kbuf[i] = (uint32_t*)ctx->sort_k[i].get(sizeof(uint32_t) * (size_t)n);
            vbuf[i] = (uint32_t*)ctx->sort_v[i].get(sizeof(uint32_t) * (size_t)n);
        }
    }
    for (int p = 0; p < passes; ++p) {
        const bool last = p == passes - 1;
        uint32_t* kout = last ? nullptr : kbuf[p & 1];
        uint32_t* vout = last ? xf->perm : vbuf[p & 1];
        if (p == 0) {
            radix_hist<MODE><<<(unsigned)ntiles, kThreads, 0, s>>>(src, n, 0, ntiles, hist);
            count_launch(ctx);
            check_launch("radix_hist");
            exclusive_scan_u32(ctx, hist, hist, 256 * ntiles, s);
            radix_scatter<MODE><<<(unsigned)ntiles, kThreads, 0, s>>>(src, n, 0, ntiles, hist, kout, vout);
            count_launch(ctx);
            check_launch("radix_scatter");
        } else {
            KeySrc arr = src;
            arr.keys = kbuf[(p - 1) & 1];
            arr.vals = vbuf[(p - 1) & 1];
            radix_hist<1><<<(unsigned)ntiles, kThreads, 0, s>>>(arr, n, 8 * p, ntiles, hist);
            count_launch(ctx);
            check_launch("radix_hist");
            exclusive_scan_u32(ctx, hist, hist, 256 * ntiles, s);
            radix_scatter<1><<<(unsigned)ntiles, kThreads, 0, s>>>(arr, n, 8 * p, ntiles, hist, kout, vout);
            count_launch(ctx);
            check_launch("radix_scatter");
        }
    }
}

} // namespace

void build_perm_seeded(cgx_ctx* ctx, cgx_xform* xf, cudaStream_t s) {
    KeySrc src{nullptr, nullptr, xf->map_seed, FastMod((uint64_t)xf->B), xf->row0};
    build_perm<0>(ctx, xf, src, s);
}

void build_perm_explicit(cgx_ctx* ctx, cgx_xform* xf, const uint32_t* keys_dev, const uint32_t* vals_dev,
                         cudaStream_t s) {
    KeySrc src{keys_dev, vals_dev, 0, FastMod(1), 0};
    build_perm<1>(ctx, xf, src, s);
}

// Validate + pack an explicit (hash, sign) pair of device arrays; returns false if any
// entry is out of range.
bool prep_explicit(cgx_ctx* ctx, const int64_t* hash, const double* sign, int64_t n, int64_t B, uint32_t* keys,
                   uint32_t* vals, cudaStream_t s) {
    int* bad = (int*)ctx->sched.get(sizeof(int));
    CGX_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    explicit_prep<<<ctx->num_sms * 4, 256, 0, s>>>(hash, sign, n, B, keys, vals, bad);
    count_launch(ctx);
    check_launch("explicit_prep");
    int hbad = 0;
    CGX_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    CGX_CUDA(cudaStreamSynchronize(s));
    return hbad == 0;
}

namespace {
__global__ void bucket_shard_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ offsets,
                                    int64_t b0, int64_t nb, uint32_t o0, int64_t count, uint32_t* __restrict__ perm_l,
                                    uint32_t* __restrict__ offsets_l, uint32_t* __restrict__ grows) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride) {
        const uint32_t pe = perm[o0 + k];
        perm_l[k] = (uint32_t)k | (pe & kNegBit);
        grows[k] = pe & kRowMask;
    }
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= nb; j += stride)
        offsets_l[j] = offsets[b0 + j] - o0;
}
} // namespace

void launch_bucket_shard(cgx_ctx* ctx, const cgx_xform* full, int64_t b0, int64_t nb, uint32_t o0, cgx_xform* local,
                         cudaStream_t s) {
    bucket_shard_kernel<<<ctx->num_sms * 8, 256, 0, s>>>(full->perm, full->offsets, b0, nb, o0, local->n, local->perm,
                                                         local->offsets, local->grows);
    count_launch(ctx);
    check_launch("bucket_shard");
}

namespace {
__global__ void xform_rows_kernel(const uint32_t* __restrict__ grows, int64_t row0, int64_t n, int64_t* __restrict__ rows) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        rows[k] = grows ? (int64_t)grows[k] : row0 + k;
}
} // namespace

void launch_xform_rows(cgx_ctx* ctx, const cgx_xform* xf, int64_t* rows, cudaStream_t s) {
    xform_rows_kernel<<<ctx->num_sms * 4, 256, 0, s>>>(xf->grows, xf->row0, xf->n, rows);
    count_launch(ctx);
    check_launch("xform_rows");
}

void launch_fill_hash_sign(cgx_ctx* ctx, const cgx_xform* xf, int64_t* hash, double* sign, cudaStream_t s) {
    const int64_t threads = xf->B * 32;
    fill_hash_sign_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(xf->perm, xf->offsets, xf->B, hash, sign);
    count_launch(ctx);
    check_launch("fill_hash_sign");
}

} // namespace cgx
