// sketch_csr.cu -- S.X for CSR X: bucket-ordered gather with an on-chip accumulator.
//
// Replaces countsketch_apply(map, SparseMatrix) (reference src/sketch.cpp:68-113).  The
// reference runs a serial row loop (every BASELINE CSR config takes that branch) or,
// when B*d <= 2^16, 8192-row chunks whose partial buffers are reduced in ascending
// chunk order.  Both orders are reproduced here bit-for-bit.
//
// B200 design: one warp owns bucket b's output row SX[b, 0..d) as an fp64 accumulator in
// shared memory (or in the output row itself when d is too large for shared memory).
// It walks the bucket's rows in ascending order (perm, construct.cu) 32 at a time:
//   1. lane k fetches row k's [rowptr[r], rowptr[r+1]) -- one random 16 B read each;
//   2. a warp prefix sum flattens the 32 rows' nonzeros into one item range, which the
//      warp then reads in coalesced 32-item waves (consecutive items of a row are
//      consecutive in memory), several waves in flight at once;
//   3. each wave is applied in item order: items that hit the same column (only
//      possible across rows) are serialized by lane rank via __match_any_sync, so
//      every (bucket, column) sums its rows in ascending row order -- the reference's.
// No atomics, deterministic, bit-identical to the reference.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <climits>

namespace cgx {
namespace {

constexpr int kWaves = 4;  // item waves loaded before they are applied
#ifndef CGX_CSR_MINB
#define CGX_CSR_MINB 4  // 4 CTAs/SM: c5 sketch 17.9 -> 15.3 ms (tools/sweep_csr.sh)
#endif
#ifndef CGX_CSR_KW
#define CGX_CSR_KW 6  // item waves in flight per warp: c5 12.95 -> 12.82 ms against 4 (8: 14.0, spills)
#endif

// Random short reads: a global load that does not allocate in L1 (the gathered rows are
// never re-read by this SM) and asks L2 for a 64 B fetch.  Without the L2::64B hint every
// L1 miss is promoted to a 128 B L2/DRAM fetch: a random 4 B load then costs 128 B of DRAM
// traffic, with it 64 B (tools/microbench/sector_fetch.cu; 64 B is the smallest hint).
#ifndef CGX_CSR_FETCH
#define CGX_CSR_FETCH "64B"
#endif
template <typename T>
__device__ __forceinline__ T ld_na(const T* p) {
    if constexpr (sizeof(T) == 8) {
        unsigned long long v;
        asm volatile("ld.global.L1::no_allocate.L2::" CGX_CSR_FETCH ".b64 %0, [%1];" : "=l"(v) : "l"(p));
        T out;
        memcpy(&out, &v, 8);
        return out;
    } else {
        unsigned v;
        asm volatile("ld.global.L1::no_allocate.L2::" CGX_CSR_FETCH ".b32 %0, [%1];" : "=r"(v) : "l"(p));
        T out;
        memcpy(&out, &v, 4);
        return out;
    }
}

// v with its sign bit flipped when neg is 1 (exact: -v), before the widening to fp64
__device__ __forceinline__ float flip_sign(float v, unsigned neg) { return __int_as_float(__float_as_int(v) ^ (int)(neg << 31)); }
__device__ __forceinline__ double flip_sign(double v, unsigned neg) {
    return __longlong_as_double(__double_as_longlong(v) ^ ((long long)neg << 63));
}

template <typename TV, typename TI, bool CHUNKED>
__global__ void __launch_bounds__(256) sketch_csr_kernel(const int64_t* __restrict__ rowptr,
                                                         const TI* __restrict__ cols, const TV* __restrict__ vals,
                                                         const uint32_t* __restrict__ perm,
                                                         const uint32_t* __restrict__ offsets, int64_t B, int64_t d,
                                                         double* __restrict__ sx, double* __restrict__ gpart,
                                                         int64_t chunk_rows, int use_smem, int cbits) {
    extern __shared__ double smem[];
    __shared__ int s_incl[8][32];
    __shared__ int64_t s_beg[8][32];
    __shared__ uint32_t s_pe[8][32];
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int warps_per_cta = blockDim.x >> 5;
    double* my = smem + (size_t)wid * d * (CHUNKED ? 2 : 1);

    for (int64_t b = (int64_t)blockIdx.x * warps_per_cta + wid; b < B; b += (int64_t)gridDim.x * warps_per_cta) {
        double* acc = use_smem ? my : sx + b * d;
        double* part = CHUNKED ? (use_smem ? my + d : gpart + b * d) : nullptr;
        for (int64_t j = lane; j < d; j += 32) {
            acc[j] = 0.0;
            if (CHUNKED) part[j] = 0.0;
        }
        double* tgt = CHUNKED ? part : acc;
        int64_t cur_chunk = -1;
        __syncwarp();
        const uint32_t beg = offsets[b], end = offsets[b + 1];
        for (uint32_t base = beg; base < end; base += 32) {
            const int cnt = (int)min(32u, end - base);
            uint32_t pe = 0;
            int64_t rb = 0, re = 0;
            if ((int)lane < cnt) {
                pe = __ldg(perm + base + lane);
                const int64_t row = pe & kRowMask;
                rb = ld_na(rowptr + row);
                re = ld_na(rowptr + row + 1);
            }
            const int incl = warp_incl_scan((int)(re - rb), lane);
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            s_incl[wid][lane] = incl;
            s_beg[wid][lane] = rb;
            s_pe[wid][lane] = pe;
            __syncwarp();
            for (int q0 = 0; q0 < total; q0 += 32 * kWaves) {
                TI c[kWaves];
                TV v[kWaves];
                int kk[kWaves];
#pragma unroll
                for (int w = 0; w < kWaves; ++w) {
                    const int q = q0 + w * 32 + (int)lane;
                    kk[w] = -1;
                    if (q < total) {
                        int lo = 0;  // first k with incl[k] > q
#pragma unroll
                        for (int step = 16; step > 0; step >>= 1)
                            if (s_incl[wid][lo + step - 1] <= q) lo += step;
                        const int start = lo ? s_incl[wid][lo - 1] : 0;
                        const int64_t pos = s_beg[wid][lo] + (q - start);
                        c[w] = ld_na(cols + pos);
                        v[w] = ld_na(vals + pos);
                        kk[w] = lo;
                    }
                }
#pragma unroll
                for (int w = 0; w < kWaves; ++w) {
                    const bool valid = kk[w] >= 0;
                    if (!__any_sync(0xffffffffu, valid)) break;
                    const uint32_t pe_k = valid ? s_pe[wid][kk[w]] : 0u;
                    double val = valid ? (double)v[w] : 0.0;
                    if (pe_k & kNegBit) val = -val;
                    const int64_t col = valid ? (int64_t)c[w] : -1 - (int64_t)lane;
                    bool todo = valid;
                    if (CHUNKED) {
                        const int64_t ch = valid ? (int64_t)(pe_k & kRowMask) / chunk_rows : LLONG_MAX;
                        while (__any_sync(0xffffffffu, todo)) {
                            const int64_t cmin = __reduce_min_sync(0xffffffffu, todo ? (unsigned)ch : UINT_MAX);
                            if (cmin != cur_chunk) {
                                if (cur_chunk >= 0) {
                                    for (int64_t j = lane; j < d; j += 32) {
                                        acc[j] += part[j];
                                        part[j] = 0.0;
                                    }
                                }
                                cur_chunk = cmin;
                                __syncwarp();
                            }
                            const bool mine = todo && ch == cmin;
                            const int64_t key = mine ? col : -1 - (int64_t)lane;
                            const unsigned peers = __match_any_sync(0xffffffffu, key);
                            const unsigned rank = __popc(peers & lt_mask);
                            const unsigned maxr = __reduce_max_sync(0xffffffffu, rank);
                            for (unsigned r = 0; r <= maxr; ++r) {
                                if (mine && rank == r) tgt[key] += val;
                                __syncwarp();
                            }
                            if (mine) todo = false;
                        }
                    } else {
                        // same-column lanes: ballot matching for narrow column ranges
                        // (MATCH.ANY is slow on 32 mostly-distinct values)
                        const unsigned peers =
                            cbits <= 12 ? match_any_bits(valid ? (uint32_t)col : 1u << (cbits - 1), cbits)
                                        : __match_any_sync(0xffffffffu, col);
                        const unsigned rank = __popc(peers & lt_mask);
                        const unsigned maxr = __reduce_max_sync(0xffffffffu, valid ? rank : 0u);
                        for (unsigned r = 0; r <= maxr; ++r) {
                            if (valid && rank == r) acc[col] += val;
                            __syncwarp();
                        }
                    }
                }
            }
            __syncwarp();
        }
        if (CHUNKED && cur_chunk >= 0) {
            for (int64_t j = lane; j < d; j += 32) acc[j] += part[j];
            __syncwarp();
        }
        if (use_smem) {
            for (int64_t j = lane; j < d; j += 32) sx[b * d + j] = acc[j];
        }
        __syncwarp();
    }
}

// Lean form of the serial-order gather for the common case (reference serial branch,
// accumulator in shared memory): the same bucket-ordered, row-ascending walk with far
// fewer instructions per nonzero, since at ~0.5 us of DRAM latency per row group the
// kernel was issue-bound (c5: 205 warp instructions per 32 nonzeros).
//  * item -> row: the rows starting inside each 32-item wave come from one OR-reduction
//    of start bits, and a per-group table maps (nonzero-row rank) -> lane; no search;
//  * same-column lanes: each lane stamps its lane id into a byte tag per column; if every
//    lane reads its own stamp back the wave's columns are distinct (the usual case) and
//    all adds go at once, otherwise the ballot matcher orders them by lane;
//  * the next row group's perm entries and row offsets are loaded while the current group
//    is processed, and a group's item loads are issued kW waves at a time.
// Adds happen in exactly the serial kernel's order, so S.X is bit-identical to it.
//  * warps are persistent and pull tasks of G consecutive buckets from a counter, the last
//    ones single buckets (B1 = buckets in G-groups), so no SM idles while a late CTA wave
//    finishes.
//  * SEG: a bucket's finished row goes to its owner's landing slot in peer memory (`segs`,
//    internal.h OutSegs) instead of sx: the device group's reduce-scatter transfer, spread
//    over the whole kernel (group.cu, CGX_COMBINE_P2P).
template <typename TV, typename TI, bool SEG = false>
__global__ void __launch_bounds__(256, CGX_CSR_MINB) sketch_csr_lean(const int64_t* __restrict__ rowptr, const TI* __restrict__ cols,
                                                       const TV* __restrict__ vals, const uint32_t* __restrict__ perm,
                                                       const uint32_t* __restrict__ offsets, int64_t B, int64_t d,
                                                       double* __restrict__ sx, int G, int64_t B1,
                                                       unsigned long long* __restrict__ next_task,
                                                       unsigned long long task_base,
                                                       unsigned long long* __restrict__ colmax,
                                                       const __grid_constant__ OutSegs segs) {
    constexpr int kW = CGX_CSR_KW;
    pdl_trigger();  // stage 2 may be scheduled as these CTAs drain
    extern __shared__ double smem[];
    __shared__ uint8_t s_tbl[8][32];
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u, le = lt | (1u << lane);
    const int warps_per_cta = blockDim.x >> 5;
    double* acc = smem + (size_t)wid * d;
    uint8_t* tag = reinterpret_cast<uint8_t*>(smem + (size_t)warps_per_cta * d) + (size_t)wid * d;
    uint8_t* tbl = s_tbl[wid];
    // optional: per-column max |S.X| for the tensor-core stage 2's scales (ozgemm.cu), kept
    // per CTA in shared memory and folded into `colmax` once at exit
    unsigned long long* cmax = reinterpret_cast<unsigned long long*>(
        smem + (((size_t)warps_per_cta * d * 9 + 7) / 8));
    if (colmax) {
        for (int64_t j = threadIdx.x; j < d; j += blockDim.x) cmax[j] = 0;
        __syncthreads();
    }
    const int64_t ng0 = B1 / G;
    const int64_t ntasks = ng0 + (B - B1);
    for (;;) {
      unsigned long long tk = 0;
      if (lane == 0) tk = atomicAdd(next_task, 1ull) - task_base;
      const int64_t task = (int64_t)__shfl_sync(0xffffffffu, tk, 0);
      if (task >= ntasks) break;
      const int64_t tb0 = task < ng0 ? task * G : B1 + (task - ng0);
      const int64_t tb1 = task < ng0 ? tb0 + G : tb0 + 1;
      for (int64_t b = tb0; b < tb1; ++b) {
        for (int64_t j = lane; j < d; j += 32) acc[j] = 0.0;
        __syncwarp();
        const uint32_t beg = offsets[b], end = offsets[b + 1];
        // row group g = perm[base .. base+32): lane k holds row k's (sign, begin, length)
        uint32_t npe = 0;
        int64_t nrb = 0, nre = 0;
        auto fetch = [&](uint32_t base) {
            npe = 0;
            nrb = nre = 0;
            if (base + lane < end) {
                npe = __ldg(perm + base + lane);
                const int64_t row = npe & kRowMask;
                nrb = ld_na(rowptr + row);
                nre = ld_na(rowptr + row + 1);
            }
        };
        fetch(beg);
        for (uint32_t base = beg; base < end; base += 32) {
            const uint32_t pe = npe;
            const int64_t rb = nrb;
            const int len = (int)(nre - nrb);
            fetch(base + 32);  // next group, in flight while this one is processed
            const int incl = warp_incl_scan(len, lane);
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            const int excl = incl - len;
            // item q of the group is nonzero (q - excl_k) of row k: position off_k + q
            const int64_t off = rb - excl;
            const unsigned negm = __ballot_sync(0xffffffffu, pe & kNegBit);
            const unsigned nz = __ballot_sync(0xffffffffu, len > 0);
            if (len > 0) tbl[__popc(nz & lt)] = (uint8_t)lane;
            __syncwarp();
            int kbase = 0;  // nonzero rows started in earlier waves
            for (int q0 = 0; q0 < total; q0 += 32 * kW) {
                TI c[kW];
                TV v[kW];
                unsigned neg[kW];
#pragma unroll
                for (int u = 0; u < kW; ++u) {
                    const int w0 = q0 + u * 32;
                    const bool starts_here = len > 0 && (unsigned)(excl - w0) < 32u;
                    const unsigned st = __reduce_or_sync(0xffffffffu, starts_here ? 1u << (excl - w0) : 0u);
                    const int r = kbase + __popc(st & le) - 1;
                    kbase += __popc(st);
                    const int j = tbl[r & 31];
                    const int64_t offj = __shfl_sync(0xffffffffu, off, j);
                    neg[u] = (negm >> j) & 1u;
                    const int q = w0 + (int)lane;
                    c[u] = 0;
                    v[u] = TV(0);
                    if (q < total) {
                        c[u] = ld_na(cols + (offj + q));
                        v[u] = ld_na(vals + (offj + q));
                    }
                }
#pragma unroll
                for (int u = 0; u < kW; ++u) {
                    const int w0 = q0 + u * 32;
                    if (w0 >= total) break;
                    const bool ok = w0 + (int)lane < total;
                    const uint32_t col = ok ? (uint32_t)c[u] : 0u;
                    const double x = (double)flip_sign(v[u], neg[u]);
                    if (ok) tag[col] = (uint8_t)lane;
                    __syncwarp();
                    // rep: the lane whose stamp survived in this column's tag (one per column)
                    const unsigned rep = ok ? tag[col] : lane;
                    if (__all_sync(0xffffffffu, rep == lane)) {
                        if (ok) acc[col] += x;
                    } else {  // a column twice in the wave: lane (= row) order per column
                        // Lanes sharing a column share its rep, a 5-bit lane id, so the groups
                        // come from 5 ballots whatever d is; each group then sums as a chain
                        // in lane order through shuffles, ((acc + x0) + x1) + ..., and its last
                        // lane stores -- the serial order, one shared-memory round trip.
                        const unsigned peers = match_any_bits(rep, 5);
                        const unsigned before = peers & lt;
                        const unsigned rank = __popc(before);
                        const int pred = 31 - __clz(before);  // previous lane of the group
                        const unsigned maxr = __reduce_max_sync(0xffffffffu, rank);
                        double s = x;
                        if (ok && rank == 0) s = acc[col] + x;
                        for (unsigned rr = 1; rr <= maxr; ++rr) {
                            const double t = __shfl_sync(0xffffffffu, s, pred & 31);
                            if (rank == rr) s = t + x;
                        }
                        if (ok && (peers & ~le) == 0) acc[col] = s;
                    }
                    __syncwarp();
                }
            }
        }
        __syncwarp();
        double* orow = sx + b * d;
        if (SEG) {
            const uint32_t q = (uint32_t)b / segs.per;
            orow = segs.base[q] + (int64_t)((uint32_t)b - q * segs.per) * d;
        }
        for (int64_t j = lane; j < d; j += 32) {
            orow[j] = acc[j];
            if (colmax) {  // (a plain read first: after the first buckets the max rarely moves)
                const unsigned long long u = (unsigned long long)__double_as_longlong(fabs(acc[j]));
                if (u > *(volatile unsigned long long*)&cmax[j]) atomicMax(&cmax[j], u);
            }
        }
        __syncwarp();
      }
    }
    if (colmax) {
        __syncthreads();
        for (int64_t j = threadIdx.x; j < d; j += blockDim.x)
            if (cmax[j]) atomicMax(&colmax[j], cmax[j]);
    }
}

// Boundaries of the (bucket, chunk) runs of perm: virtual bucket v = b * nc + c holds the
// rows of bucket b with row / chunk_rows == c (perm is sorted by (bucket, row)).
__global__ void chunk_offsets_kernel(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ offsets, int64_t B,
                                     int64_t nc, int64_t chunk_rows, uint32_t* __restrict__ voff) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v > B * nc) return;
    if (v == B * nc) {
        voff[v] = offsets[B];
        return;
    }
    const int64_t b = v / nc, c = v - b * nc;
    uint32_t lo = offsets[b], hi = offsets[b + 1];  // first entry with row >= c * chunk_rows
    const int64_t r = c * chunk_rows;
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if ((int64_t)(perm[mid] & kRowMask) < r) lo = mid + 1; else hi = mid;
    }
    voff[v] = lo;
}

// out[b][j] = ((0 + part[b][0][j]) + part[b][1][j]) + ...: the reference's ascending-chunk
// reduction of the per-chunk partial buffers (sketch.cpp:106-111).
__global__ void chunk_reduce_kernel(const double* __restrict__ part, int64_t B, int64_t nc, int64_t d,
                                    double* __restrict__ out) {
    const int64_t total = B * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / d, j = e - b * d;
        const double* p = part + b * nc * d + j;
        double acc = 0.0;
        for (int64_t c = 0; c < nc; ++c) acc += p[c * d];
        out[e] = acc;
    }
}

// The lean gather over `nb_total` buckets delimited by `offs`, into sx (row-major nb_total x d).
// `colmax_ok`: sx is the final S.X, so the column maxima for the tensor-core stage 2 may be
// folded in.  False when shared memory cannot hold a warp's accumulator.
template <typename TV, typename TI>
bool launch_lean(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const TI* cols, const TV* vals, int64_t d,
                 int64_t nb_total, const uint32_t* offs, double* sx, bool colmax_ok, cudaStream_t s) {
    const size_t per_warp_l = (sizeof(double) + 1) * (size_t)d;
    int wl = (int)((96 * 1024) / per_warp_l);
    wl = wl > 8 ? 8 : wl;
    if (wl < 1) return false;
    const OutSegs* segs = ctx->out_segs;  // (a partial sketch: its column maxima are not S.X's)
    if (segs && !colmax_ok) fail(CGX_ECUDA, "internal: the chunked CSR sketch cannot write peer landing slots");
    unsigned long long* colmax = nullptr;
    if (colmax_ok && !segs && oz_stage2_applies(ctx, xf, d)) {
        colmax = (unsigned long long*)ctx->oz_b.get(sizeof(unsigned long long) * (size_t)d);
        CGX_CUDA(cudaMemsetAsync(colmax, 0, sizeof(unsigned long long) * (size_t)d, s));
        ctx->oz_colmax_for = sx;
        ctx->oz_colmax_d = d;
    }
    const size_t sm = (per_warp_l * wl + 7) / 8 * 8 + (colmax ? sizeof(unsigned long long) * (size_t)d : 8);
    auto lk = segs ? sketch_csr_lean<TV, TI, true> : sketch_csr_lean<TV, TI>;
    CGX_CUDA(cudaFuncSetAttribute(lk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = 0;
    CGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lk, wl * 32, sm));
    int64_t nb = (nb_total + wl - 1) / wl;
    const int64_t sms = ctx->opt_gather_sms > 0 && ctx->opt_gather_sms < ctx->num_sms ? ctx->opt_gather_sms : ctx->num_sms;
    const int64_t cap = sms * (per_sm < 1 ? 1 : per_sm);  // persistent: one wave
    if (nb > cap) nb = cap;
    // tasks of ~rows_per_task rows (whole buckets), single buckets for the last tail_tasks
    // per warp
    const int64_t rows_per_bucket = xf->n / nb_total + 1;
    int64_t G = rows_per_task(ctx, xf->n) / rows_per_bucket;
    G = G < 1 ? 1 : (G > 64 ? 64 : G);
    int64_t B1 = nb_total - ctx->opt_tail_tasks * nb * wl;
    B1 = B1 < 0 ? 0 : B1 / G * G;
    const unsigned long long base = take_tasks(ctx, B1 / G + nb_total - B1, nb * wl);
    lk<<<(unsigned)nb, wl * 32, sm, s>>>(rowptr, cols, vals, xf->perm, offs, nb_total, d, sx, (int)G, B1,
                                         ctx->task_ctr, base, colmax, segs ? *segs : OutSegs{});
    count_launch(ctx);
    tasks_launched(ctx, s);
    check_launch("sketch_csr_lean");
    return true;
}

template <typename TV, typename TI, bool CHUNKED>
void launch(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const TI* cols, const TV* vals, int64_t d,
            double* sx, int64_t chunk_rows, cudaStream_t s) {
    const size_t per_warp = sizeof(double) * (size_t)d * (CHUNKED ? 2 : 1);
    const size_t budget = 96 * 1024;
    int warps = (int)(budget / per_warp);
    if (warps > 8) warps = 8;
    int use_smem = warps >= 1;
    double* gpart = nullptr;
    size_t smem = 0;
    if (use_smem) {
        smem = per_warp * warps;
    } else {
        warps = 8;
        CGX_CUDA(cudaMemsetAsync(sx, 0, sizeof(double) * (size_t)(xf->B * d), s));
        if (CHUNKED) gpart = (double*)ctx->zpart.get(sizeof(double) * (size_t)(xf->B * d));
    }
    if (d <= 8192) {
        if (!CHUNKED) {
            if (launch_lean<TV, TI>(ctx, xf, rowptr, cols, vals, d, xf->B, xf->offsets, sx, true, s)) return;
        } else {
            // The reference's chunked branch (sketch.cpp:74-111) computes one partial per
            // 8192-row chunk and sums the partials in chunk order.  The partials are
            // independent, so each (bucket, chunk) pair is a bucket of its own here: its rows
            // are a contiguous run of the bucket's (bucket, row)-sorted perm entries, found by
            // binary search.  The lean gather then runs over B * n_chunks virtual buckets
            // (parallel even when B is tiny -- e.g. B = 80 in acceptance criterion 11, where
            // one warp per bucket left the GPU idle), and a second kernel sums each output
            // entry's partials in chunk order, starting from +0.0, as the reference does.
            const int64_t nc = (xf->n + chunk_rows - 1) / chunk_rows;
            const int64_t vb = xf->B * nc;
            uint32_t* voff = (uint32_t*)ctx->counts.get(sizeof(uint32_t) * (size_t)(vb + 1));
            double* part = (double*)ctx->zpart.get(sizeof(double) * (size_t)(vb * d));
            chunk_offsets_kernel<<<(unsigned)((vb + 1 + 255) / 256), 256, 0, s>>>(xf->perm, xf->offsets, xf->B, nc,
                                                                                 chunk_rows, voff);
            count_launch(ctx);
            check_launch("chunk_offsets");
            if (launch_lean<TV, TI>(ctx, xf, rowptr, cols, vals, d, vb, voff, part, false, s)) {
                const int64_t total = xf->B * d;
                chunk_reduce_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)ctx->num_sms * 8), 256,
                                      0, s>>>(part, xf->B, nc, d, sx);
                count_launch(ctx);
                check_launch("chunk_reduce");
                return;
            }
        }
    }
    if (ctx->out_segs) fail(CGX_ECUDA, "internal: this CSR sketch kernel cannot write peer landing slots");
    auto kern = sketch_csr_kernel<TV, TI, CHUNKED>;
    if (smem > 40 * 1024) CGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int64_t blocks = (xf->B + warps - 1) / warps;
    const int64_t cap = (int64_t)ctx->num_sms * 32;
    if (blocks > cap) blocks = cap;
    int cbits = 1;  // bits of a column index plus one sentinel value
    while (((int64_t)1 << (cbits - 1)) < d) ++cbits;
    kern<<<(unsigned)blocks, warps * 32, smem, s>>>(rowptr, cols, vals, xf->perm, xf->offsets, xf->B, d, sx, gpart,
                                                   chunk_rows, use_smem, cbits);
    count_launch(ctx);
    check_launch("sketch_csr");
}

template <typename TV, typename TI>
void dispatch_chunk(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols, const void* vals,
                    int64_t d, double* sx, int64_t chunk_rows, cudaStream_t s) {
    if (chunk_rows > 0)
        launch<TV, TI, true>(ctx, xf, rowptr, (const TI*)cols, (const TV*)vals, d, sx, chunk_rows, s);
    else
        launch<TV, TI, false>(ctx, xf, rowptr, (const TI*)cols, (const TV*)vals, d, sx, 0, s);
}

} // namespace

// Mirrors launch<>(): the lean gather, unchunked, with a warp's accumulator in shared memory.
bool sketch_csr_fuses_segs(const cgx_ctx* ctx, int64_t d, int64_t chunk_rows) {
    (void)ctx;
    return chunk_rows == 0 && d <= 8192;
}

void launch_sketch_csr(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols, int idx_type,
                       const void* vals, int dtype, int64_t n, int64_t d, double* sx, int64_t chunk_rows,
                       cudaStream_t s) {
    (void)n;
    if (dtype == CGX_F32) {
        if (idx_type == CGX_I32)
            dispatch_chunk<float, int32_t>(ctx, xf, rowptr, cols, vals, d, sx, chunk_rows, s);
        else
            dispatch_chunk<float, int64_t>(ctx, xf, rowptr, cols, vals, d, sx, chunk_rows, s);
    } else {
        if (idx_type == CGX_I32)
            dispatch_chunk<double, int32_t>(ctx, xf, rowptr, cols, vals, d, sx, chunk_rows, s);
        else
            dispatch_chunk<double, int64_t>(ctx, xf, rowptr, cols, vals, d, sx, chunk_rows, s);
    }
}

} // namespace cgx
