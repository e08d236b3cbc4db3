// sketch_dense.cu -- S.X for dense X: the bucket-ordered gather.
//
// Replaces countsketch_apply(map, DenseMatrix) (reference src/sketch.cpp:52-66), which
// scatters sign[i]*x(i,j) into out(hash[i], j) one column at a time, rows ascending.
//
// B200 design: one warp owns one (bucket, column-chunk) of the B x d output.  It walks
// the bucket's rows in ascending order from the transform's perm (construct.cu) and
// reads each row's chunk with coalesced (up to 128-bit) loads straight from HBM: the
// row is the unit of transfer, so every 32 B sector fetched is fully used.  Each lane
// keeps its columns' fp64 accumulators in registers and adds the rows in ascending order
// -- the reference's order -- so S.X is bit-identical to the reference (sign*x is exact,
// the accumulator starts at +0.0 like the reference's zero-filled DenseMatrix) and the
// result is deterministic: no atomics, no races, no reduction tree.
//
// Traffic per call: X once (n*d*sizeof(T)), perm once (4 B/row), S.X written once
// (B*d*8) -- the algorithmic bytes plus 4 B/row.  Loads of up to 16 rows are issued
// before their adds so each warp keeps ~2-4 KB in flight.
//
// X must be row-major here (row stride ld); column-major inputs are first transposed on
// the device (launch_transpose_x), because a gathered column-major row touches d
// separate sectors.
#include <cuda/barrier>

#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

template <typename T, int V>
struct Vec;
template <>
struct Vec<float, 1> { using type = float; };
template <>
struct Vec<float, 2> { using type = float2; };
template <>
struct Vec<float, 4> { using type = float4; };
template <>
struct Vec<double, 1> { using type = double; };
template <>
struct Vec<double, 2> { using type = double2; };

template <typename T, int V>
__device__ __forceinline__ void load_vec(const T* p, T (&out)[V]) {
    using VT = typename Vec<T, V>::type;
    VT v = __ldcs(reinterpret_cast<const VT*>(p));  // streamed once: evict-first
    const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int k = 0; k < V; ++k) out[k] = e[k];
}

template <typename T, int V>
__device__ __forceinline__ void load_smem_vec(const T* p, T (&out)[V]) {
    using VT = typename Vec<T, V>::type;
    VT v = *reinterpret_cast<const VT*>(p);
    const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int k = 0; k < V; ++k) out[k] = e[k];
}

__device__ __forceinline__ float negate_if(float v, uint32_t neg) {
    return __int_as_float(__float_as_int(v) ^ (int)(neg & kNegBit));
}
__device__ __forceinline__ double negate_if(double v, uint32_t neg) {
    return __longlong_as_double(__double_as_longlong(v) ^ ((long long)(neg & kNegBit) << 32));
}
// bit in {0,1}: exact negation by flipping the IEEE sign bit
__device__ __forceinline__ float flip_sign(float v, uint32_t bit) {
    return __int_as_float(__float_as_int(v) ^ (int)(bit << 31));
}
__device__ __forceinline__ double flip_sign(double v, uint32_t bit) {
    return __longlong_as_double(__double_as_longlong(v) ^ ((long long)bit << 63));
}

// R rows per warp-wide load step (L = 32/R lanes per row), V elements per lane.
template <typename T, int V, int R>
__global__ void __launch_bounds__(256) sketch_dense_kernel(const T* __restrict__ x, int64_t ld, int64_t d,
                                                           const uint32_t* __restrict__ perm,
                                                           const uint32_t* __restrict__ offsets, int64_t B,
                                                           int64_t nchunks, double* __restrict__ sx, int accumulate) {
    constexpr int L = 32 / R;
    constexpr int CW = L * V;          // columns per chunk
    constexpr int U = (16 / V) > (32 / R) ? (32 / R) : (16 / V);  // load steps in flight
    const unsigned lane = threadIdx.x & 31;
    const unsigned g = lane / L, sub = lane % L;
    const int64_t nitems = B * nchunks;
    for (int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; item < nitems;
         item += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b = item / nchunks;
        const int64_t col0 = (item - b * nchunks) * CW + (int64_t)sub * V;
        const bool colok = col0 < d;  // V | d is guaranteed by the host for V > 1
        double acc[V];
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = 0.0;
        if (accumulate && colok) {
#pragma unroll
            for (int k = 0; k < V; ++k) acc[k] = sx[b * d + col0 + k];
        }
        const uint32_t beg = offsets[b], end = offsets[b + 1];
        for (uint32_t base = beg; base < end; base += 32) {
            const int cnt = (int)min(32u, end - base);
            const uint32_t pe = (int)lane < cnt ? __ldg(perm + base + lane) : 0u;
            const int nsteps = (cnt + R - 1) / R;
            for (int s0 = 0; s0 < nsteps; s0 += U) {
                T v[U][V];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int t = (s0 + u) * R + (int)g;
                    const uint32_t e = __shfl_sync(0xffffffffu, pe, t & 31);
                    // unconditional load (padding entries read row 0, column 0) so that
                    // nothing consumes a loaded register before the whole batch is issued
                    load_vec<T, V>(x + (int64_t)(e & kRowMask) * ld + (colok ? col0 : 0), v[u]);
                }
                // signs applied only here, after every load of the batch is in flight
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int t = (s0 + u) * R + (int)g;
                    const uint32_t e = __shfl_sync(0xffffffffu, pe, t & 31);
                    const bool ok = colok && t < cnt;
#pragma unroll
                    for (int k = 0; k < V; ++k) v[u][k] = ok ? negate_if(v[u][k], e) : T(0);
                    if (R == 1) {
#pragma unroll
                        for (int k = 0; k < V; ++k) acc[k] += (double)v[u][k];
                    } else {
                        // ascending row order: group 0's row, then group 1's, ...
#pragma unroll
                        for (int gg = 0; gg < R; ++gg)
#pragma unroll
                            for (int k = 0; k < V; ++k)
                                acc[k] += (double)__shfl_sync(0xffffffffu, v[u][k], gg * L + sub);
                    }
                }
            }
        }
        if (g == 0 && colok) {
#pragma unroll
            for (int k = 0; k < V; ++k) sx[b * d + col0 + k] = acc[k];
        }
    }
}

// Wide rows (one row chunk spans the warp): the streaming form.  A warp owns nb <= 31
// consecutive buckets, whose rows are one contiguous stretch of perm; it streams that
// stretch 32 entries at a time (the next 32 perm entries prefetched while the current
// rows are in flight), issues U row loads back to back (2 KB per warp in flight), and
// adds them in order, handing the accumulator to `sink(i, acc)` whenever the stretch
// crosses the end of bucket b0+i (boundaries come from one coalesced load of the nb+1
// offsets).  Signs are applied only after a batch's loads are all issued (a consumer of
// a loaded register placed between the loads would serialize them), and a full chunk
// with no boundary inside takes a branch-free path: per row and lane one shuffle, one
// load, one sign flip, one convert, one add.
template <typename T, int V, int INFLIGHT = 2048, typename Sink>
__device__ __forceinline__ void stream_buckets(const T* __restrict__ x, int64_t ld, int64_t col0, bool colok,
                                               const uint32_t* __restrict__ perm,
                                               const uint32_t* __restrict__ offsets, int64_t b0, int nb,
                                               Sink&& sink) {
    constexpr int U = INFLIGHT / (32 * V * (int)sizeof(T));  // rows per load batch (INFLIGHT B per warp)
    const unsigned lane = threadIdx.x & 31;
    const uint32_t offk = (int)lane <= nb ? __ldg(offsets + b0 + lane) : 0u;
    const uint32_t P0 = __shfl_sync(0xffffffffu, offk, 0);
    const uint32_t P1 = __shfl_sync(0xffffffffu, offk, nb);
    int cur = 0;
    uint32_t nextb = __shfl_sync(0xffffffffu, offk, 1);
    double acc[V];
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = 0.0;

    auto flush = [&]() {
        sink(cur, acc);
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = 0.0;
        ++cur;
        nextb = __shfl_sync(0xffffffffu, offk, min(cur + 1, 31));
    };

    // per row: one shuffle, one IMAD.WIDE (row * row_bytes + column base), one load
    const char* xcol = reinterpret_cast<const char*>(x + (colok ? col0 : 0));
    const uint32_t row_bytes = (uint32_t)(ld * (int64_t)sizeof(T));  // host guarantees < 2^32
    uint32_t pe_next = P0 + lane < P1 ? __ldg(perm + P0 + lane) : 0u;
    for (uint32_t base = P0; base < P1; base += 32) {
        const uint32_t pe = pe_next;
        if (base + 32 + lane < P1) pe_next = __ldg(perm + base + 32 + lane);
        const int cnt = (int)min(32u, P1 - base);
        const uint32_t negmask = __ballot_sync(0xffffffffu, pe & kNegBit);  // bit t: row t negative
        const uint32_t prow = pe & kRowMask;
        // common case: a full chunk with no bucket boundary inside -> branch-free adds
        const bool fast = cnt == 32 && nextb >= base + 32;
#pragma unroll 1
        for (int s0 = 0; s0 < cnt; s0 += U) {
            T v[U][V];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                // padding rows read row 0 (a valid address) and are skipped when added
                const uint32_t r = __shfl_sync(0xffffffffu, prow, (s0 + u) & 31);
                load_vec<T, V>(reinterpret_cast<const T*>(xcol + (size_t)r * row_bytes), v[u]);
            }
            const uint32_t nm = negmask >> s0;
            if (fast) {
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int k = 0; k < V; ++k) {
                        acc[k] += (double)flip_sign(v[u][k], (nm >> u) & 1u);
                    }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (s0 + u < cnt) {
                        const uint32_t pos = base + s0 + u;
                        while (pos == nextb) flush();
#pragma unroll
                        for (int k = 0; k < V; ++k) {
                        acc[k] += (double)flip_sign(v[u][k], (nm >> u) & 1u);
                        }
                    }
                }
            }
        }
    }
    while (cur < nb) flush();
}

// stream_buckets with the row gather moved off the register file: each 32-row chunk of
// the warp's perm stretch is fetched by cp.async (16 B pieces, Q per row) into an
// S-slot ring in shared memory, S-1 chunks ahead of the adds, so every warp keeps
// (S-1) x 32 rows in flight continuously instead of a batch that drains before each
// round of adds.  The perm entries of a chunk are loaded one chunk before its copies are
// issued, the chunk's sign bits ride along in the ring (sneg), and the adds are the same
// ascending-order adds as stream_buckets -- S.X stays bit-identical.
// Requires: row pitch, column base and the warp's in-range columns in whole 16 B pieces
// (host-checked); x 16 B aligned.  `qv` = valid 16 B pieces per row of this chunk.
template <typename T, int V, int S, typename Sink>
__device__ __forceinline__ void stream_buckets_async(const T* __restrict__ x, int64_t ld, int64_t cw0, int qv,
                                                     const uint32_t* __restrict__ perm,
                                                     const uint32_t* __restrict__ offsets, int64_t b0, int nb,
                                                     T* ring, uint32_t* sneg, Sink&& sink) {
    constexpr int CW = 32 * V;
    constexpr int CB = CW * (int)sizeof(T);  // bytes per row chunk
    constexpr int Q = CB / 16;               // 16 B pieces per row chunk (power of two)
    const unsigned lane = threadIdx.x & 31;
    const uint32_t offk = (int)lane <= nb ? __ldg(offsets + b0 + lane) : 0u;
    const uint32_t P0 = __shfl_sync(0xffffffffu, offk, 0);
    const uint32_t P1 = __shfl_sync(0xffffffffu, offk, nb);
    int cur = 0;
    uint32_t nextb = __shfl_sync(0xffffffffu, offk, 1);
    double acc[V];
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = 0.0;
    auto flush = [&]() {
        sink(cur, acc);
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = 0.0;
        ++cur;
        nextb = __shfl_sync(0xffffffffu, offk, min(cur + 1, 31));
    };

    const char* xc = reinterpret_cast<const char*>(x + cw0);
    const uint32_t row_bytes = (uint32_t)(ld * (int64_t)sizeof(T));
    const uint32_t nchunk = (P1 - P0 + 31) / 32;
    auto perm_of = [&](uint32_t j) -> uint32_t {
        const uint32_t pos = P0 + j * 32 + lane;
        return (j < nchunk && pos < P1) ? __ldg(perm + pos) : kNegBit;  // kNegBit alone = padding
    };
    auto issue = [&](uint32_t j, uint32_t pe) {
        if (j < nchunk) {
            const int slot = (int)(j % S);
            char* dst = reinterpret_cast<char*>(ring) + (size_t)slot * 32 * CB;
            const uint32_t cnt = min(32u, P1 - (P0 + j * 32));
            const uint32_t neg = __ballot_sync(0xffffffffu, pe & kNegBit);
            if (lane == 0) sneg[slot] = neg;
            const uint32_t prow = pe & kRowMask;
#pragma unroll
            for (int k = 0; k < Q; ++k) {
                const int e = (int)lane + 32 * k;
                const int t = e / Q, q = e % Q;
                const uint32_t r = __shfl_sync(0xffffffffu, prow, t);
                if ((uint32_t)t < cnt && q < qv) cpa16(dst + t * CB + q * 16, xc + (size_t)r * row_bytes + q * 16);
            }
        }
        cpa_commit();  // one group per chunk slot, empty past the end: uniform group counting
    };

    uint32_t pe_next = perm_of(0);
#pragma unroll
    for (int j = 0; j < S - 1; ++j) {
        const uint32_t pe = pe_next;
        pe_next = perm_of(j + 1);
        issue(j, pe);
    }
    for (uint32_t j = 0; j < nchunk; ++j) {
        {   // keep S-1 chunks in flight: issue chunk j+S-1 into the slot freed at j-1
            const uint32_t pe = pe_next;
            pe_next = perm_of(j + S);
            issue(j + S - 1, pe);
        }
        cpa_wait<S - 1>();
        __syncwarp();
        const int slot = (int)(j % S);
        const T* src = ring + (size_t)slot * 32 * CW + lane * V;
        const uint32_t nm = sneg[slot];
        const uint32_t base = P0 + j * 32;
        const int cnt = (int)min(32u, P1 - base);
        if (cnt == 32 && nextb >= base + 32) {
#pragma unroll 8
            for (int t = 0; t < 32; ++t) {
                T v[V];
                load_smem_vec<T, V>(src + t * CW, v);
#pragma unroll
                for (int k = 0; k < V; ++k) acc[k] += (double)flip_sign(v[k], (nm >> t) & 1u);
            }
        } else {
            for (int t = 0; t < cnt; ++t) {
                while (base + t == nextb) flush();
                T v[V];
                load_smem_vec<T, V>(src + t * CW, v);
#pragma unroll
                for (int k = 0; k < V; ++k) acc[k] += (double)flip_sign(v[k], (nm >> t) & 1u);
            }
        }
        __syncwarp();  // every lane is done with this slot before it is refilled
    }
    cpa_wait<0>();
    while (cur < nb) flush();
}

// Persistent stream sketch over the cp.async ring (option async_stages = S): same tasks
// and output as sketch_dense_stream.  Shared memory: per warp S x 32 x CB ring + S masks.
// Tasks are handed out in bucket order: groups of G buckets for the first B1 buckets, then
// single buckets, so the last tasks -- which set the kernel's tail -- are short.
// SEG: the finished rows go to `segs` (the bucket-range owners' landing slots in peer memory,
// internal.h OutSegs) instead of sx -- the stores of the partial sketch are the transfer of
// the device group's reduce-scatter, spread over the whole kernel (group.cu, CGX_COMBINE_P2P).
template <typename T, int V, int S, bool SEG = false>
__global__ void __launch_bounds__(256) sketch_dense_async(const T* __restrict__ x, int64_t ld, int64_t d,
                                                          const uint32_t* __restrict__ perm,
                                                          const uint32_t* __restrict__ offsets, int64_t B,
                                                          int64_t nchunks, int G, int64_t B1, double* __restrict__ sx,
                                                          unsigned long long* __restrict__ next_task,
                                                          unsigned long long task_base,
                                                          const __grid_constant__ OutSegs segs) {
    pdl_trigger();  // stage 2 may be scheduled as these CTAs drain
    constexpr int CW = 32 * V;
    extern __shared__ __align__(16) unsigned char dsm[];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T* ring = reinterpret_cast<T*>(dsm) + (size_t)warp * S * 32 * CW;
    uint32_t* sneg = reinterpret_cast<uint32_t*>(reinterpret_cast<T*>(dsm) + (size_t)(blockDim.x >> 5) * S * 32 * CW) +
                     warp * S;
    const int64_t ng0 = B1 / G;  // B1 is a multiple of G
    const int64_t ngroups = ng0 + (B - B1);
    const int64_t ntasks = ngroups * nchunks;
    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(next_task, 1ull) - task_base;
        const int64_t task = (int64_t)__shfl_sync(0xffffffffu, t, 0);
        if (task >= ntasks) break;
        const int64_t bg = task / nchunks;
        const int64_t cw0 = (task - bg * nchunks) * CW;
        const int64_t col0 = cw0 + (int64_t)lane * V;
        const bool colok = col0 < d;
        const int qv = (int)min((int64_t)(CW * sizeof(T) / 16), (d - cw0) * (int64_t)sizeof(T) / 16);
        const int64_t b0 = bg < ng0 ? bg * G : B1 + (bg - ng0);
        const int nb = bg < ng0 ? G : 1;
        double* out = sx + b0 * d + col0;
        stream_buckets_async<T, V, S>(x, ld, cw0, qv, perm, offsets, b0, nb, ring, sneg,
                                      [&](int i, const double (&acc)[V]) {
                                          if (colok) {
                                              double* o = out + (int64_t)i * d;
                                              if (SEG) {
                                                  const uint32_t b = (uint32_t)(b0 + i), q = b / segs.per;
                                                  o = segs.base[q] + (int64_t)(b - q * segs.per) * d + col0;
                                              }
#pragma unroll
                                              for (int k = 0; k < V; ++k) o[k] = acc[k];
                                          }
                                      });
    }
}

template <typename T, int V>
__global__ void __launch_bounds__(256, 3) sketch_dense_stream(const T* __restrict__ x, int64_t ld, int64_t d,
                                                              const uint32_t* __restrict__ perm,
                                                              const uint32_t* __restrict__ offsets, int64_t B,
                                                              int64_t nchunks, int G, double* __restrict__ sx,
                                                              unsigned* __restrict__ next_task) {
    // Persistent warps pull (bucket group, column chunk) tasks from a counter: no warp
    // idles while a slow sibling holds its CTA slot.  Every bucket is still summed by one
    // warp in ascending row order, so S.X does not depend on the assignment.
    constexpr int CW = 32 * V;
    const unsigned lane = threadIdx.x & 31;
    const int64_t ngroups = (B + G - 1) / G;
    const int64_t ntasks = ngroups * nchunks;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(next_task, 1u);
        const int64_t task = __shfl_sync(0xffffffffu, t, 0);
        if (task >= ntasks) break;
        const int64_t bg = task / nchunks;
        const int64_t col0 = (task - bg * nchunks) * CW + (int64_t)lane * V;
        const bool colok = col0 < d;
        const int64_t b0 = bg * G;
        const int nb = (int)min((int64_t)G, B - b0);
        double* out = sx + b0 * d + col0;
        stream_buckets<T, V, 4096>(x, ld, col0, colok, perm, offsets, b0, nb, [&](int i, const double (&acc)[V]) {
            if (colok) {
#pragma unroll
                for (int k = 0; k < V; ++k) out[(int64_t)i * d + k] = acc[k];
            }
        });
    }
}

// countgauss_apply in one pass (dense, wide rows): sketch + G generation + G.(S.X).
// A persistent CTA of 8 warps takes bucket tiles of 8*Gw consecutive buckets (static
// round-robin, so the summation grouping -- and Z -- is deterministic).  Each warp
// streams Gw buckets (stream_buckets) into the tile's S.X slab in shared memory and
// generates the m x Gw slab of G for its buckets (SplitMix64 + Acklam + Halley, the
// reference's quantile) -- FP64 work that hides under the other warps' HBM traffic.
// After a CTA barrier, warp w adds G[rows_w, tile] . SX[tile, :] into its own Z rows
// (RW = ceil(m/8) rows x V columns per lane, kept in registers across tiles) in a fixed
// order.  At the end each CTA writes its m x d partial; reduce_splits sums the partials
// in CTA order.  G and S.X never touch HBM; X is read exactly once.
template <typename T, int V, int RW>
__global__ void __launch_bounds__(256, 4) countgauss_dense_fused(const T* __restrict__ x, int64_t ld, int64_t d,
                                                                 const uint32_t* __restrict__ perm,
                                                                 const uint32_t* __restrict__ offsets, int64_t B,
                                                                 int64_t m, uint64_t g_seed,
                                                                 const double* __restrict__ g_explicit, int Gw,
                                                                 double* __restrict__ zpart) {
    constexpr int CW = 32 * V;
    extern __shared__ double fsm[];
    __shared__ cuda::barrier<cuda::thread_scope_block> full[2], freed[2];
    const int TB = 8 * Gw;                           // buckets per tile
    const int slab_sz = TB * CW + (int)m * TB;       // S.X [TB][CW] then G [m][TB]
    double* sZ = fsm + 2 * slab_sz;                  // [m][CW]: Z rows, each owned by one warp
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t col0 = (int64_t)lane * V;
    const bool colok = col0 < d;
    const int64_t ntiles = (B + TB - 1) / TB;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            init(&full[i], blockDim.x);
            init(&freed[i], blockDim.x);
        }
    }
    for (int e = threadIdx.x; e < (int)m * CW; e += blockDim.x) sZ[e] = 0.0;
    __syncthreads();
    cuda::barrier<cuda::thread_scope_block>::arrival_token tok_full[2], tok_freed[2];

    // Z rows of this warp += G[rows, tile] . SX[tile, my columns]   (fixed order)
    auto consume = [&](int buf) {
        const double* sSX = fsm + buf * slab_sz;
        const double* sG = sSX + TB * CW;
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) {
            const int r = (int)warp * RW + rr;
            if (r < m) {
                const double* grow = sG + (int64_t)r * TB;
                double zr[V];
#pragma unroll
                for (int k = 0; k < V; ++k) zr[k] = sZ[r * CW + lane * V + k];
                for (int s = 0; s < TB; ++s) {
                    const double gv = grow[s];
#pragma unroll
                    for (int k = 0; k < V; ++k) zr[k] = fma(gv, sSX[s * CW + lane * V + k], zr[k]);
                }
#pragma unroll
                for (int k = 0; k < V; ++k) sZ[r * CW + lane * V + k] = zr[k];
            }
        }
    };

    int64_t k = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int buf = (int)(k & 1);
        if (k >= 2) freed[buf].wait(std::move(tok_freed[buf]));  // slab buf consumed (tile k-2)
        double* sSX = fsm + buf * slab_sz;
        double* sG = sSX + TB * CW;
        const int64_t tb0 = tile * TB;
        const int64_t b0 = tb0 + (int64_t)warp * Gw;
        const int nb = b0 < B ? (int)min((int64_t)Gw, B - b0) : 0;
        // S.X rows of this warp's buckets -> shared slab (zero rows for absent buckets)
        double* slab = sSX + (int64_t)warp * Gw * CW + lane * V;
        if (nb > 0) {
            stream_buckets<T, V>(x, ld, col0, colok, perm, offsets, b0, nb, [&](int i, const double (&acc)[V]) {
#pragma unroll
                for (int k = 0; k < V; ++k) slab[i * CW + k] = colok ? acc[k] : 0.0;
            });
        }
        for (int i = nb; i < Gw; ++i)
#pragma unroll
            for (int k = 0; k < V; ++k) slab[i * CW + k] = 0.0;
        // G[:, b0 .. b0+Gw) -> sG[r][warp*Gw + i]  (zero for absent buckets / rows)
        for (int e = lane; e < m * Gw; e += 32) {
            const int i = e / (int)m, r = e - i * (int)m;
            const int64_t b = b0 + i;
            double g = 0.0;
            if (i < nb) g = g_explicit ? g_explicit[b * m + r] : gauss_entry(g_seed, (uint64_t)m, (uint64_t)r, (uint64_t)b);
            sG[(int64_t)r * TB + warp * Gw + i] = g;
        }
        tok_full[buf] = full[buf].arrive();
        // Deferred by one tile: the previous slab is (nearly always) complete by now, so
        // warps rarely wait here and never idle at a full CTA barrier.
        if (k >= 1) {
            const int pb = buf ^ 1;
            full[pb].wait(std::move(tok_full[pb]));
            consume(pb);
            tok_freed[pb] = freed[pb].arrive();
        }
    }
    if (k >= 1) {
        const int lb = (int)((k - 1) & 1);
        full[lb].wait(std::move(tok_full[lb]));
        consume(lb);
    }
    __syncwarp();
    // partial Z of this CTA, column-major m x d (each warp writes the rows it owns)
    double* zp = zpart + (int64_t)blockIdx.x * m * d;
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
        const int r = (int)warp * RW + rr;
        if (r < m && colok) {
#pragma unroll
            for (int k = 0; k < V; ++k) zp[(col0 + k) * m + r] = sZ[r * CW + lane * V + k];
        }
    }
}

template <typename E>
__global__ void transpose_kernel(const E* __restrict__ src, int64_t rows, int64_t cols, int64_t lds,
                                 E* __restrict__ dst, int64_t ldd) {
    // src: rows x cols row-major (stride lds) -> dst: cols x rows row-major (stride ldd)
    __shared__ E tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = r0 + k, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[k][threadIdx.x] = src[r * lds + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t c = c0 + k, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][k];
    }
}

template <typename E>
void transpose(cgx_ctx* ctx, const E* src, int64_t rows, int64_t cols, int64_t lds, E* dst, int64_t ldd,
               cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return;
    const int64_t gx = (cols + 31) / 32, gy = (rows + 31) / 32;
    for (int64_t y0 = 0; y0 < gy; y0 += 65535) {
        const int64_t ny = gy - y0 < 65535 ? gy - y0 : 65535;
        transpose_kernel<E><<<dim3((unsigned)gx, (unsigned)ny), dim3(32, 8), 0, s>>>(
            src + y0 * 32 * lds, rows - y0 * 32, cols, lds, dst + y0 * 32, ldd);
        count_launch(ctx);
        check_launch("transpose");
    }
}

// The cp.async ring kernel applies: 16 B pieces all the way (and a row pitch below 4 GB).
inline bool async_ring_ok(int S, const void* x, size_t es, int64_t ld, int64_t d) {
    return S >= 2 && (uintptr_t)x % 16 == 0 && (ld * es) % 16 == 0 && (d * es) % 16 == 0;
}
// Paths that cannot store into a device group's landing slots: capi.cu's SegsFallback has
// cleared ctx->out_segs for them (sketch_dense_fuses_segs said so).
inline void no_segs(const cgx_ctx* ctx) {
    if (ctx->out_segs) fail(CGX_ECUDA, "internal: this sketch kernel cannot write peer landing slots");
}

template <typename T, int V, int R>
void launch(cgx_ctx* ctx, const cgx_xform* xf, const T* x, int64_t ld, int64_t d, double* sx, int accumulate,
            cudaStream_t s) {
    constexpr int CW = (32 / R) * V;
    if (R == 1 && !accumulate && ld * (int64_t)sizeof(T) < ((int64_t)1 << 32)) {
        // ~1K rows per warp task, at most 31 buckets (one offsets load)
        const int64_t rows_per_bucket = xf->n / xf->B + 1;
        int64_t G = rows_per_task(ctx, xf->n) / rows_per_bucket;
        G = G < 1 ? 1 : (G > 31 ? 31 : G);
        const int64_t nchunks = (d + CW - 1) / CW;
        const int64_t tasks = (xf->B + G - 1) / G * nchunks;
        const int S = (int)ctx->opt_async;
        const size_t CB = (size_t)CW * sizeof(T);
        if (async_ring_ok(S, x, sizeof(T), ld, d)) {
            // cp.async ring: W warps per CTA, each with S x 32 rows x CB of shared memory
            const size_t per_warp = (size_t)S * 32 * CB + (size_t)S * 4;
            int W = (int)((200 * 1024) / per_warp);
            W = W > 8 ? 8 : (W < 1 ? 1 : W);
            const size_t smem = per_warp * W;
            const OutSegs* segs = ctx->out_segs;  // (only with S == 2: sketch_dense_fuses_segs)
            auto kern = segs     ? sketch_dense_async<T, V, 2, true>
                        : S == 2 ? sketch_dense_async<T, V, 2>
                        : S == 3 ? sketch_dense_async<T, V, 3>
                                 : sketch_dense_async<T, V, 4>;
            CGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            int per_sm = 0;
            CGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * W, smem));
            int64_t blocks = (int64_t)ctx->num_sms * (per_sm < 1 ? 1 : per_sm);
            if (blocks > (tasks + W - 1) / W) blocks = (tasks + W - 1) / W;
            // tail: the last ~2 single-bucket tasks per warp (option tail_tasks, per warp)
            const int64_t tail = ctx->opt_tail_tasks * blocks * W / nchunks;
            int64_t B1 = xf->B - tail;
            B1 = B1 < 0 ? 0 : B1 / G * G;
            const unsigned long long base = take_tasks(ctx, (B1 / G + xf->B - B1) * nchunks, blocks * W);
            kern<<<(unsigned)blocks, 32 * W, smem, s>>>(x, ld, d, xf->perm, xf->offsets, xf->B, nchunks, (int)G, B1,
                                                        sx, ctx->task_ctr, base, segs ? *segs : OutSegs{});
            count_launch(ctx);
            tasks_launched(ctx, s);
            check_launch("sketch_dense_async");
            return;
        }
        no_segs(ctx);
        auto kern = sketch_dense_stream<T, V>;
        int per_sm = 0;
        CGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
        int64_t blocks = (int64_t)ctx->num_sms * (per_sm < 1 ? 1 : per_sm) * ctx->opt_grid_waves;
        if (blocks > (tasks + 7) / 8) blocks = (tasks + 7) / 8;
        unsigned* ctr = (unsigned*)ctx->sched.get(sizeof(unsigned));
        CGX_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), s));
        kern<<<(unsigned)blocks, 256, 0, s>>>(x, ld, d, xf->perm, xf->offsets, xf->B, nchunks, (int)G, sx, ctr);
        count_launch(ctx);
        check_launch("sketch_dense_stream");
        return;
    }
    no_segs(ctx);
    const int64_t nchunks = (d + CW - 1) / CW;
    const int64_t warps = xf->B * nchunks;
    int64_t blocks = (warps + 7) / 8;
    const int64_t cap = (int64_t)ctx->num_sms * 64;
    if (blocks > cap) blocks = cap;
    sketch_dense_kernel<T, V, R><<<(unsigned)blocks, 256, 0, s>>>(x, ld, d, xf->perm, xf->offsets, xf->B, nchunks,
                                                                  sx, accumulate);
    count_launch(ctx);
    check_launch("sketch_dense");
}

template <typename T>
void dispatch(cgx_ctx* ctx, const cgx_xform* xf, const T* x, int64_t ld, int64_t d, double* sx, int accumulate,
              cudaStream_t s) {
    auto aligned = [&](int v) {
        return ((uintptr_t)x % (sizeof(T) * v)) == 0 && ld % v == 0 && d % v == 0;
    };
    if (d >= 32) {
        if (sizeof(T) == 4 && d >= 128 && aligned(4)) return launch<T, (sizeof(T) == 4 ? 4 : 2), 1>(ctx, xf, x, ld, d, sx, accumulate, s);
        if (d >= 64 && aligned(2)) return launch<T, 2, 1>(ctx, xf, x, ld, d, sx, accumulate, s);
        return launch<T, 1, 1>(ctx, xf, x, ld, d, sx, accumulate, s);
    }
    if (d > 16) return launch<T, 1, 1>(ctx, xf, x, ld, d, sx, accumulate, s);
    if (d > 8) return launch<T, 1, 2>(ctx, xf, x, ld, d, sx, accumulate, s);
    if (d > 4) return launch<T, 1, 4>(ctx, xf, x, ld, d, sx, accumulate, s);
    if (d > 2) return launch<T, 1, 8>(ctx, xf, x, ld, d, sx, accumulate, s);
    if (d > 1) return launch<T, 1, 16>(ctx, xf, x, ld, d, sx, accumulate, s);
    return launch<T, 1, 32>(ctx, xf, x, ld, d, sx, accumulate, s);
}

// Warp-specialized one-pass countgauss_apply.  CTA = 8 sketch warps + 4 math warps.
//  * sketch warps only stream X (4 KB of row loads in flight per warp) and deposit each
//    bucket's S.X row into a double-buffered shared slab; they never stop to compute,
//    so the CTA's HBM request stream stays full;
//  * math warps generate the m x TB slab of G for the tile ahead of time (G does not
//    depend on X), wait for the tile's S.X slab, and accumulate Z += G_tile . SX_tile
//    into registers (MR rows x V columns per thread), fixed order -> deterministic.
// Hand-off: mbarrier `full[buf]` (256 sketch arrivals) and `freed[buf]` (128 math
// arrivals) per slab; a named barrier orders the math warps' G slab reuse.
// S > 0: the sketch warps gather through an S-slot cp.async ring (stream_buckets_async)
// placed after the two slabs in dynamic shared memory, instead of register batches.
template <typename T, int V, int MR, int S>
__global__ void __launch_bounds__(384, 2) countgauss_dense_ws(const T* __restrict__ x, int64_t ld, int64_t d,
                                                              const uint32_t* __restrict__ perm,
                                                              const uint32_t* __restrict__ offsets, int64_t B,
                                                              int64_t m, uint64_t g_seed,
                                                              const double* __restrict__ g_explicit, int Gw,
                                                              double* __restrict__ zpart) {
    constexpr int CW = 32 * V;
    extern __shared__ double fsm[];
    __shared__ uint64_t full[2], freed[2];
    const int TB = 8 * Gw;
    const int slab_sz = TB * CW + (int)m * TB;  // S.X [TB][CW], then G [m][TB]
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (B + TB - 1) / TB;
    if (tid == 0) {
        mbar_init(&full[0], 256);
        mbar_init(&full[1], 256);
        mbar_init(&freed[0], 128);
        mbar_init(&freed[1], 128);
    }
    __syncthreads();

    if (warp < 8) {  // ---------------------------------------------------------- sketch
        const int64_t col0 = (int64_t)lane * V;
        const bool colok = col0 < d;
        int64_t k = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
            const int buf = (int)(k & 1);
            if (k >= 2) mbar_wait(&freed[buf], (unsigned)(((k - 2) >> 1) & 1));
            double* slab = fsm + buf * slab_sz + (int64_t)warp * Gw * CW + lane * V;
            const int64_t b0 = tile * TB + (int64_t)warp * Gw;
            const int nb = b0 < B ? (int)min((int64_t)Gw, B - b0) : 0;
            auto sink = [&](int i, const double (&acc)[V]) {
#pragma unroll
                for (int q = 0; q < V; ++q) slab[i * CW + q] = colok ? acc[q] : 0.0;
            };
            if (nb > 0) {
                if constexpr (S > 0) {
                    T* ring = reinterpret_cast<T*>(fsm + 2 * slab_sz) + (size_t)warp * S * 32 * CW;
                    uint32_t* sneg = reinterpret_cast<uint32_t*>(reinterpret_cast<T*>(fsm + 2 * slab_sz) +
                                                                 (size_t)8 * S * 32 * CW) + warp * S;
                    const int qv = (int)min((int64_t)(CW * sizeof(T) / 16), d * (int64_t)sizeof(T) / 16);
                    stream_buckets_async<T, V, S>(x, ld, 0, qv, perm, offsets, b0, nb, ring, sneg, sink);
                } else {
                    stream_buckets<T, V, 4096>(x, ld, col0, colok, perm, offsets, b0, nb, sink);
                }
            }
            for (int i = nb; i < Gw; ++i)
#pragma unroll
                for (int q = 0; q < V; ++q) slab[i * CW + q] = 0.0;
            mbar_arrive(&full[buf]);
        }
        return;
    }
    // ------------------------------------------------------------------------------ math
    const unsigned mt = tid - 256, mw = mt >> 5;  // 128 threads, 4 warps
    double z[MR][V];
#pragma unroll
    for (int q = 0; q < MR; ++q)
#pragma unroll
        for (int c = 0; c < V; ++c) z[q][c] = 0.0;
    int64_t k = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int buf = (int)(k & 1);
        const double* sSX = fsm + buf * slab_sz;
        double* sG = fsm + buf * slab_sz + TB * CW;
        const int64_t tb0 = tile * TB;
        for (int e = (int)mt; e < (int)m * TB; e += 128) {
            const int s = e / (int)m, r = e - s * (int)m;
            const int64_t b = tb0 + s;
            double g = 0.0;
            if (b < B) g = g_explicit ? g_explicit[b * m + r] : gauss_entry(g_seed, (uint64_t)m, (uint64_t)r, (uint64_t)b);
            sG[r * TB + s] = g;
        }
        named_sync(1, 128);
        mbar_wait(&full[buf], (unsigned)((k >> 1) & 1));
        for (int s = 0; s < TB; ++s) {
            double sx[V];
#pragma unroll
            for (int c = 0; c < V; ++c) sx[c] = sSX[s * CW + lane * V + c];
#pragma unroll
            for (int q = 0; q < MR; ++q) {
                const int r = (int)mw + 4 * q;
                if (r < m) {
                    const double g = sG[r * TB + s];
#pragma unroll
                    for (int c = 0; c < V; ++c) z[q][c] = fma(g, sx[c], z[q][c]);
                }
            }
        }
        mbar_arrive(&freed[buf]);
    }
    double* zp = zpart + (int64_t)blockIdx.x * m * d;
#pragma unroll
    for (int q = 0; q < MR; ++q) {
        const int r = (int)mw + 4 * q;
#pragma unroll
        for (int c = 0; c < V; ++c) {
            const int64_t col = (int64_t)lane * V + c;
            if (r < m && col < d) zp[col * m + r] = z[q][c];
        }
    }
}


template <typename T, int V, int MR>
void launch_ws(cgx_ctx* ctx, const cgx_xform* xf, const T* x, int64_t ld, int64_t d, double* z, cudaStream_t s) {
    constexpr int CW = 32 * V;
    const int64_t B = xf->B, m = xf->m;
    int S = (int)ctx->opt_async;
    if (S > 3 || (uintptr_t)x % 16 != 0 || (ld * sizeof(T)) % 16 != 0 || (d * sizeof(T)) % 16 != 0 ||
        8 * (size_t)S * 32 * CW * sizeof(T) > 128 * 1024)
        S = 0;
    auto kern = S == 2 ? countgauss_dense_ws<T, V, MR, 2>
                       : (S == 3 ? countgauss_dense_ws<T, V, MR, 3> : countgauss_dense_ws<T, V, MR, 0>);
    int64_t Gw = B / (8 * 32 * (int64_t)ctx->num_sms * 2);
    Gw = Gw < 1 ? 1 : (Gw > 8 ? 8 : Gw);
    if (ctx->opt_ws_gw > 0) Gw = ctx->opt_ws_gw;
    const int64_t TB = 8 * Gw;
    const int64_t ntiles = (B + TB - 1) / TB;
    const size_t ring = S > 0 ? 8 * ((size_t)S * 32 * CW * sizeof(T) + (size_t)S * 4) : 0;
    const size_t smem = sizeof(double) * (size_t)(2 * (TB * CW + m * TB)) + ring;
    CGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 384, smem));
    if (per_sm < 1) per_sm = 1;
    const int64_t grid_cap = (int64_t)ctx->num_sms * per_sm;
    const int64_t grid = ntiles < grid_cap ? ntiles : grid_cap;
    double* zpart = (double*)ctx->zpart.get(sizeof(double) * (size_t)(grid * m * d));
    kern<<<(unsigned)grid, 384, smem, s>>>(x, ld, d, xf->perm, xf->offsets, B, m, xf->g_seed,
                                           xf->g_dev, (int)Gw, zpart);
    count_launch(ctx);
    check_launch("countgauss_dense_ws");
    launch_reduce_splits(ctx, zpart, grid, m * d, z, s);
}

template <typename T, int V, int RW>
void launch_fused(cgx_ctx* ctx, const cgx_xform* xf, const T* x, int64_t ld, int64_t d, double* z, cudaStream_t s) {
    constexpr int CW = 32 * V;
    const int64_t B = xf->B, m = xf->m;
    auto kern = countgauss_dense_fused<T, V, RW>;
    // persistent grid: every CTA resident (occupancy-limited), >= ~8 tiles per CTA
    int64_t Gw = B / (64 * (int64_t)ctx->num_sms * 4);
    Gw = Gw < 1 ? 1 : (Gw > 8 ? 8 : Gw);
    const int64_t TB = 8 * Gw;
    const int64_t ntiles = (B + TB - 1) / TB;
    const size_t smem = sizeof(double) * (size_t)(2 * (TB * CW + m * TB) + m * CW);
    CGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    if (per_sm < 1) per_sm = 1;
    const int64_t grid_cap = (int64_t)ctx->num_sms * per_sm;
    const int64_t grid = ntiles < grid_cap ? ntiles : grid_cap;
    double* zpart = (double*)ctx->zpart.get(sizeof(double) * (size_t)(grid * m * d));
    kern<<<(unsigned)grid, 256, smem, s>>>(x, ld, d, xf->perm, xf->offsets, B, m, xf->g_seed,
                                           xf->g_dev, (int)Gw, zpart);
    count_launch(ctx);
    check_launch("countgauss_dense_fused");
    launch_reduce_splits(ctx, zpart, grid, m * d, z, s);
}

template <typename T, int V>
bool fused_rw(cgx_ctx* ctx, const cgx_xform* xf, const T* x, int64_t ld, int64_t d, double* z, cudaStream_t s) {
    const int64_t m = xf->m;
    if (ctx->fuse_mode == 2) {  // warp-specialized
        if (m <= 4) return launch_ws<T, V, 1>(ctx, xf, x, ld, d, z, s), true;
        if (m <= 8) return launch_ws<T, V, 2>(ctx, xf, x, ld, d, z, s), true;
        if (m <= 16) return launch_ws<T, V, 4>(ctx, xf, x, ld, d, z, s), true;
        if constexpr (V <= 2) {
            if (m <= 32) return launch_ws<T, V, 8>(ctx, xf, x, ld, d, z, s), true;
        }
        if constexpr (V == 1) {
            if (m <= 64) return launch_ws<T, V, 16>(ctx, xf, x, ld, d, z, s), true;
        }
    }
    if (m <= 8) return launch_fused<T, V, 1>(ctx, xf, x, ld, d, z, s), true;
    if (m <= 16) return launch_fused<T, V, 2>(ctx, xf, x, ld, d, z, s), true;
    if (m <= 32) return launch_fused<T, V, 4>(ctx, xf, x, ld, d, z, s), true;
    if (V <= 2 && m <= 64) return launch_fused<T, V, 8>(ctx, xf, x, ld, d, z, s), true;
    if (V == 1 && m <= 128) return launch_fused<T, V, 16>(ctx, xf, x, ld, d, z, s), true;
    return false;
}

template <typename T>
bool fused_dispatch(cgx_ctx* ctx, const cgx_xform* xf, const T* x, int64_t ld, int64_t d, double* z, cudaStream_t s) {
    auto aligned = [&](int v) { return ((uintptr_t)x % (sizeof(T) * v)) == 0 && ld % v == 0 && d % v == 0; };
    if (d < 17) return false;  // narrow rows: several rows per warp load, two-stage path
    if (ld * (int64_t)sizeof(T) >= ((int64_t)1 << 32)) return false;  // 32-bit row pitch in stream_buckets
    if (d <= 32) return fused_rw<T, 1>(ctx, xf, x, ld, d, z, s);
    if (d <= 64 && aligned(2)) return fused_rw<T, 2>(ctx, xf, x, ld, d, z, s);
    if (sizeof(T) == 4 && d <= 128 && aligned(4)) return fused_rw<T, (sizeof(T) == 4 ? 4 : 2)>(ctx, xf, x, ld, d, z, s);
    return false;
}

} // namespace

bool launch_countgauss_dense_fused(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int64_t ld,
                                   int64_t d, double* z, cudaStream_t s) {
    if (dtype == CGX_F32) return fused_dispatch<float>(ctx, xf, (const float*)x, ld, d, z, s);
    return fused_dispatch<double>(ctx, xf, (const double*)x, ld, d, z, s);
}

// Mirrors dispatch() + launch(): R == 1 (d > 16), the async ring with its default depth.
bool sketch_dense_fuses_segs(const cgx_ctx* ctx, const void* x, int dtype, int64_t ld, int64_t d) {
    const size_t es = dtype == CGX_F32 ? 4 : 8;
    return d > 16 && ld * (int64_t)es < ((int64_t)1 << 32) && ctx->opt_async == 2 && async_ring_ok(2, x, es, ld, d);
}

void launch_sketch_dense(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int64_t ld, int64_t n,
                         int64_t d, double* sx, cudaStream_t s) {
    (void)n;
    if (dtype == CGX_F32)
        dispatch<float>(ctx, xf, (const float*)x, ld, d, sx, 0, s);
    else
        dispatch<double>(ctx, xf, (const double*)x, ld, d, sx, 0, s);
}

void launch_transpose_x(cgx_ctx* ctx, const void* x, int dtype, int64_t ld, int64_t n, int64_t d, void* dst,
                        cudaStream_t s) {
    // column-major n x d (stride ld) == row-major d x n; transpose into row-major n x d.
    if (dtype == CGX_F32)
        transpose<float>(ctx, (const float*)x, d, n, ld, (float*)dst, d, s);
    else
        transpose<double>(ctx, (const double*)x, d, n, ld, (double*)dst, d, s);
}

void launch_transpose_sx(cgx_ctx* ctx, const double* src, int64_t B, int64_t d, double* dst, cudaStream_t s) {
    transpose<double>(ctx, src, B, d, d, dst, B, s);
}

} // namespace cgx
