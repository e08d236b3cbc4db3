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

// Wide rows (one row chunk spans the warp): the streaming form.  A warp owns G
// consecutive buckets, whose rows are one contiguous stretch of perm; it streams that
// stretch 32 entries at a time (the next 32 perm entries prefetched while the current
// rows are in flight), issues U row loads back to back (4 KB per warp in flight), and
// adds them in order, flushing the accumulator to SX whenever the stretch crosses a
// bucket boundary (bucket boundaries come from one coalesced load of the G+1 offsets).
// Per row and lane: one shuffle, one load, one convert, one add -- the warp's
// instruction stream no longer restarts per bucket, so rows keep flowing.
template <typename T, int V>
__global__ void __launch_bounds__(256, 4) sketch_dense_stream(const T* __restrict__ x, int64_t ld, int64_t d,
                                                           const uint32_t* __restrict__ perm,
                                                           const uint32_t* __restrict__ offsets, int64_t B,
                                                           int64_t nchunks, int G, double* __restrict__ sx) {
    constexpr int CW = 32 * V;
    constexpr int U = 64 / (V * (int)sizeof(T));  // rows per load batch: 2 KB per warp
    const unsigned lane = threadIdx.x & 31;
    const int64_t ngroups = (B + G - 1) / G;
    const int64_t task = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (task >= ngroups * nchunks) return;
    const int64_t bg = task / nchunks;
    const int64_t col0 = (task - bg * nchunks) * CW + (int64_t)lane * V;
    const bool colok = col0 < d;
    const int64_t b0 = bg * G;
    const int nb = (int)min((int64_t)G, B - b0);
    const uint32_t offk = (int)lane <= nb ? __ldg(offsets + b0 + lane) : 0u;
    const uint32_t P0 = __shfl_sync(0xffffffffu, offk, 0);
    const uint32_t P1 = __shfl_sync(0xffffffffu, offk, nb);
    double* out = sx + b0 * d + col0;
    int cur = 0;
    uint32_t nextb = __shfl_sync(0xffffffffu, offk, 1);
    double acc[V];
#pragma unroll
    for (int k = 0; k < V; ++k) acc[k] = 0.0;

    auto flush = [&]() {
        if (colok) {
#pragma unroll
            for (int k = 0; k < V; ++k) out[(int64_t)cur * d + k] = acc[k];
        }
#pragma unroll
        for (int k = 0; k < V; ++k) acc[k] = 0.0;
        ++cur;
        nextb = __shfl_sync(0xffffffffu, offk, min(cur + 1, 31));
    };

    uint32_t pe_next = P0 + lane < P1 ? __ldg(perm + P0 + lane) : 0u;
    for (uint32_t base = P0; base < P1; base += 32) {
        const uint32_t pe = pe_next;
        if (base + 32 + lane < P1) pe_next = __ldg(perm + base + 32 + lane);
        const int cnt = (int)min(32u, P1 - base);
        const uint32_t negmask = __ballot_sync(0xffffffffu, pe & kNegBit);  // bit t: row t negative
        // common case: a full chunk with no bucket boundary inside -> branch-free adds
        const bool fast = cnt == 32 && nextb >= base + 32;
#pragma unroll 1
        for (int s0 = 0; s0 < cnt; s0 += U) {
            T v[U][V];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t e = __shfl_sync(0xffffffffu, pe, (s0 + u) & 31);
                load_vec<T, V>(x + (int64_t)(e & kRowMask) * ld + (colok ? col0 : 0), v[u]);
            }
            const uint32_t nm = negmask >> s0;
            if (fast) {
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int k = 0; k < V; ++k) acc[k] += (double)flip_sign(v[u][k], (nm >> u) & 1u);
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (s0 + u < cnt) {
                        const uint32_t pos = base + s0 + u;
                        while (pos == nextb) flush();
#pragma unroll
                        for (int k = 0; k < V; ++k) acc[k] += (double)flip_sign(v[u][k], (nm >> u) & 1u);
                    }
                }
            }
        }
    }
    while (cur < nb) flush();
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

template <typename T, int V, int R>
void launch(cgx_ctx* ctx, const cgx_xform* xf, const T* x, int64_t ld, int64_t d, double* sx, int accumulate,
            cudaStream_t s) {
    constexpr int CW = (32 / R) * V;
    if (R == 1 && !accumulate) {
        // ~1K rows per warp task, at most 31 buckets (one offsets load)
        const int64_t rows_per_bucket = xf->n / xf->B + 1;
        int64_t G = 1024 / rows_per_bucket;
        G = G < 1 ? 1 : (G > 31 ? 31 : G);
        const int64_t nchunks = (d + CW - 1) / CW;
        const int64_t tasks = (xf->B + G - 1) / G * nchunks;
        const int64_t blocks = (tasks + 7) / 8;
        sketch_dense_stream<T, V><<<(unsigned)blocks, 256, 0, s>>>(x, ld, d, xf->perm, xf->offsets, xf->B, nchunks,
                                                                   (int)G, sx);
        count_launch(ctx);
        check_launch("sketch_dense_stream");
        return;
    }
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

} // namespace

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
