// extremes.cu -- per-row argmax / argmin of Z for CountGauss NMF anchor selection.
//
// Replaces select_extremes (reference src/nmf.cpp:99-118): per row r of the m x d
// projected matrix, the column of the maximum and of the minimum with strict compares
// (ties resolve to the lowest column index) and whether either extreme is attained more
// than once (tie_rows).  NaN entries never win and never tie, except that a NaN in
// column 0 pins both extremes to column 0 -- exactly what the reference's sequential
// scan does.  One warp per row; lanes scan strided columns in ascending order and the
// (value, index, hits) triples are merged with lowest-index tie breaking.
#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

struct Ext {
    double v;
    int64_t a;
    int64_t h;  // hits; 0 = empty
};

template <bool MAX>
__device__ __forceinline__ Ext merge(Ext x, Ext y) {
    if (y.h == 0) return x;
    if (x.h == 0) return y;
    const bool y_better = MAX ? (y.v > x.v) : (y.v < x.v);
    const bool x_better = MAX ? (x.v > y.v) : (x.v < y.v);
    if (y_better) return y;
    if (x_better) return x;
    return Ext{x.v, x.a < y.a ? x.a : y.a, x.h + y.h};
}

template <bool MAX>
__device__ __forceinline__ Ext warp_merge(Ext e) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Ext y;
        y.v = __shfl_xor_sync(0xffffffffu, e.v, o);
        y.a = __shfl_xor_sync(0xffffffffu, e.a, o);
        y.h = __shfl_xor_sync(0xffffffffu, e.h, o);
        e = merge<MAX>(e, y);
    }
    return e;
}

__global__ void select_extremes_kernel(const double* __restrict__ z, int64_t m, int64_t d, int64_t* amax,
                                       int64_t* amin, int64_t* tie) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (r >= m) return;
    if (isnan(z[r])) {  // reference: vmax = vmin = NaN and nothing compares greater/equal
        if (lane == 0) {
            amax[r] = 0;
            amin[r] = 0;
            tie[r] = 0;
        }
        return;
    }
    Ext mx{0.0, 0, 0}, mn{0.0, 0, 0};
    for (int64_t j = lane; j < d; j += 32) {
        const double v = z[j * m + r];
        if (isnan(v)) continue;
        mx = merge<true>(mx, Ext{v, j, 1});
        mn = merge<false>(mn, Ext{v, j, 1});
    }
    mx = warp_merge<true>(mx);
    mn = warp_merge<false>(mn);
    if (lane == 0) {
        amax[r] = mx.a;
        amin[r] = mn.a;
        tie[r] = (mx.h > 1 || mn.h > 1) ? 1 : 0;
    }
}

} // namespace

void launch_select_extremes(cgx_ctx* ctx, const double* z, int64_t m, int64_t d, int64_t* amax, int64_t* amin,
                            int64_t* tie_flags, cudaStream_t s) {
    const int64_t threads = m * 32;
    select_extremes_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(z, m, d, amax, amin, tie_flags);
    count_launch(ctx);
    check_launch("select_extremes");
}

} // namespace cgx
