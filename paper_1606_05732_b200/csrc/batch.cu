// batch.cu -- batched tiny sketches: the Monte-Carlo inner loop of distcheck
// (reference src/distcheck.cpp:107-113, moment_suite):
//
//   for t in trials:  SeededRng r(mix64(master, t));
//                     map = countsketch_new(B, n, r);       // sketch.cpp:12-28
//                     su  = countsketch_apply(map, U);      // sketch.cpp:52-66
//                     M   = gram(su);                       // matrix.cpp:149-165
//
// The reference runs one OpenMP thread per trial over thousands of trials of a small U.
// Here one warp owns one trial and all trials of a batch go in one launch:
//  * 32 rows at a time, lane k computes row k's bucket and sign from the trial's map seed
//    (the SplitMix64 index map, no hash array), then the rows are added one by one, in
//    ascending order, with the lanes spread over U's columns -- each su(b, j) sums its rows
//    in the reference's order, so su is bit-identical;
//  * gram: lanes take (i <= j) column pairs and sum su(l, i) * su(l, j) over l ascending
//    with separate multiply and add (__dmul_rn / __dadd_rn; the reference is built without
//    FMA), then mirror -- bit-identical as well;
//  * su lives in shared memory when B*d fits (12 KB per warp), else in global scratch.
#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

constexpr int kWarps = 4;
constexpr int kSmemDoubles = 1536;  // per warp

__global__ void __launch_bounds__(32 * kWarps) batch_sketch_gram(uint64_t master, int64_t t0, int64_t trials, int64_t B,
                                                                 FastMod mod, const double* __restrict__ u, int64_t ld,
                                                                 int64_t n, int64_t d, double* __restrict__ su_out,
                                                                 double* __restrict__ gram_out, int su_in_smem) {
    extern __shared__ double bsm[];
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t t = (int64_t)blockIdx.x * kWarps + wid;
    if (t >= trials) return;
    const int64_t bd = B * d;
    double* su = su_in_smem ? bsm + (size_t)wid * kSmemDoubles : su_out + t * bd;  // col-major B x d
    for (int64_t e = lane; e < bd; e += 32) su[e] = 0.0;
    __syncwarp();
    const uint64_t trial_seed = mix64(master, (uint64_t)(t0 + t));
    const uint64_t map_seed = rng_draw(trial_seed, 0);  // map.seed = r.next_u64()
    for (int64_t i0 = 0; i0 < n; i0 += 32) {
        const int64_t i = i0 + lane;
        uint32_t h = 0, neg = 0;
        if (i < n) {
            h = cs_bucket(map_seed, (uint64_t)i, mod);
            neg = cs_negative(map_seed, (uint64_t)i);
        }
        const int cnt = (int)min((int64_t)32, n - i0);
        for (int k = 0; k < cnt; ++k) {
            const uint32_t hk = __shfl_sync(0xffffffffu, h, k);
            const uint32_t nk = __shfl_sync(0xffffffffu, neg, k);
            for (int64_t j = lane; j < d; j += 32) {
                const double x = u[j * ld + i0 + k];
                su[j * B + hk] += nk ? -x : x;
            }
        }
    }
    __syncwarp();
    if (su_in_smem && su_out)
        for (int64_t e = lane; e < bd; e += 32) su_out[t * bd + e] = su[e];
    if (gram_out) {
        double* g = gram_out + t * d * d;  // col-major d x d
        const int64_t pairs = d * (d + 1) / 2;
        for (int64_t p = lane; p < pairs; p += 32) {
            int64_t j = 0;  // pair p -> (ii <= j), enumerated column by column
            while ((j + 1) * (j + 2) / 2 <= p) ++j;
            const int64_t ii = p - j * (j + 1) / 2;
            const double* ai = su + ii * B;
            const double* aj = su + j * B;
            double s = 0.0;
            for (int64_t l = 0; l < B; ++l) s = __dadd_rn(s, __dmul_rn(ai[l], aj[l]));
            g[j * d + ii] = s;
            g[ii * d + j] = s;
        }
    }
}

} // namespace

void launch_batch_sketch_gram(cgx_ctx* ctx, uint64_t master, int64_t t0, int64_t trials, int64_t B, const double* u,
                              int64_t ld, int64_t n, int64_t d, double* su_out, double* gram_out, cudaStream_t s) {
    const bool in_smem = B * d <= kSmemDoubles;
    double* su = su_out;
    if (!in_smem && !su) su = (double*)ctx->xstage.get(sizeof(double) * (size_t)(trials * B * d));
    const size_t smem = in_smem ? sizeof(double) * kSmemDoubles * kWarps : 0;
    const int64_t blocks = (trials + kWarps - 1) / kWarps;
    CGX_CUDA(cudaFuncSetAttribute(batch_sketch_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    batch_sketch_gram<<<(unsigned)blocks, 32 * kWarps, smem, s>>>(master, t0, trials, B, FastMod((uint64_t)B), u, ld, n,
                                                                  d, su, gram_out, in_smem ? 1 : 0);
    count_launch(ctx);
    check_launch("batch_sketch_gram");
}

} // namespace cgx
