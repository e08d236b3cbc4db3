// datagen.cu -- seeded synthetic inputs for the BASELINE configs, generated in HBM.
//
// The reference benchmarks no public dataset (BASELINE.json "published": {}); these
// counter-based generators stand in for it with the configs' shapes and value
// distributions.  Entry e of a stream with seed s is the fp32 N(0,1) quantile of draw e
// of SeededRng(s) (oracle/cgoracle.c cgo_normal_f32 is the CPU twin).
//   dense  : entry (i, j) = stream entry i*d + j
//   CSR    : entry (i, j) present iff uniform(draw i*d+j of mix64(seed,1)) < density;
//            its value is entry i*d + j of stream mix64(seed,2).  Columns come out sorted
//            and distinct per row (the CSR invariant, reference matrix.cpp:92-109).
#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

template <typename T>
__global__ void gen_dense_kernel(uint64_t seed, int64_t row0, int64_t n, int64_t d, int layout, T* x) {
    const int64_t total = n * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        // e enumerates the destination in its own layout for coalesced stores
        int64_t i, j;
        if (layout == CGX_ROW_MAJOR) {
            i = e / d;
            j = e - i * d;
        } else {
            j = e / n;
            i = e - j * n;
        }
        x[e] = (T)datagen_normal(seed, (uint64_t)((row0 + i) * d + j));
    }
}

__global__ void gen_csr_counts_kernel(uint64_t mseed, int64_t n, int64_t d, double density, int64_t* counts) {
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (row >= n) return;
    int64_t c = 0;
    for (int64_t j = lane; j < d; j += 32) c += uniform53(rng_draw(mseed, (uint64_t)(row * d + j))) < density;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[row] = c;
}

__global__ void gen_csr_fill_kernel(uint64_t mseed, uint64_t vseed, int64_t n, int64_t d, double density,
                                    const int64_t* rowptr, int32_t* cols, float* vals) {
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    if (row >= n) return;
    int64_t pos = rowptr[row];
    for (int64_t j0 = 0; j0 < d; j0 += 32) {
        const int64_t j = j0 + lane;
        const bool in = j < d && uniform53(rng_draw(mseed, (uint64_t)(row * d + j))) < density;
        const unsigned mask = __ballot_sync(0xffffffffu, in);
        if (in) {
            const int64_t p = pos + __popc(mask & ((1u << lane) - 1u));
            cols[p] = (int32_t)j;
            vals[p] = datagen_normal(vseed, (uint64_t)(row * d + j));
        }
        pos += __popc(mask);
    }
}

} // namespace

void launch_gen_dense(cgx_ctx* ctx, uint64_t seed, int64_t row0, int64_t n, int64_t d, int dtype, int layout, void* x,
                      cudaStream_t s) {
    const int blocks = ctx->num_sms * 16;
    if (dtype == CGX_F32)
        gen_dense_kernel<float><<<blocks, 256, 0, s>>>(seed, row0, n, d, layout, (float*)x);
    else
        gen_dense_kernel<double><<<blocks, 256, 0, s>>>(seed, row0, n, d, layout, (double*)x);
    count_launch(ctx);
    check_launch("gen_dense");
}

void launch_gen_csr_counts(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, double density, int64_t* rowptr,
                           cudaStream_t s) {
    const int64_t threads = n * 32;
    gen_csr_counts_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(mix64(seed, 1), n, d, density, rowptr);
    count_launch(ctx);
    check_launch("gen_csr_counts");
    CGX_CUDA(cudaMemsetAsync(rowptr + n, 0, sizeof(int64_t), s));
    exclusive_scan_i64(ctx, rowptr, rowptr, n + 1, s);
}

void launch_gen_csr_fill(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, double density, const int64_t* rowptr,
                         int32_t* cols, float* vals, cudaStream_t s) {
    const int64_t threads = n * 32;
    gen_csr_fill_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(mix64(seed, 1), mix64(seed, 2), n, d,
                                                                         density, rowptr, cols, vals);
    count_launch(ctx);
    check_launch("gen_csr_fill");
}

} // namespace cgx
