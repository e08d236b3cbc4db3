// scan.cu -- device exclusive prefix sums (reduce-then-scan, recursive over block sums).
// Used for bucket offsets (B+1), radix-sort digit offsets and CSR row offsets.
#include "internal.h"

namespace cgx {
namespace {

constexpr int kThreads = 1024;
constexpr int kItems = 4;
constexpr int kTile = kThreads * kItems;

template <typename T>
__device__ T block_excl_scan(T v, T* warp_sums, T* total) {
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)lane >= o) incl += t;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T w = lane < (kThreads / 32) ? warp_sums[lane] : T(0);
        T wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T t = __shfl_up_sync(0xffffffffu, wi, o);
            if ((int)lane >= o) wi += t;
        }
        if (lane < (kThreads / 32)) warp_sums[lane] = wi - w;
        if (lane == 31) *total = wi;
    }
    __syncthreads();
    return incl - v + warp_sums[warp];
}

template <typename T>
__global__ void __launch_bounds__(kThreads) scan_tiles(const T* in, T* out, T* sums, int64_t count) {
    __shared__ T warp_sums[32];
    __shared__ T total;
    const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kItems;
    T v[kItems];
    T run = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        v[k] = base + k < count ? in[base + k] : T(0);
        T t = v[k];
        v[k] = run;
        run += t;
    }
    T pre = block_excl_scan<T>(run, warp_sums, &total);
#pragma unroll
    for (int k = 0; k < kItems; ++k)
        if (base + k < count) out[base + k] = v[k] + pre;
    if (threadIdx.x == 0 && sums) sums[blockIdx.x] = total;
}

template <typename T>
__global__ void add_tile_offsets(T* out, const T* sums, int64_t count) {
    const int64_t base = (int64_t)blockIdx.x * kTile;
    const T add = sums[blockIdx.x];
    for (int64_t i = base + threadIdx.x; i < base + kTile && i < count; i += blockDim.x) out[i] += add;
}

template <typename T>
void scan_rec(cgx_ctx* ctx, const T* in, T* out, int64_t count, T* tmp, cudaStream_t s) {
    if (count <= 0) return;
    const int64_t tiles = (count + kTile - 1) / kTile;
    if (tiles == 1) {
        scan_tiles<T><<<1, kThreads, 0, s>>>(in, out, nullptr, count);
        count_launch(ctx);
        check_launch("scan_tiles");
        return;
    }
    T* sums = tmp;
    scan_tiles<T><<<(unsigned)tiles, kThreads, 0, s>>>(in, out, sums, count);
    count_launch(ctx);
    check_launch("scan_tiles");
    scan_rec<T>(ctx, sums, sums, tiles, tmp + tiles, s);
    add_tile_offsets<T><<<(unsigned)tiles, 256, 0, s>>>(out, sums, count);
    count_launch(ctx);
    check_launch("add_tile_offsets");
}

template <typename T>
void scan_entry(cgx_ctx* ctx, const T* in, T* out, int64_t count, cudaStream_t s) {
    // Total temp over all recursion levels < count / (kTile - 1) + levels.
    int64_t need = 0;
    for (int64_t c = count; c > 1;) {
        c = (c + kTile - 1) / kTile;
        need += c;
        if (c == 1) break;
    }
    T* tmp = (T*)ctx->tmp.get(sizeof(T) * (size_t)(need + 1));
    scan_rec<T>(ctx, in, out, count, tmp, s);
}

} // namespace

void exclusive_scan_u32(cgx_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t count, cudaStream_t s) {
    scan_entry<uint32_t>(ctx, in, out, count, s);
}
void exclusive_scan_i64(cgx_ctx* ctx, const int64_t* in, int64_t* out, int64_t count, cudaStream_t s) {
    scan_entry<int64_t>(ctx, in, out, count, s);
}

} // namespace cgx
