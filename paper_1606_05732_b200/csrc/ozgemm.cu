// ozgemm.cu -- stage 2 (Z = G . S.X, `gemm` in matrix.cpp:111-129) on the 5th-generation
// tensor cores.  sm_100a has no FP64 tcgen05 kind, so the FP64 product is emulated exactly
// the way an int8 tensor core can: Ozaki-style slicing.
//
//   * every row r of G (and every column j of S.X) gets a power-of-two scale 2^E with
//     max |row| < 2^E;
//   * each entry becomes the integer Y = trunc(x * 2^(8S-2-E)) (|Y| < 2^(8S-2): 54 bits at
//     S = 7, more than an fp64 mantissa) written as S balanced base-256 digits d_s in
//     [-128, 127], Y = sum_s d_s 256^(S-1-s) (oz_digits);
//   * Z(r, j) = 2^(E_r + F_j) * sum_{p < S} 2^(-8p-12) * sum_{s+t=p} (a_s . b_t): each digit
//     dot product a_s . b_t is an int8 x int8 -> int32 tcgen05.mma (kind::i8), exact;
//     the terms with s + t >= S (below 2^-(8S+4) relative) are dropped;
//   * products with the same weight p share one int32 accumulator in TMEM (S groups of 64
//     columns); a group holds at most S products of |128 * 128| per k, so it is drained to
//     fp64 registers every OZ_FK values of k (S * 2^14 * OZ_FK < 2^31).
//
// The only roundings are the fp64 drain of exact integers and the dropped terms: measured
// 4e-15 - 8e-15 relative Frobenius against cuBLAS fp64 at S = 7 on the c3/c5 shapes (the
// DMMA path's bar is 1e-12; the reference's own is 1e-8, test_sketch.cpp:192-209), 7e-13 at
// S = 6, 1.5e-10 at S = 5.
//
// Kernels: oz_absmax (per-row / per-column max), oz_slice (G's digits written straight into
// the UMMA canonical K-major no-swizzle tile image once per transform, so the GEMM moves one
// contiguous chunk per k-block with a 1-D bulk copy), oz_gemm (warp-specialized: S.X rows by
// bulk copy -> converter warps cut them into digit planes in shared memory -> one thread
// issues the tcgen05.mma -> TMEM -> epilogue warps drain to fp64).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

constexpr int OZ_MT = 128;    // MMA M (rows of G per CTA tile = TMEM lanes)
constexpr int OZ_NT = 64;     // MMA N (columns of S.X per CTA tile)
constexpr int OZ_KB = 32;     // k per MMA (int8: 32 bytes)
constexpr int OZ_FK = 16384;  // k per int32 accumulation before the drain to fp64

// ---- tcgen05 / TMEM wrappers ----------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major, no swizzle: core matrices of 8 rows x 16 B (128 B contiguous); the two core
// matrices of one 32 B k-step sit LBO = 128 B apart, consecutive 8-row groups SBO = 256 B.
__device__ __forceinline__ uint64_t umma_desc(unsigned saddr, unsigned lbo = 128, unsigned sbo = 256) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}
// kind::i8 instruction descriptor: D s32, A/B signed 8-bit, both K-major, M x N
constexpr uint32_t oz_idesc(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// arrive on `bar` once every previously issued tcgen05.mma of this thread has completed
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}
// the same arrive on the mbarrier at this offset in every CTA of `mask` (cluster)
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_addr(bar)),
        "h"(mask)
        : "memory");
}
// 1-D bulk copy landing at the same offset in every CTA of `mask`, completing on each one's
// mbarrier at `bar`'s offset
__device__ __forceinline__ void bulk_g2s_mc(void* smem, const void* gmem, unsigned bytes, uint64_t* bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_addr(bar)), "h"(mask)
        : "memory");
}
// TMA tile load of a 2-D tensor: box at (c0 = inner coordinate, r0 = row) -> smem, counted
// on `bar` (out-of-range elements are zero-filled and still counted)
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int c0, int r0, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_addr(smem)),
        "l"(map), "r"(c0), "r"(r0), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the address of this CTA's shared-memory word `a` in cluster CTA `rank`
__device__ __forceinline__ unsigned cluster_map(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_v2(unsigned addr, uint32_t x, uint32_t y) {
    asm volatile("st.shared::cluster.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(x), "r"(y) : "memory");
}
// bulk copy of `bytes` from this CTA's shared memory into a peer's (cluster addresses from
// cluster_map), completing on the peer's mbarrier
__device__ __forceinline__ void bulk_s2peer(unsigned dst_cluster, const void* src, unsigned bytes, unsigned bar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst_cluster),
                 "r"(smem_addr(src)), "r"(bytes), "r"(bar_cluster)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(unsigned cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// mbar_wait with cluster-scope acquire: the phase may complete by arrivals (and shared-memory
// writes) of another CTA of the cluster
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITC_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// amax[w] = max over k of |X[k * W + w]| as the bit pattern of a non-negative double
// (bit patterns of non-negative doubles order like the values).  W <= 4096.  With W even
// and a grid stride that is a multiple of W, every thread owns one column pair and keeps
// its maxima in registers over 16 B loads, 8 in flight.
__global__ void oz_absmax(const double* __restrict__ X, int64_t K, int64_t W, unsigned long long* __restrict__ amax) {
    extern __shared__ unsigned long long sm_max[];
    for (int64_t w = threadIdx.x; w < W; w += blockDim.x) sm_max[w] = 0;
    __syncthreads();
    auto bits = [](double v) { return (unsigned long long)__double_as_longlong(fabs(v)); };
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    if (W % 2 == 0 && (nthr * 2) % W == 0 && ((uintptr_t)X % 16) == 0) {
        const double2* X2 = reinterpret_cast<const double2*>(X);
        const int64_t total = K * W / 2;
        unsigned long long m0 = 0, m1 = 0;
        int64_t e = tid;
        for (; e + 7 * nthr < total; e += 8 * nthr) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(X2 + e + u * nthr);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                m0 = max(m0, bits(v[u].x));
                m1 = max(m1, bits(v[u].y));
            }
        }
        for (; e < total; e += nthr) {
            const double2 v = __ldg(X2 + e);
            m0 = max(m0, bits(v.x));
            m1 = max(m1, bits(v.y));
        }
        const int64_t w0 = (2 * tid) % W;
        if (tid < total) {
            atomicMax(&sm_max[w0], m0);
            atomicMax(&sm_max[w0 + 1], m1);
        }
    } else {
        for (int64_t e = tid; e < K * W; e += nthr) atomicMax(&sm_max[e % W], bits(X[e]));
    }
    __syncthreads();
    for (int64_t w = threadIdx.x; w < W; w += blockDim.x)
        if (sm_max[w]) atomicMax(&amax[w], sm_max[w]);
}

// exponent E with max < 2^E (0 for an all-zero row)
__device__ __forceinline__ int oz_exp(unsigned long long amax_bits) {
    if (amax_bits == 0) return 0;
    int e;
    frexp(__longlong_as_double((long long)amax_bits), &e);
    return e;
}

// Digits of NV consecutive k of one w, packed 4 per 32-bit word per plane (byte kk % 4 of
// word kk / 4).  Balanced base-256 digits: Y = trunc(x * 2^(8S-2-E)) (|Y| < 2^(8S-2)), and
// U = Y + O with O = 0x80 in each of the S low bytes; byte b of U minus 128 (= byte ^ 0x80)
// is digit S-1-b of Y, d in [-128, 127], Y = sum_s d_s 256^(S-1-s).  One byte permute per
// digit: no per-digit arithmetic.  Y itself comes from the bits of x with integer shifts:
// x = m * 2^(max(e,1) - 1075) (m the significand with its implicit bit, e the exponent
// field), so Y = m shifted by max(e,1) - 1077 + 8S - E (<= 1, since |x| < 2^E), negated for
// negative x -- the same integer as trunc(x * 2^(8S-2-E)) (that product is exact whenever
// it is >= 1), without the fp64 multiply and the F2I.S64.F64 conversion, whose throughput
// bounded the converter warps.
template <int S, int NV>
__device__ __forceinline__ void oz_digits(const double (&v)[NV], int E, uint32_t (&dig)[S][NV / 4]) {
    constexpr unsigned long long O = 0x0080808080808080ull >> (8 * (7 - S));
    const int tb = 1077 - 8 * S + E;
#pragma unroll
    for (int q = 0; q < NV / 4; ++q) {
        uint32_t lo[4], hi[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const long long bits = __double_as_longlong(v[4 * q + b]);
            const int ef = (int)((unsigned long long)bits >> 52) & 0x7ff;
            const unsigned long long m = ((unsigned long long)bits & 0xFFFFFFFFFFFFFull) | ((unsigned long long)(ef != 0) << 52);
            const int t = (ef > 1 ? ef : 1) - tb;
            unsigned long long y = t >= 0 ? m << (t < 63 ? t : 63) : m >> (-t < 63 ? -t : 63);
            if (bits < 0) y = 0ull - y;
            const unsigned long long U = y + O;
            lo[b] = (uint32_t)U;
            hi[b] = (uint32_t)(U >> 32);
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int bp = S - 1 - s;  // byte of U holding digit s
            const uint32_t* X = bp < 4 ? lo : hi;
            const uint32_t sel = (uint32_t)(bp & 3) | ((uint32_t)(4 + (bp & 3)) << 4);
            const uint32_t t01 = __byte_perm(X[0], X[1], sel), t23 = __byte_perm(X[2], X[3], sel);
            dig[s][q] = __byte_perm(t01, t23, 0x5410) ^ 0x80808080u;
        }
    }
}

// X (K x W, W contiguous) -> S digit planes in the UMMA tile image:
//   [w / R][k / 32][s][ (w%R)/8 ][ (k%32)/16 ][ w%8 ][ k%16 ]   (R x 32 bytes per plane)
// One thread: 16 consecutive k of one w -> one 16 B store per digit plane.  Padding (w >= W
// or k >= K) is written as zero digits.
template <int S, int R>
__global__ void oz_slice(const double* __restrict__ X, int64_t K, int64_t W, int64_t Wp, int64_t nkb,
                         const unsigned long long* __restrict__ amax, int8_t* __restrict__ img) {
    const int64_t groups = Wp * nkb * 2;  // (w, 16-k group)
    for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups;
         gi += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = gi % Wp, kg = gi / Wp;  // consecutive threads: consecutive w (coalesced reads)
        const int64_t k0 = kg * 16;
        const int E = w < W ? oz_exp(amax[w]) : 0;
        double v[16];
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) v[kk] = (w < W && k0 + kk < K) ? X[(k0 + kk) * W + w] : 0.0;
        uint32_t dig[S][4];
        oz_digits<S, 16>(v, E, dig);
        const int64_t wt = w / R, r = w % R, kb = k0 / OZ_KB, kc = (k0 % OZ_KB) / 16;
        int8_t* base = img + ((wt * nkb + kb) * S) * (int64_t)(R * OZ_KB) + (r / 8) * 256 + kc * 128 + (r % 8) * 16;
#pragma unroll
        for (int s = 0; s < S; ++s)
            *reinterpret_cast<uint4*>(base + (int64_t)s * R * OZ_KB) = make_uint4(dig[s][0], dig[s][1], dig[s][2], dig[s][3]);
    }
}

// shared memory: an MMA ring (G planes | S.X planes per stage, freed by the MMA commit) and
// a deeper ring of raw fp64 S.X tiles (freed as soon as the converters hold them in registers)
constexpr int OZ_RAW = OZ_KB * OZ_NT * 8;
template <int S>
constexpr int oz_stage_bytes() { return S * (OZ_MT + OZ_NT) * OZ_KB; }
constexpr int OZ_MAX_RING = 8;
constexpr int OZ_SMEM_MAX = 225 << 10;  // of the 227 KB opt-in, leaving the static barriers room
#ifndef OZ_CONVERTER_WARPS
#define OZ_CONVERTER_WARPS 8
#endif
#ifndef OZ_EXP
#define OZ_EXP 0  // measurement only: 1 = converters skip the digits, 2 = no G loads, 3 = no MMAs,
                 // 4 = no S.X loads and no MMAs, 5 = no S.X loads
#endif
constexpr int OZ_CW = OZ_CONVERTER_WARPS;   // converter warps: 32 * OZ_CW threads = 2 groups x 64 columns x k-groups
constexpr int OZ_GT = 16 * OZ_CW;           // threads per converter group
constexpr int OZ_VPT = OZ_KB * OZ_NT / OZ_GT;  // values of k per converter thread (16 or 8)
static_assert(OZ_VPT == 16 || OZ_VPT == 8, "converter warps: 8 or 16");
constexpr int OZ_THREADS = 32 * (OZ_CW + 7);

// position in a ring of n slots: slot index and the parity of the current pass (no division
// in the loops: the depths are runtime values)
struct RingPos {
    int idx = 0, n;
    unsigned phase = 0;
    __device__ explicit RingPos(int n_) : n(n_) {}
    __device__ void next() {
        if (++idx == n) {
            idx = 0;
            phase ^= 1u;
        }
    }
};

// One CTA: a 128 x 64 tile of Z over k-blocks [kb0, kb1) of its split.
//   warps 0-7:  converters, two groups of 4 on alternate k-blocks -- take the 32 x 64 fp64 S.X tile (TMA-staged, or loaded
//               directly), cut it into S digit planes in the UMMA image in shared memory;
//   warps 8-11: epilogue  -- drain the TMEM accumulators (lanes 32(w-8).. = tile rows) every
//               OZ_FK values of k, scale, and add into the split's partial tile in HBM;
//   warp 12:    producer  -- G's digit planes, one bulk copy per k-block (multicast across a
//               cluster of N tiles when csize > 1);
//   warp 13:    MMA       -- one thread issues the tcgen05.mma, S + S/2 per k-block;
//   warp 14:    producer  -- the S.X tile, one TMA load per k-block.
// MP (M-tile pairs, c5's m = 256): the two CTAs of a cluster hold the two M tiles of the same
// (N tile, split) and need the same S.X planes.  Each loads half of every S.X tile (16 of its
// 32 k), converts it, and sends its half of the planes to the peer with one DSMEM bulk copy,
// so every S.X value is converted once instead of once per M tile; G's planes are each CTA's
// own (no N-tile multicast in this mode).  The B planes are laid out k-half-major (each
// half of all S planes contiguous: LBO = S KB, SBO = 128 B) so that a half is one copy.  A
// stage is free once both CTAs' MMAs read it (their commits multicast to both `empty`
// barriers); `bfull` completes on one local arrive plus the peer's copy bytes.
template <int S, int MP>
__global__ void __launch_bounds__(OZ_THREADS, 1)
oz_gemm(const int8_t* __restrict__ aimg, int64_t a_nkb, int64_t a_kb0, const double* __restrict__ sx, int64_t K,
        int64_t d, int64_t nkb, int64_t kb_per_split, const unsigned long long* __restrict__ amax_a,
        const unsigned long long* __restrict__ amax_b, int64_t m, double* __restrict__ zpart, int staged, int nst,
        int nrs, int csize, const __grid_constant__ CUtensorMap sx_map) {
    constexpr int A_BYTES = S * OZ_MT * OZ_KB;
    constexpr int STAGE = oz_stage_bytes<S>();  // A planes | B planes
    constexpr int KH = MP ? OZ_KB / 2 : OZ_KB;   // k rows of the raw S.X tile this CTA loads and converts
    constexpr int VPT = KH * OZ_NT / OZ_GT;      // values per converter thread per k-block
    constexpr int RAWB = KH * OZ_NT * 8;         // bytes per raw S.X slot
    constexpr int FKB = OZ_FK / OZ_KB;           // k-blocks per accumulation
    constexpr int W_EPI = OZ_CW, W_PROD = OZ_CW + 4, W_MMA = OZ_CW + 5, W_RAW = OZ_CW + 6;
    const int OZ_STAGES = nst, RS = nrs;         // ring depths (<= OZ_MAX_RING each)
    // the dynamic window is only guaranteed 16 B alignment under separate compilation: the
    // ring starts at the next 1 KB boundary (1 KB extra requested); operand images that
    // straddle it produce wrong products
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
    uint8_t* raw_ring = smem + OZ_STAGES * STAGE;
    __shared__ uint64_t full[OZ_MAX_RING], bfull[OZ_MAX_RING], empty[OZ_MAX_RING], acc_full, acc_empty;
    __shared__ uint64_t rfull[OZ_MAX_RING], rempty[OZ_MAX_RING];
    __shared__ uint32_t tmem_slot;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t mt = blockIdx.x, nt = blockIdx.y, split = blockIdx.z;
    const int64_t kb0 = split * kb_per_split;
    const int64_t kb1 = kb0 + kb_per_split < nkb ? kb0 + kb_per_split : nkb;
    const int64_t nk = kb1 - kb0;
    const int64_t nchunks = (nk + FKB - 1) / FKB;
    pdl_trigger();

    if (threadIdx.x == 0) {
        for (int i = 0; i < OZ_STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&bfull[i], MP ? 1 : OZ_GT);  // MP: the group's elected arrive (+ the peer's copy bytes)
            mbar_init(&empty[i], csize);  // every CTA of the cluster has read the stage
        }
        for (int i = 0; i < RS; ++i) {
            mbar_init(&rfull[i], 1);
            mbar_init(&rempty[i], OZ_GT);
        }
        mbar_init(&acc_full, 1);
        mbar_init(&acc_empty, 128);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == W_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (csize > 1) cluster_sync_all();  // barriers initialized cluster-wide before any remote arrive
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    pdl_wait();  // S.X and its column maxima (the sketch before) are complete
    // cluster of csize CTAs along the N tiles: same (M tile, split), so the same G planes; each
    // CTA fetches 1/csize of every G chunk and multicasts it to all of them
    const unsigned crank = csize > 1 ? cluster_rank() : 0u;
    const uint16_t cmask = (uint16_t)((1u << csize) - 1u);

    if (warp < OZ_CW) {
        // converters, in two groups that take alternate k-blocks: while one group waits for
        // its raw tile or for the MMAs to free its stage, the other converts (one group of
        // all converter warps on every k-block spent most of its time in those waits:
        // stage 2 with the MMAs removed took nearly as long as with them).
        // thread = (column j of the tile, k-group kq of the k-block: OZ_VPT values of k)
        const int grp = (int)threadIdx.x / OZ_GT, gt = (int)threadIdx.x % OZ_GT;
        const int j = gt % OZ_NT, kq = gt / OZ_NT;
        const int64_t col = nt * OZ_NT + j;
        const bool colok = col < d;
        const int F = colok ? oz_exp(amax_b[col]) : 0;
        const double* src = sx + (colok ? col : 0);
        // canonical K-major image: 8-row group j/8, 16 B core matrix, row j%8, byte within it
        const int kloc = kq * VPT;                          // k within this CTA's part of the tile
        const int kofs = (MP ? (int)crank * KH : 0) + kloc;  // k within the k-block
        // plane s of this thread's values: non-MP -- [s][j/8: 256 B][k/16: 128 B][j%8: 16 B][k%16];
        // MP -- [k/16: S KB][s: 1 KB][j/8: 128 B][j%8: 16 B][k%16] (a k-half is contiguous)
        const uint32_t soff = MP ? (uint32_t)((kofs / 16) * S * 1024 + (j / 8) * 128 + (j % 8) * 16 + (kofs % 16))
                                 : (uint32_t)((j / 8) * 256 + (kofs / 16) * 128 + (j % 8) * 16 + (kofs % 16));
        constexpr int PSTRIDE = MP ? 1024 : OZ_NT * OZ_KB;  // bytes between planes
        double cur[VPT];
        RingPos sp(OZ_STAGES), rp(RS);
        if (grp) {
            sp.next();
            rp.next();
        }
        for (int64_t i = grp; i < nk; i += 2, sp.next(), sp.next(), rp.next(), rp.next()) {
            uint8_t* stage = smem + sp.idx * STAGE;
            if (staged) {  // TMA zero-fills past K and d
                mbar_wait(&rfull[rp.idx], rp.phase);
                const double* raw = reinterpret_cast<const double*>(raw_ring + rp.idx * RAWB) + kloc * OZ_NT + j;
#pragma unroll
                for (int kk = 0; kk < VPT; ++kk) cur[kk] = raw[kk * OZ_NT];
            } else {  // direct path: straight from global
                const int64_t k0 = (kb0 + i) * OZ_KB + kofs;
#pragma unroll
                for (int kk = 0; kk < VPT; ++kk) cur[kk] = (colok && k0 + kk < K) ? __ldg(src + (k0 + kk) * d) : 0.0;
            }
            uint32_t dig[S][VPT / 4];
            if (OZ_EXP != 1) oz_digits<S, VPT>(cur, F, dig);
            if (i >= OZ_STAGES) {  // MMAs of k-block i - STAGES done (a peer's, too, with clusters: cluster scope)
                if (csize > 1)
                    mbar_wait_cluster(&empty[sp.idx], sp.phase ^ 1u);
                else
                    mbar_wait(&empty[sp.idx], sp.phase ^ 1u);
            }
            uint8_t* bp = stage + A_BYTES + soff;
#pragma unroll
            for (int s = 0; s < S * (OZ_EXP != 1); ++s) {
                if constexpr (VPT == 16)
                    *reinterpret_cast<uint4*>(bp + s * PSTRIDE) = make_uint4(dig[s][0], dig[s][1], dig[s][2], dig[s][3]);
                else
                    *reinterpret_cast<uint2*>(bp + s * PSTRIDE) = make_uint2(dig[s][0], dig[s][1]);
            }
            // one proxy fence orders both this thread's generic accesses before the async
            // proxy: the plane writes before the MMA reads them, and the raw-tile reads before
            // the next TMA overwrite of that slot (releasing the slot before a fence raced at
            // S = 6; a second fence per k-block cost c5 0.7 ms)
            if constexpr (MP) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(OZ_GT) : "memory");  // the group's half is written
                if (gt == 0) {
                    const uint32_t half = (uint32_t)crank * S * 1024;
                    mbar_arrive_expect_tx(&bfull[sp.idx], S * 1024);  // local arrive; the peer's half follows
                    bulk_s2peer(cluster_map(smem_addr(stage + A_BYTES + half), crank ^ 1u), stage + A_BYTES + half,
                                S * 1024, cluster_map(smem_addr(&bfull[sp.idx]), crank ^ 1u));
                }
            } else {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&bfull[sp.idx]);
            }
            if (staged) mbar_arrive(&rempty[rp.idx]);
        }
    } else if (warp < W_PROD) {
        // epilogue: every accumulation's integer groups -> fp64 (smallest weight first), scaled
        // by 2^(E_r + F_j) (exact), added into the split's partial tile (row = lane)
        const int ew = warp - W_EPI;
        const uint32_t trow = tmem + ((uint32_t)(ew * 32) << 16);
        const int64_t r = mt * OZ_MT + ew * 32 + lane;
        const bool rok = r < m;
        const int Er = rok ? oz_exp(amax_a[r]) : 0;
        double* zp = zpart + split * m * d;
        for (int64_t c = 0; c < nchunks; ++c) {
            mbar_wait_sleep(&acc_full, (unsigned)(c & 1), 256);  // a whole accumulation: sleep between polls
            tc_fence_after();
#pragma unroll 1
            for (int q = 0; q < OZ_NT / 16; ++q) {
                double part[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) part[jj] = 0.0;
#pragma unroll
                for (int p = S - 1; p >= 0; --p) {
                    int v[16];
                    tmem_ld16(trow + (uint32_t)(p * OZ_NT + q * 16), v);
                    const double wgt = ldexp(1.0, -8 * p - 12);
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) part[jj] = fma((double)v[jj], wgt, part[jj]);
                }
                if (rok) {
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        const int64_t col = nt * OZ_NT + q * 16 + jj;
                        if (col < d) {
                            const double v = ldexp(part[jj], Er + oz_exp(amax_b[col]));
                            zp[col * m + r] = c == 0 ? v : zp[col * m + r] + v;
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&acc_empty);
        }
    } else if (warp == W_PROD) {
        if (lane == 0) {  // producer: G's digit planes, one bulk copy per stage
            const int8_t* ga = aimg + (mt * a_nkb + a_kb0 + kb0) * (int64_t)A_BYTES;
            RingPos sp(OZ_STAGES);
            for (int64_t i = 0; i < nk; ++i, sp.next()) {
                if (i >= OZ_STAGES) {
                    if (csize > 1)
                        mbar_wait_cluster(&empty[sp.idx], sp.phase ^ 1u);
                    else
                        mbar_wait(&empty[sp.idx], sp.phase ^ 1u);
                }
                if (OZ_EXP == 2) { mbar_arrive(&full[sp.idx]); continue; }
                mbar_arrive_expect_tx(&full[sp.idx], A_BYTES);
                if (csize > 1 && !MP) {
                    const unsigned part = A_BYTES / csize;
                    bulk_g2s_mc(smem + sp.idx * STAGE + crank * part, ga + i * A_BYTES + crank * part, part,
                                &full[sp.idx], cmask);
                } else {
                    bulk_g2s(smem + sp.idx * STAGE, ga + i * A_BYTES, A_BYTES, &full[sp.idx]);
                }
            }
            // producer tail: the last stages' empty[] phases count every cluster peer's commit
            // (an asynchronous multicast arrive), so once they complete no peer still has an
            // arrive in flight towards this CTA's shared memory when the teardown sync lets it
            // exit
            if (csize > 1) {
                const int64_t i0 = nk > OZ_STAGES ? nk - OZ_STAGES : 0;
                for (int64_t i = i0; i < nk; ++i) mbar_wait_cluster(&empty[i % OZ_STAGES], (unsigned)((i / OZ_STAGES) & 1));
            }
        }
        __syncwarp();
    } else if (warp == W_RAW) {
        if (staged && lane == 0) {  // producer: the block's 32 x 64 fp64 S.X tile, one TMA load
            // (32 row-sized bulk copies cost ~64 cycles of issue each: they bounded the GEMM)
            RingPos rp(RS);
            for (int64_t i = 0; i < nk; ++i, rp.next()) {
                if (i >= RS) mbar_wait(&rempty[rp.idx], rp.phase ^ 1u);
                if (OZ_EXP == 4 || OZ_EXP == 5) { mbar_arrive(&rfull[rp.idx]); continue; }
                mbar_arrive_expect_tx(&rfull[rp.idx], KH * OZ_NT * 8);
                tma_load_2d(raw_ring + rp.idx * RAWB, &sx_map, (int)(nt * OZ_NT),
                            (int)((kb0 + i) * OZ_KB + (MP ? crank * KH : 0)), &rfull[rp.idx]);
            }
        }
        __syncwarp();
    } else if (warp == W_MMA) {
        if (lane == 0) {  // MMA issuer
            const unsigned sbase = smem_addr(smem);
            RingPos sp(OZ_STAGES);
            for (int64_t i = 0; i < nk; ++i, sp.next()) {
                const int st = sp.idx;
                const int64_t c = i / FKB;
                const bool first = (i % FKB) == 0;
                if (first && c > 0) mbar_wait(&acc_empty, (unsigned)((c - 1) & 1));  // drained
                mbar_wait(&full[st], sp.phase);
                if (MP)
                    mbar_wait_cluster(&bfull[st], sp.phase);
                else
                    mbar_wait(&bfull[st], sp.phase);
                tc_fence_after();
                const unsigned sa = sbase + st * STAGE, sb = sa + A_BYTES;
                // A plane s against B planes t0 .. t0+w-1 in one MMA: the planes sit
                // consecutively in shared memory, so they form one N = 64w operand, and the
                // products land in groups s+t0 .. s+t0+w-1, consecutive TMEM columns.  Up to
                // N = 256 per instruction: S(S+1)/2 products in ~S + S/2 instructions (an
                // N = 64 MMA costs ~3x its share of the tensor pipe, tools/microbench/umma_i8.cu).
#pragma unroll
                for (int s = 0; s < S * (OZ_EXP != 3 && OZ_EXP != 4); ++s)
#pragma unroll
                    for (int t0 = 0; t0 < S - s; t0 += 4) {
                        const int w = S - s - t0 < 4 ? S - s - t0 : 4;
                        mma_i8(tmem + (uint32_t)((s + t0) * OZ_NT), umma_desc(sa + s * OZ_MT * OZ_KB),
                               MP ? umma_desc(sb + t0 * 1024, S * 1024, 128) : umma_desc(sb + t0 * OZ_NT * OZ_KB),
                               oz_idesc(OZ_MT, OZ_NT * w),
                               (first && s == 0) ? 0 : 1);
                    }
                if (csize > 1)
                    mma_commit_mc(&empty[st], cmask);  // stage free in every CTA's view
                else
                    mma_commit(&empty[st]);  // stage free once these MMAs have read it
                if ((i % FKB) == FKB - 1 || i == nk - 1) mma_commit(&acc_full);
            }
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (csize > 1) cluster_sync_all();  // no CTA leaves while its peers may still multicast into it
    if (warp == W_MMA) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// Rows of G and columns of S.X that the digit planes cannot represent -- a maximum that is
// NaN or +-Inf (bits >= 0x7ff0...), or below 2^-960 (the scale 2^(8S-2-E) would overflow)
// -- get their Z entries recomputed here in plain fp64, the reference's way (gemm,
// matrix.cpp:111-129: ascending l, zero S.X entries skipped, separate multiply and add), so
// NaN and Inf propagate as they do there.  Launched after every tensor-core stage 2; a block
// whose row / column is representable returns at once.
__device__ __forceinline__ bool oz_bad(unsigned long long bits) {
    const unsigned long long e = bits >> 52;
    return e >= 0x7ff || (bits != 0 && e < 63);
}

__global__ void oz_fixup(const double* __restrict__ g, const double* __restrict__ sx, int64_t m, int64_t K, int64_t d,
                         const unsigned long long* __restrict__ amax_a, const unsigned long long* __restrict__ amax_b,
                         double* __restrict__ z) {
    const int64_t b = blockIdx.x;
    if (b < d) {  // column b of Z
        if (!oz_bad(amax_b[b])) return;
        for (int64_t r = threadIdx.x; r < m; r += blockDim.x) {
            double acc = 0.0;
            for (int64_t l = 0; l < K; ++l) {
                const double x = sx[l * d + b];
                if (x == 0.0) continue;
                acc = __dadd_rn(acc, __dmul_rn(g[l * m + r], x));
            }
            z[b * m + r] = acc;
        }
    } else {  // row r of Z
        const int64_t r = b - d;
        if (!oz_bad(amax_a[r])) return;
        for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
            double acc = 0.0;
            for (int64_t l = 0; l < K; ++l) {
                const double x = sx[l * d + j];
                if (x == 0.0) continue;
                acc = __dadd_rn(acc, __dmul_rn(g[l * m + r], x));
            }
            z[j * m + r] = acc;
        }
    }
}

void run_absmax(cgx_ctx* ctx, const double* X, int64_t K, int64_t W, unsigned long long* out, cudaStream_t s) {
    // 256 threads; blocks chosen so that 2 * threads * blocks is a multiple of W when W is even
    const int64_t t = 256;
    int64_t blocks = ctx->num_sms * 4;
    if (W % 2 == 0) {
        const int64_t q = W / 2;  // thread count must be a multiple of q
        auto gcd = [](int64_t a, int64_t b) { while (b) { const int64_t r = a % b; a = b; b = r; } return a; };
        const int64_t unit = q / gcd(q, t);  // blocks must be a multiple of unit
        blocks = (blocks + unit - 1) / unit * unit;
    }
    const int64_t need = (K * W / 2 + t - 1) / t;
    if (blocks > need && W % 2 != 0) blocks = need < 1 ? 1 : need;
    oz_absmax<<<(unsigned)blocks, (unsigned)t, sizeof(unsigned long long) * (size_t)W, s>>>(X, K, W, out);
    count_launch(ctx);
    check_launch("oz_absmax");
}

// digit image of G (m x K column-major) and its row maxima
template <int S>
void build_g_image(cgx_ctx* ctx, const double* g, int64_t m, int64_t K, unsigned long long* amax, int8_t* img,
                   cudaStream_t s) {
    const int64_t nkb = (K + OZ_KB - 1) / OZ_KB, mp = (m + OZ_MT - 1) / OZ_MT * OZ_MT;
    CGX_CUDA(cudaMemsetAsync(amax, 0, sizeof(unsigned long long) * (size_t)m, s));
    run_absmax(ctx, g, K, m, amax, s);
    int64_t b = (mp * nkb * 2 + 255) / 256;
    if (b > ctx->num_sms * 16) b = ctx->num_sms * 16;
    oz_slice<S, OZ_MT><<<(unsigned)b, 256, 0, s>>>(g, K, m, mp, nkb, amax, img);
    count_launch(ctx);
    check_launch("oz_slice(G)");
}

template <int S>
bool run_ozaki(cgx_ctx* ctx, const cgx_xform* xf, int64_t b0, int64_t b1, const double* sx, int64_t d, double* z,
               cudaStream_t s) {
    const int64_t m = xf->m, K = b1 - b0;
    const int64_t nkb = (K + OZ_KB - 1) / OZ_KB;
    const int64_t tm = (m + OZ_MT - 1) / OZ_MT, tn = (d + OZ_NT - 1) / OZ_NT;
    const int64_t mp = tm * OZ_MT;
    // G's digit image: built once per transform (G is part of the transform, like t.g) and
    // kept until G changes; a view or an unaligned bucket range slices its own copy
    const int8_t* aimg;
    const unsigned long long* amax_a;
    int64_t a_nkb, a_kb0;
    if (!xf->view && b0 % OZ_KB == 0) {
        cgx_xform* mx = const_cast<cgx_xform*>(xf);
        if (mx->oz_gS != S) {
            oz_drop_image(mx);
            const int64_t fkb = (xf->B + OZ_KB - 1) / OZ_KB;
            // (7/8 of G's bytes; if HBM cannot hold it, stage 2 stays on the FP64 DMMA pipe)
            if (cudaMalloc((void**)&mx->oz_gimg, (size_t)(S * mp * fkb * OZ_KB)) != cudaSuccess ||
                cudaMalloc((void**)&mx->oz_gmax, sizeof(unsigned long long) * (size_t)m) != cudaSuccess) {
                cudaGetLastError();
                if (mx->oz_gimg) cudaFree(mx->oz_gimg);
                mx->oz_gimg = nullptr;
                mx->oz_gmax = nullptr;
                return false;
            }
            build_g_image<S>(ctx, xf->g_dev, m, xf->B, mx->oz_gmax, mx->oz_gimg, s);
            mx->oz_gS = S;
        }
        aimg = xf->oz_gimg;
        amax_a = xf->oz_gmax;
        a_nkb = (xf->B + OZ_KB - 1) / OZ_KB;
        a_kb0 = b0 / OZ_KB;
    } else {
        unsigned long long* am = (unsigned long long*)ctx->oz_max.get(sizeof(unsigned long long) * (size_t)m);
        int8_t* img = (int8_t*)ctx->oz_a.get((size_t)(S * mp * nkb * OZ_KB));
        build_g_image<S>(ctx, xf->g_dev + b0 * m, m, K, am, img, s);
        aimg = img;
        amax_a = am;
        a_nkb = nkb;
        a_kb0 = 0;
    }
    // column maxima of S.X: already folded in by the sketch that produced it (the CSR gather),
    // or one pass here
    unsigned long long* amax_b = (unsigned long long*)ctx->oz_b.get(sizeof(unsigned long long) * (size_t)d);
    if (!(ctx->oz_colmax_for == sx && ctx->oz_colmax_d == d && b0 == 0 && b1 == xf->B)) {
        CGX_CUDA(cudaMemsetAsync(amax_b, 0, sizeof(unsigned long long) * (size_t)d, s));
        run_absmax(ctx, sx, K, d, amax_b, s);
    }
    ctx->oz_colmax_for = nullptr;
    // M-tile pairs (MP kernel): the two M tiles of each (N tile, split) share one conversion of
    // S.X (option oz_mpair; needs an even number of M tiles)
    const bool mpair = ctx->opt_oz_mpair && tm % 2 == 0;
    // S.X tiles staged by TMA when its rows are 16 B aligned (a tensor map of the K x d
    // row-major block; boxes of 32 rows x 64 columns -- 16 rows for MP -- zero-filled past the
    // edges)
    CUtensorMap sx_map;
    memset(&sx_map, 0, sizeof(sx_map));
    int staged = ctx->opt_oz_staged && d % 2 == 0 && ((uintptr_t)sx % 16) == 0 && K < (1ll << 31);
    if (staged) {
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        if (!encode) {
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                encode = nullptr;
        }
        const cuuint64_t gdim[2] = {(cuuint64_t)d, (cuuint64_t)K};
        const cuuint64_t gstride[1] = {(cuuint64_t)d * 8};
        const cuuint32_t box[2] = {OZ_NT, (cuuint32_t)(mpair ? OZ_KB / 2 : OZ_KB)}, estride[2] = {1, 1};
        staged = encode && encode(&sx_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)sx, gdim, gstride, box, estride,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    // ring depths: the MMA ring as configured (default 3 stages at S >= 6, else 4), the raw
    // S.X ring takes what is left (<= 8)
    int nst = ctx->opt_oz_st > 0 ? (int)ctx->opt_oz_st : (S >= 6 ? 3 : 4);
    const int64_t stage_bytes = oz_stage_bytes<S>();
    if (nst > OZ_MAX_RING) nst = OZ_MAX_RING;
    const int64_t raw_bytes = mpair ? OZ_RAW / 2 : OZ_RAW;  // MP: a CTA stages half of each tile
    const int64_t raw_min = staged ? 2 * raw_bytes : 0;     // the direct path needs no raw ring
    while (nst > 2 && nst * stage_bytes + raw_min + 1024 > OZ_SMEM_MAX) --nst;
    int nrs = staged ? (int)((OZ_SMEM_MAX - 1024 - nst * stage_bytes) / raw_bytes) : 0;
    // (option oz_rs counts tiles of 16 KB: MP's half tiles get twice as many slots in the same bytes)
    const int64_t rs_req = ctx->opt_oz_rs * (mpair ? 2 : 1);
    if (rs_req > 0 && rs_req < nrs) nrs = (int)rs_req;
    if (nrs > OZ_MAX_RING) nrs = OZ_MAX_RING;
    // the two converter groups take alternate k-blocks: an even raw ring gives each group its
    // own slots (with an odd one a group's consecutive waits on a slot would be two phases
    // apart, which a parity wait cannot tell from one)
    if (staged) nrs = nrs < 2 ? 2 : nrs & ~1;
    const size_t smem = (size_t)(nst * stage_bytes + nrs * raw_bytes + 1024);
    auto kern = mpair ? oz_gemm<S, 1> : oz_gemm<S, 0>;
    CGX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // clusters along the N tiles share G's planes by multicast: the GEMM is bound by the
    // operand traffic out of L2, and every N tile otherwise re-reads the same G chunks
    int csize = mpair ? 2 : (int)ctx->opt_oz_cluster;
    while (csize > 1 && !mpair && tn % csize) csize >>= 1;
    if (csize < 1) csize = 1;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    cfg.blockDim = dim3(OZ_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = mpair ? 2u : 1u;  // MP: the M-tile pair; else N tiles sharing G's planes
    attr[0].val.clusterDim.y = mpair ? 1u : (unsigned)csize;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ctx->opt_pdl ? 2 : 1;
    // one wave: as many splits as co-resident clusters allow (clusters must fit in a GPC)
    int64_t resident = ctx->num_sms;
    if (csize > 1) {
        cfg.gridDim = dim3((unsigned)tm, (unsigned)tn, 1);
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters > 0)
            resident = (int64_t)nclusters * csize;
        cudaGetLastError();
    }
    int64_t splits = resident / (tm * tn);
    if (splits < 1) splits = 1;
    if (splits > nkb) splits = nkb;
    const int64_t kps = (nkb + splits - 1) / splits;
    splits = (nkb + kps - 1) / kps;
    double* zpart = (double*)ctx->zpart.get(sizeof(double) * (size_t)(splits * m * d));
    cfg.gridDim = dim3((unsigned)tm, (unsigned)tn, (unsigned)splits);
    CGX_CUDA(cudaLaunchKernelEx(&cfg, kern, aimg, a_nkb, a_kb0, sx, K, d, nkb, kps, amax_a, amax_b, m, zpart,
                                staged, nst, nrs, csize, sx_map));
    count_launch(ctx);
    check_launch("oz_gemm");
    launch_reduce_splits(ctx, zpart, splits, m * d, z, s);
    oz_fixup<<<(unsigned)(d + m), 128, 0, s>>>(xf->g_dev + b0 * m, sx, m, K, d, amax_a, amax_b, z);
    count_launch(ctx);
    check_launch("oz_fixup");
    return true;
}

} // namespace

void oz_drop_image(cgx_xform* xf) {
    if (xf->oz_gimg) cudaFree(xf->oz_gimg);
    if (xf->oz_gmax) cudaFree(xf->oz_gmax);
    xf->oz_gimg = nullptr;
    xf->oz_gmax = nullptr;
    xf->oz_gS = 0;
}

bool oz_stage2_applies(const cgx_ctx* ctx, const cgx_xform* xf, int64_t d) {
    const int64_t S = ctx->opt_oz_slices;
    return S >= 3 && S <= 7 && xf->g_dev && xf->m <= 4096 && d >= 1 && d <= 4096 &&
           xf->m * d >= ctx->opt_oz_min_z;  // small Z: the split-K DMMA stream is faster
}

bool launch_gemm_ozaki(cgx_ctx* ctx, const cgx_xform* xf, int64_t b0, int64_t b1, const double* sx, int64_t d,
                       double* z, cudaStream_t s) {
    const int S = (int)ctx->opt_oz_slices;
    if (!oz_stage2_applies(ctx, xf, d) || b1 <= b0) {
        ctx->oz_colmax_for = nullptr;
        return false;
    }
    switch (S) {
        case 3: return run_ozaki<3>(ctx, xf, b0, b1, sx, d, z, s);
        case 4: return run_ozaki<4>(ctx, xf, b0, b1, sx, d, z, s);
        case 5: return run_ozaki<5>(ctx, xf, b0, b1, sx, d, z, s);
        case 6: return run_ozaki<6>(ctx, xf, b0, b1, sx, d, z, s);
        case 7: return run_ozaki<7>(ctx, xf, b0, b1, sx, d, z, s);
        default: return false;
    }
}

} // namespace cgx
