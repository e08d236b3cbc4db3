// csr_atomic.cu -- S.X for CSR X by bucket-range partition + L2-resident fp64 atomics.
//
// Replaces countsketch_apply(map, SparseMatrix) (reference src/sketch.cpp:68-113) for
// short-row CSR, where the bucket-ordered row gather (sketch_csr.cu) is bound by the DRAM
// random-access rate: every row costs three random reads (its offsets, columns, values),
// so c3 (2.56 nnz/row) moves 14 GB of 64 B sectors for 2.45 GB of data.
// Here X is read once, sequentially:
//   1. count:   per row, bucket = the seeded hash of its global index (sketch.cpp:21-26),
//               kept as a 4-byte row record; nonzeros per (partition = bucket >> pshift,
//               sub-cursor) (reads row offsets only);
//   2. scatter: each CTA takes a tile of rows, turns its nonzeros into 8-byte records
//               (key = bucket << cbits | column, value = sign * x as fp32 -- exact), stages
//               them grouped by partition in shared memory and stores each partition's run
//               coalesced into the partition's region (one global reservation per partition
//               and tile);
//   3. accumulate: the records, partition after partition, are added into S.X with fp64
//               RED.ADD; a partition's S.X slice (8 MB by default) is zero-filled just before
//               its records arrive, so the adds resolve in L2 and S.X is written to DRAM once.
// DRAM traffic ~ row offsets twice + X + records twice + S.X once (ncu: c3 5.9 GB against
// 14.3 GB for the gather).  The adds of one (bucket, column) entry run in no fixed order,
// so S.X equals the reference's to fp64 rounding (entries with one or two contributions --
// 97% of c3's -- are exact, a + b being commutative) and Z stays within the 1e-12 bar;
// csr_mode = 1 keeps the bit-exact gather.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

constexpr int kMaxParts = 1024;  // partitions (the accumulate queue's smem tables)

struct HashSrc {
    uint64_t cs_seed;
    FastMod mod;
    int64_t row0;
    uint64_t pow2_mask;  // B - 1 when B is a power of two (then mod B is a mask), else 0
};

__device__ __forceinline__ uint32_t row_bucket(const HashSrc& h, int64_t i, uint32_t* neg) {
    const uint64_t gi = (uint64_t)(h.row0 + i);
    *neg = cs_negative(h.cs_seed, gi);
    if (h.pow2_mask) return (uint32_t)(rng_draw(h.cs_seed, 2 * gi) & h.pow2_mask);
    return cs_bucket(h.cs_seed, gi, h.mod);
}

// 1. nonzeros per (partition, sub-cursor): sub = (row / tile) % nsub, as the scatter uses
// it.  Per-warp shared-memory histograms (u32), so a row's atomic only collides inside its
// warp, folded into the global counts once per CTA.
__global__ void __launch_bounds__(256) count_kernel(const int64_t* __restrict__ rowptr, int64_t n, HashSrc h, int pshift,
                                                    int nbins, int nsub, int tile_shift,
                                                    unsigned long long* __restrict__ counts,
                                                    uint32_t* __restrict__ rowinfo) {
    extern __shared__ uint32_t hist[];  // [8 warps][nbins]
    const int wid = threadIdx.x >> 5;
    for (int p = threadIdx.x; p < 8 * nbins; p += blockDim.x) hist[p] = 0;
    __syncthreads();
    uint32_t* my = hist + wid * nbins;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t neg;
        const uint32_t b = row_bucket(h, i, &neg);
        rowinfo[i] = b << 1 | neg;  // the scatter reads this instead of hashing again
        const uint32_t len = (uint32_t)(rowptr[i + 1] - rowptr[i]);
        if (len) atomicAdd(&my[(b >> pshift) * nsub + (int)((i >> tile_shift) & (nsub - 1))], len);
    }
    __syncthreads();
    for (int p = threadIdx.x; p < nbins; p += blockDim.x) {
        unsigned long long t = 0;
        for (int w = 0; w < 8; ++w) t += hist[w * nbins + p];
        if (t) red_add(&counts[p], t);
    }
}

// exclusive scan of the (partition, sub) counts into the write cursors; per-partition
// record counts for the accumulate pass (one CTA of 1024 threads, nbins <= 2048)
__global__ void cursor_kernel(const unsigned long long* __restrict__ counts, int nbins, int nsub,
                              unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ pcount) {
    __shared__ unsigned long long s[2048];
    const int t = threadIdx.x;
    for (int k = t; k < 2048; k += 1024) s[k] = k < nbins ? counts[k] : 0;
    __syncthreads();
    for (int o = 1; o < 2048; o <<= 1) {
        unsigned long long v0 = t >= o ? s[t - o] : 0, v1 = t + 1024 >= o ? s[t + 1024 - o] : 0;
        __syncthreads();
        s[t] += v0;
        s[t + 1024] += v1;
        __syncthreads();
    }
    for (int k = t; k < nbins; k += 1024) cursor[k] = s[k] - counts[k];
    for (int p = t; p < nbins / nsub; p += 1024) {
        const int k = (p + 1) * nsub - 1;
        pcount[p] = s[k] - (s[p * nsub] - counts[p * nsub]);
    }
}

// 2. records.  A CTA of kScThreads takes a tile of kTile consecutive rows (kGroups per
// lane).  Phase 1: a lane holds a row (offsets, bucket, sign, partition) and reserves len
// places in its partition's run for this tile with one shared-memory atomic; one global
// atomic per (partition, sub-cursor) then places the tile's runs (kSub cursors per partition,
// tile t using sub-cursor t % kSub, keep the cursors from serializing in one L2 slice).
// Phase 2: each lane copies its row's nonzeros into the tile's shared-memory staging area,
// grouped by partition (rows are short here, and a warp's consecutive rows span a few lines
// that its later steps reuse from L1).  Phase 3: one warp per partition stores the run out
// coalesced (direct 4-byte stores from phase 2 touch up to 32 partitions per instruction:
// 2.6 ms on c3 against ~0.5 ms of streaming).  A tile with more records than the staging
// area stores from phase 2 directly.
constexpr int kScThreads = 256;
constexpr int kStage = 4096;  // staged records per tile
constexpr int kSubMax = 8;
template <typename TV, typename TI, int kGroups, int kMinB>
__global__ void __launch_bounds__(kScThreads, kMinB) scatter_kernel(const int64_t* __restrict__ rowptr,
                                                             const TI* __restrict__ cols, const TV* __restrict__ vals,
                                                             int64_t n, const uint32_t* __restrict__ rowinfo, int pshift,
                                                             int nparts, int nsub, int cbits,
                                                             unsigned long long* __restrict__ cursor,
                                                             uint32_t* __restrict__ rkey, float* __restrict__ rval) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* s_key = (uint32_t*)smem_raw;                                // kStage
    float* s_val = (float*)(s_key + kStage);                               // kStage
    unsigned long long* s_gbase = (unsigned long long*)(s_val + kStage);  // nparts
    uint32_t* s_cnt = (uint32_t*)(s_gbase + nparts);                       // nparts
    uint32_t* s_off = s_cnt + nparts;                                      // nparts (exclusive scan)
    uint16_t* s_part = (uint16_t*)(s_off + nparts);                        // kStage: partition of each staged record
    __shared__ uint32_t s_total;
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int kTile = kScThreads * kGroups;  // rows per tile
    const int64_t ntiles = (n + kTile - 1) / kTile;
    // the next tile's row offsets and row records are loaded while this tile is staged and
    // stored (the tile's phases are separated by barriers, so unhidden load latency at the
    // start of every tile held the kernel at ~2.5 TB/s)
    int64_t nrb[kGroups], nre[kGroups];
    uint32_t nbk[kGroups];
    auto prefetch = [&](int64_t t) {
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
            const int64_t row = t * kTile + g * kScThreads + threadIdx.x;
            nrb[g] = nre[g] = 0;
            nbk[g] = 0;
            if (t < ntiles && row < n) {
                nrb[g] = rowptr[row];
                nre[g] = rowptr[row + 1];
                nbk[g] = __ldcs(rowinfo + row);
            }
        }
    };
    prefetch(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int p = threadIdx.x; p < nparts; p += kScThreads) s_cnt[p] = 0;
        __syncthreads();
        int64_t rb[kGroups];
        int len[kGroups];
        uint32_t bk[kGroups], off[kGroups];
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
            rb[g] = nrb[g];
            len[g] = (int)(nre[g] - nrb[g]);
            bk[g] = nbk[g];
            off[g] = 0;
            if (len[g]) off[g] = atomicAdd(&s_cnt[(bk[g] >> 1) >> pshift], (uint32_t)len[g]);
        }
        prefetch(tile + gridDim.x);
        __syncthreads();
        const int sub = (int)(tile & (nsub - 1));
        if (wid == 0) {  // staging offsets: exclusive scan of the partition counts
            uint32_t run = 0;
            for (int p0 = 0; p0 < nparts; p0 += 32) {
                const int p = p0 + (int)lane;
                const uint32_t c = p < nparts ? s_cnt[p] : 0u;
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                    if ((int)lane >= o) incl += t;
                }
                if (p < nparts) s_off[p] = run + incl - c;
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) s_total = run;
        }
        __syncthreads();
        const bool staged = s_total <= (uint32_t)kStage;
        // the tile's global reservations (needed only by the write-out) are claimed by the
        // last warps while the others already copy their rows: the atomics' round trip to the
        // cursors overlaps the nonzeros' DRAM loads instead of preceding them (for an unstaged
        // tile the places are needed now, so every thread waits for them)
        for (int p = (int)threadIdx.x - (kScThreads - nparts % kScThreads) % kScThreads; p < nparts;
             p += kScThreads)
            if (p >= 0 && s_cnt[p]) s_gbase[p] = atomicAdd(&cursor[p * nsub + sub], (unsigned long long)s_cnt[p]);
        if (!staged) __syncthreads();
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
            const uint32_t b = bk[g] >> 1;
            const uint32_t p = b >> pshift;
            const uint32_t kb = b << cbits;
            const bool neg = bk[g] & 1u;
            if (staged) {
                const uint32_t slot = s_off[p] + off[g];
                // four nonzeros' loads in flight per lane before their stores (c3 rows hold
                // 2.56 on average, so most rows take one step)
                for (int k0 = 0; k0 < len[g]; k0 += 4) {
                    float x[4];
                    uint32_t c[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const bool ok = k0 + u < len[g];
                        x[u] = ok ? (float)__ldg(vals + rb[g] + k0 + u) : 0.0f;
                        c[u] = ok ? (uint32_t)__ldg(cols + rb[g] + k0 + u) : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (k0 + u < len[g]) {
                            s_key[slot + k0 + u] = kb | c[u];
                            s_val[slot + k0 + u] = neg ? -x[u] : x[u];
                            s_part[slot + k0 + u] = (uint16_t)p;
                        }
                    }
                }
            } else {
                const unsigned long long dst = s_gbase[p] + off[g];
                for (int k = 0; k < len[g]; ++k) {
                    const float x = (float)__ldg(vals + rb[g] + k);
                    rkey[dst + k] = kb | (uint32_t)__ldg(cols + rb[g] + k);
                    rval[dst + k] = neg ? -x : x;
                }
            }
        }
        __syncthreads();
        if (staged) {
            // flat over the staged records (all lanes busy; consecutive records of one
            // partition go to consecutive places, so the stores coalesce within its run) --
            // a warp per partition left most lanes idle in its ~40-record runs (31% of the
            // kernel's instructions on c3)
            const uint32_t total = s_total;
            for (uint32_t i = threadIdx.x; i < total; i += kScThreads) {
                const uint32_t p = s_part[i];
                const unsigned long long dst = s_gbase[p] + (i - s_off[p]);
                __stcs(rkey + dst, s_key[i]);
                __stcs(rval + dst, s_val[i]);
            }
        }
        __syncthreads();
    }
}

// 3. fp64 RED into S.X (row-major B x d).  One persistent kernel works through a queue of
// items in the order Z0 Z1 R0 Z2 R1 ... Z(P-1) R(P-2) R(P-1), where Z(p) zero-fills S.X slice
// p (64 KB per item) and R(p) adds partition p's records (kRecItem per item).  R(p) items
// wait for Z(p) to complete (a per-partition counter), which was queued two groups earlier,
// so they rarely wait.  The zero stores leave the slice's lines valid in L2, so the adds hit
// L2 instead of reading zeros back from DRAM (a cudaMemset of S.X first cost 0.54 GB of
// extra DRAM reads on c3 and held the adds at ~125 G/s).
constexpr int kZeroItem = 8192;   // doubles zeroed per Z item
constexpr int kRecItem = 4096;    // records per R item
constexpr int kAccThreads = 256;

__global__ void __launch_bounds__(kAccThreads) accumulate_kernel(const uint32_t* __restrict__ rkey,
                                                                  const float* __restrict__ rval,
                                                                  const unsigned long long* __restrict__ pcount,
                                                                  int nparts, int pshift, int64_t B, int cbits, int64_t d,
                                                                  double* __restrict__ sx,
                                                                  unsigned int* __restrict__ next_item,
                                                                  unsigned int* __restrict__ zdone, int zero_inline) {
    __shared__ unsigned long long s_pstart[kMaxParts + 1];  // record start of each partition
    __shared__ unsigned int s_gstart[2 * kMaxParts + 1];    // first item of each queue group
    __shared__ unsigned int s_item;
    const int ngroups = 2 * nparts;
    const int64_t W = (int64_t)1 << pshift;
    auto zitems = [&](int p) -> unsigned {
        if (!zero_inline) return 0u;  // S.X zero-filled before the launch
        const int64_t e = (min(B, (p + 1) * W) - p * W) * d;
        return (unsigned)((e + kZeroItem - 1) / kZeroItem);
    };
    // queue group k: 0 -> Z0, 1 -> Z1, then R(k/2 - 1) for even k >= 2, Z(k/2 + ...) ...:
    // the sequence Z0, Z1, R0, Z2, R1, Z3, ..., Z(P-1), R(P-2), R(P-1)
    auto group = [&](int k, bool* isz) -> int {
        if (k < 2 && k < nparts) {
            *isz = true;
            return k;
        }
        if (nparts == 1) {
            *isz = false;
            return 0;
        }
        const int j = k - 2;  // pairs (R(j/2), Z(j/2 + 2)) while Z remain
        const int r = j / 2;
        if ((j & 1) == 0) {
            *isz = false;
            return r;
        }
        if (r + 2 < nparts) {
            *isz = true;
            return r + 2;
        }
        *isz = false;  // past the last Z: the remaining R groups
        return r + 1;
    };
    if (threadIdx.x == 0) {
        unsigned long long acc = 0;
        for (int p = 0; p < nparts; ++p) {
            s_pstart[p] = acc;
            acc += pcount[p];
        }
        s_pstart[nparts] = acc;
        unsigned g = 0;
        // walk the sequence: its length is 2P groups (P Z's and P R's)
        for (int k = 0; k < ngroups; ++k) {
            s_gstart[k] = g;
            bool isz;
            const int p = group(k, &isz);
            g += isz ? zitems(p) : (unsigned)((s_pstart[p + 1] - s_pstart[p] + kRecItem - 1) / kRecItem);
        }
        s_gstart[ngroups] = g;
    }
    __syncthreads();
    const unsigned total = s_gstart[ngroups];
    const uint32_t cmask = (1u << cbits) - 1u;
    // the next item is claimed while the current one runs: the claim's round trip to the
    // (contended) counter stays off the critical path
    if (threadIdx.x == 0) s_item = atomicAdd(next_item, 1u);
    __syncthreads();
    unsigned it = s_item;
    for (;;) {
        __syncthreads();
        if (it >= total) break;
        unsigned nxt = 0;
        if (threadIdx.x == 0) nxt = atomicAdd(next_item, 1u);
        int lo = 0, hi = ngroups;  // group: last k with s_gstart[k] <= it
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_gstart[mid] <= it) lo = mid; else hi = mid;
        }
        bool isz;
        const int p = group(lo, &isz);
        const unsigned sub = it - s_gstart[lo];
        if (isz) {
            const int64_t base = p * W * d + (int64_t)sub * kZeroItem;
            const int64_t end = min((int64_t)min(B, (p + 1) * W) * d, base + kZeroItem);
            for (int64_t e = base + threadIdx.x * 2; e < end; e += kAccThreads * 2) {
                if (e + 1 < end)
                    *reinterpret_cast<double2*>(sx + e) = make_double2(0.0, 0.0);
                else
                    sx[e] = 0.0;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(&zdone[p], 1u);
            }
        } else {
            if (threadIdx.x == 0) {
                const unsigned need = zitems(p);
                while (true) {
                    unsigned v;
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(zdone + p) : "memory");
                    if (v >= need) break;
                    __nanosleep(200);
                }
            }
            __syncthreads();
            const unsigned long long r0 = s_pstart[p] + (unsigned long long)sub * kRecItem;
            const unsigned long long r1 = min(s_pstart[p + 1], r0 + kRecItem);
            // all of this thread's records in flight before the adds: with the loads issued one
            // or four at a time the kernel sat on their DRAM latency (long_scoreboard 78%)
            constexpr int kPer = kRecItem / kAccThreads;
            uint32_t kk[kPer];
            float vv[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const unsigned long long e = r0 + threadIdx.x + (unsigned long long)u * kAccThreads;
                kk[u] = 0;
                vv[u] = 0.0f;
                if (e < r1) {
                    kk[u] = __ldcs(rkey + e);
                    vv[u] = __ldcs(rval + e);
                }
            }
            // (validity by position: with bucket bits + column bits = 32 every key value,
            // 0xffffffff included, is a record)
#pragma unroll
            for (int u = 0; u < kPer; ++u)
                if (r0 + threadIdx.x + (unsigned long long)u * kAccThreads < r1)
                    red_add(sx + (int64_t)(kk[u] >> cbits) * d + (kk[u] & cmask), (double)vv[u]);
        }
        if (threadIdx.x == 0) s_item = nxt;
        __syncthreads();
        it = s_item;
    }
}

} // namespace

// Shapes the record path covers: a seeded map (hash = index function of the seed), fp32
// values (records carry fp32 -- fp64 inputs take the gather), key = bucket:column in 32 bits.
bool csr_atomic_applies(const cgx_ctx* ctx, const cgx_xform* xf, int64_t n, int64_t d, int64_t nnz, int dtype) {
    if (ctx->opt_csr_mode == 1 || ctx->opt_csr_mode == 2) return false;
    if (!xf->seeded_map || xf->grows || dtype != CGX_F32 || nnz <= 0 || d < 1) return false;
    int bbits = 0, cbits = 0;
    while (((int64_t)1 << bbits) < xf->B) ++bbits;
    while (((int64_t)1 << cbits) < d) ++cbits;
    if (bbits + cbits > 32) return false;
    if (ctx->opt_csr_mode == 3) return true;
    // auto: short rows, where the gather pays three random DRAM reads per few nonzeros
    return (double)nnz / (double)n < 8.0 && xf->B * d >= ((int64_t)1 << 22) && nnz >= ((int64_t)1 << 22);
}

template <typename TI>
void run_atomic(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const TI* cols, const float* vals, int64_t n,
                int64_t d, int64_t nnz, double* sx, cudaStream_t s) {
    int cbits = 0;
    while (((int64_t)1 << cbits) < d) ++cbits;
    // partition slice <= ~16 MB of S.X: pshift = log2(buckets per partition)
    const int64_t slice_target = ctx->opt_csr_slice_mb << 20;
    int pshift = 0;
    while (((int64_t)2 << pshift) * d * 8 <= slice_target && ((int64_t)1 << pshift) < xf->B) ++pshift;
    int nparts = (int)((xf->B + ((int64_t)1 << pshift) - 1) >> pshift);
    while (nparts > kMaxParts) {
        ++pshift;
        nparts = (int)((xf->B + ((int64_t)1 << pshift) - 1) >> pshift);
    }
    const uint64_t Bu = (uint64_t)xf->B;
    const HashSrc h{xf->map_seed, FastMod(Bu), xf->row0, (Bu & (Bu - 1)) == 0 ? Bu - 1 : 0};
    int nsub = 1;  // sub-cursors per partition: a power of two, nparts * nsub <= 2048
    while (nsub * 2 <= kSubMax && nparts * nsub * 2 <= 2048) nsub *= 2;
    const int nbins = nparts * nsub;
    unsigned long long* counts = (unsigned long long*)ctx->part[0].get(sizeof(unsigned long long) * 3 * 2048);
    unsigned long long* cursor = counts + 2048;
    unsigned long long* pcount = cursor + 2048;
    uint32_t* rkey = (uint32_t*)ctx->part[1].get(sizeof(uint32_t) * (size_t)nnz);
    float* rval = (float*)ctx->part[2].get(sizeof(float) * (size_t)nnz);
    CGX_CUDA(cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * (size_t)nbins, s));
    const int grid = ctx->num_sms * 8;
    const size_t csm = sizeof(uint32_t) * 8 * (size_t)nbins;
    CGX_CUDA(cudaFuncSetAttribute(count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm));
    uint32_t* rowinfo = (uint32_t*)ctx->part[4].get(sizeof(uint32_t) * (size_t)n);
    // scatter: 4 rows per lane per 1024-row tile, 4 CTAs per SM (c3: 1.15 ms; 2 rows x 6 CTAs
    // measured 1.49 ms, 4 x 3 CTAs 1.27 ms)
    auto sk = scatter_kernel<float, TI, 4, 4>;
    const int groups = 4;
    const size_t smem = (sizeof(uint32_t) + sizeof(float) + sizeof(uint16_t)) * kStage +
                        (sizeof(unsigned long long) + 2 * sizeof(uint32_t)) * (size_t)nparts;
    const int tile_rows = kScThreads * groups;
    int tile_shift = 0;
    while ((1 << tile_shift) < tile_rows) ++tile_shift;
    count_kernel<<<grid, 256, csm, s>>>(rowptr, n, h, pshift, nbins, nsub, tile_shift, counts, rowinfo);
    cursor_kernel<<<1, 1024, 0, s>>>(counts, nbins, nsub, cursor, pcount);
    CGX_CUDA(cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sk, kScThreads, smem));
    const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
    const int sgrid = (int)std::min<int64_t>(ntiles, (int64_t)ctx->num_sms * std::max(per_sm, 1));
    sk<<<sgrid, kScThreads, smem, s>>>(rowptr, cols, vals, n, rowinfo, pshift, nparts, nsub, cbits, cursor, rkey, rval);
    unsigned int* next_item = (unsigned int*)ctx->part[3].get(sizeof(unsigned int) * (kMaxParts + 1));
    unsigned int* zdone = next_item + 1;
    CGX_CUDA(cudaMemsetAsync(next_item, 0, sizeof(unsigned int) * (size_t)(nparts + 1), s));
    // (a grid-stride kernel over all records after a cudaMemset of S.X measured 1.69 ms on c3
    // against 1.45 ms for this queue: its warps drift across partitions and the L2 thrashes)
    int acc_per_sm = 0;
    CGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&acc_per_sm, accumulate_kernel, kAccThreads, 0));
    const int zero_inline = ctx->opt_csr_zero == 1;
    if (!zero_inline) CGX_CUDA(cudaMemsetAsync(sx, 0, sizeof(double) * (size_t)(xf->B * d), s));
    accumulate_kernel<<<ctx->num_sms * std::max(acc_per_sm, 1), kAccThreads, 0, s>>>(
        rkey, rval, pcount, nparts, pshift, xf->B, cbits, d, sx, next_item, zdone, zero_inline);
    count_launch(ctx, 4);
    check_launch("sketch_csr_atomic");
}

void launch_sketch_csr_atomic(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols, int idx_type,
                              const void* vals, int64_t n, int64_t d, int64_t nnz, double* sx, cudaStream_t s) {
    if (idx_type == CGX_I32)
        run_atomic<int32_t>(ctx, xf, rowptr, (const int32_t*)cols, (const float*)vals, n, d, nnz, sx, s);
    else
        run_atomic<int64_t>(ctx, xf, rowptr, (const int64_t*)cols, (const float*)vals, n, d, nnz, sx, s);
}

} // namespace cgx
