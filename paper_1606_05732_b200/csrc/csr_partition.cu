// csr_partition.cu -- S.X for short-row CSR X by a stable two-level partition of the
// nonzeros (the "bucket-sorted transposition" of X), bit-identical to the reference.
//
// Replaces the same reference loop as sketch_csr.cu (src/sketch.cpp:68-113: rows in
// ascending order, each row's nonzeros in stored order, out(hash[i], j) += sign[i]*v).
// The gather in sketch_csr.cu reads every row at a random place: three reads (offsets,
// columns, values) of a few bytes each per row, which on rows of ~3 nonzeros costs ~10x
// the useful bytes in DRAM fetch granules.  Here every pass streams:
//
//   A1  rows, tile by tile: per-tile nonzero counts of each coarse bin `hi`;
//   A3  rows again: each row's nonzeros are copied, in row order, into its coarse bin,
//       as (key, value) pairs -- a stable partition; a CTA writes all of its runs within
//       microseconds, so L2 merges the partial sectors before they reach DRAM;
//   B1  within each coarse bin: per-tile counts of the fine digit `lo`;
//   B3  the stable partition of each coarse bin by `lo`, keys narrowed to 16 bits;
//   C   one warp per final bin F = (bucket group g, column slice cs): its nonzeros
//       arrive in ascending (row, position) order and are added, in that order, into an
//       SB x CS fp64 tile in shared memory (same-slot lanes serialized by rank), which
//       is then written to S.X rows g*SB.. at columns cs*CS.. (coalesced).
//
// Both partitions are stable, so every S.X(b, j) receives its contributions in exactly
// the reference's order: bit-identical, deterministic, no atomics on values.
// Bins: F = (b >> sb_log) << ncs_log | (col >> cs_log);  hi = F >> L;  lo = F & (2^L-1).
// Because 2^L is a multiple of the slice count, `hi` depends on the bucket only, so pass
// A moves whole rows.
#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

constexpr unsigned kFull = 0xffffffffu;

struct RowKeys {  // bucket | neg<<31 of local row i
    const uint32_t* rowkey;  // explicit maps: precomputed per row; null for seeded maps
    uint64_t cs_seed;
    FastMod mod;
    int64_t row0;
    __device__ __forceinline__ uint32_t operator()(int64_t i) const {
        if (rowkey) return __ldg(rowkey + i);
        const uint64_t gi = (uint64_t)(row0 + i);
        return cs_bucket(cs_seed, gi, mod) | (cs_negative(cs_seed, gi) << 31);
    }
};

struct Plan {
    int sb_log, cs_log, ncs_log, L;
    int NH;       // coarse bins
    int64_t R;    // rows per pass-A CTA tile
    int64_t NT;   // pass-A tiles
    int64_t TE;   // entries per pass-B CTA tile
    int64_t NTB;  // pass-B grid (upper bound on tiles)
    int kshift;   // sb_log + cs_log + 1: position of lo in the pass-A key
    int hbits;    // bits of a coarse bin index (NH <= 2^hbits)
};

__device__ __forceinline__ uint32_t hi_of(uint32_t b, const Plan& p) { return (b >> p.sb_log) >> (p.L - p.ncs_log); }

// ------------------------------------------------------------------ block-level helpers
// Inclusive scan of v over the 256 threads of the CTA; `total` gets the CTA sum.
// wtot: 8 words of shared scratch.  Contains __syncthreads (call uniformly).
__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, uint32_t* wtot, uint32_t& total) {
    const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t x = (uint32_t)warp_incl_scan((int)v, lane);
    if (lane == 31) wtot[w] = x;
    __syncthreads();
    uint32_t off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t t = wtot[i];
        off += i < (int)w ? t : 0u;
        tot += t;
    }
    __syncthreads();
    total = tot;
    return x + off;
}

// off[0..nb] = exclusive scan of cnt[0..nb) (nb <= 1024), off[nb] = total.
__device__ __forceinline__ void block_excl_scan_bins(const uint32_t* cnt, uint32_t* off, int nb, uint32_t* wtot) {
    const int t = threadIdx.x, c = (nb + 255) / 256;
    const int b0 = min(nb, t * c), b1 = min(nb, b0 + c);
    uint32_t s = 0;
    for (int b = b0; b < b1; ++b) s += cnt[b];
    uint32_t tot;
    uint32_t run = block_incl_scan(s, wtot, tot) - s;
    for (int b = b0; b < b1; ++b) {
        off[b] = run;
        run += cnt[b];
    }
    if (t == 0) off[nb] = tot;
    __syncthreads();
}

// ---------------------------------------------------------------------------- pass A
// CTA tile = R consecutive rows.  cntA[hi * NT + tile] = nonzeros of the tile in bin hi.
__global__ void __launch_bounds__(256) part_count_rows(const int64_t* __restrict__ rowptr, int64_t n, RowKeys rk,
                                                       Plan p, uint32_t* __restrict__ cntA) {
    extern __shared__ uint32_t hs[];
    const int64_t tile = blockIdx.x;
    for (int j = threadIdx.x; j < p.NH; j += 256) hs[j] = 0;
    __syncthreads();
    const int64_t r0 = tile * p.R, r1 = min(n, r0 + p.R);
    for (int64_t i = r0 + threadIdx.x; i < r1; i += 256) {
        const uint32_t len = (uint32_t)(rowptr[i + 1] - rowptr[i]);
        if (len) atomicAdd(&hs[hi_of(rk(i) & kRowMask, p)], len);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < p.NH; j += 256) cntA[(int64_t)j * p.NT + tile] = hs[j];
}

constexpr int kRowsPerLane = 8;     // pass A: rows per lane (warp chunk = 256 rows)
constexpr int kCapA = 8192;         // pass A: staged nonzeros per tile
constexpr int kCapB = 4096;         // pass B: entries per CTA tile
constexpr int kEntPerLane = kCapB / 256;  // pass B: entries per lane (warp chunk = 512)

// Stable partition of the tile's rows into coarse bins, written straight to their final
// positions.  Warp w owns rows [r0 + 256w, r0 + 256w + 256): every lane holds 8 of them
// (rounds) in registers.  Phase 1 counts each warp's nonzeros per bin; the CTA turns the
// counts into per-(warp, bin) global offsets (bin runs of a tile are ordered by warp, so
// the order is rows ascending); phase 2 gives each row its run position (rows of one bin
// inside a round by lane order, via match_any_bits); phase 3 copies each round's input
// range with coalesced loads into a shared-memory image of the tile's bin runs, which
// then leaves run by run in coalesced bursts (scattered 4 B stores would be bound by the
// L2 sector-write rate).
template <typename TV, typename TI>
__global__ void __launch_bounds__(256) part_scatter_rows(const int64_t* __restrict__ rowptr,
                                                         const TI* __restrict__ cols, const TV* __restrict__ vals,
                                                         int64_t n, RowKeys rk, Plan p, const uint32_t* __restrict__ posA,
                                                         uint32_t* __restrict__ keyA, TV* __restrict__ valA) {
    extern __shared__ __align__(16) uint32_t sa[];
    const int NH = p.NH;
    const unsigned t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t* offw = sa;                 // [8][NH] per-warp bin counts, then offsets
    uint32_t* wl = offw + 8 * NH;        // [8][32] leader scratch
    uint32_t* soff = wl + 256;           // [NH+1] staging offsets of the tile's bin runs
    uint32_t* gbase = soff + NH + 1;     // [NH] global start of the tile's bin runs
    uint32_t* tot = gbase + NH;          // [NH] nonzeros of the tile per bin
    uint32_t* wtot = tot + NH;           // [8]
    TV* sval = reinterpret_cast<TV*>((reinterpret_cast<uintptr_t>(wtot + 8) + 15) & ~uintptr_t(15));  // [kCapA]
    uint32_t* skey = reinterpret_cast<uint32_t*>(sval + kCapA);                                       // [kCapA]
    const int64_t tile = blockIdx.x;
    for (int j = t; j < 8 * NH; j += 256) offw[j] = 0;
    __syncthreads();
    const int64_t wr0 = tile * p.R + (int64_t)w * 32 * kRowsPerLane;
    uint32_t key[kRowsPerLane], len[kRowsPerLane], hi[kRowsPerLane];
    int64_t rs0 = 0;
#pragma unroll
    for (int u = 0; u < kRowsPerLane; ++u) {
        const int64_t i = wr0 + u * 32 + lane;
        const bool ok = i < n;
        const int64_t rs = ok ? rowptr[i] : 0;
        len[u] = ok ? (uint32_t)(rowptr[i + 1] - rs) : 0u;
        if (u == 0) rs0 = rs;
        key[u] = ok ? rk(i) : 0u;
        hi[u] = ok ? hi_of(key[u] & kRowMask, p) : 0xffffffffu;
    }
    const int64_t in0 = __shfl_sync(kFull, rs0, 0);  // the warp's rows are consecutive
    uint32_t* cw = offw + w * NH;
#pragma unroll
    for (int u = 0; u < kRowsPerLane; ++u)
        if (len[u]) atomicAdd(&cw[hi[u]], len[u]);
    __syncthreads();
    for (int h = t; h < NH; h += 256) {
        uint32_t c = 0;
#pragma unroll
        for (int v = 0; v < 8; ++v) c += offw[v * NH + h];
        tot[h] = c;
        gbase[h] = posA[(int64_t)h * p.NT + tile];
    }
    __syncthreads();
    block_excl_scan_bins(tot, soff, NH, wtot);
    // staged (the tile fits kCapA): runs are assembled in shared memory and leave bin by
    // bin in coalesced bursts; otherwise rows are written straight to their destinations
    const bool staged = soff[NH] <= (uint32_t)kCapA;
    for (int h = t; h < NH; h += 256) {  // per-(warp, bin) offsets
        uint32_t run = staged ? soff[h] : gbase[h];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            const uint32_t c = offw[v * NH + h];
            offw[v * NH + h] = run;
            run += c;
        }
    }
    __syncthreads();
    uint32_t* wlw = wl + w * 32;
    const uint32_t lo_mask = (1u << p.L) - 1u;
    auto pack = [&](uint32_t kj, uint32_t col) {  // pass-A key of nonzero (row key kj, column col)
        const uint32_t b = kj & kRowMask;
        const uint32_t F = ((b >> p.sb_log) << p.ncs_log) | (col >> p.cs_log);
        return ((F & lo_mask) << p.kshift) | ((b & ((1u << p.sb_log) - 1u)) << (p.cs_log + 1)) |
               ((col & ((1u << p.cs_log) - 1u)) << 1) | (kj >> 31);
    };
    constexpr int kW = 4;            // waves of loads in flight in the copy
    const unsigned lt = (1u << lane) - 1u;
    uint32_t base = 0;               // nonzeros of the warp's earlier rounds
#pragma unroll
    for (int u = 0; u < kRowsPerLane; ++u) {
        // ---- phase 2: run position of each row (rows of a bin in lane order)
        const bool ok = hi[u] != 0xffffffffu;
        wlw[lane] = len[u];
        __syncwarp();
        const unsigned grp = match_any_bits(ok ? hi[u] : 1u << p.hbits, p.hbits + 1);
        if (ok && (int)lane == __ffs(grp) - 1) {
            uint32_t c = cw[hi[u]];
            for (unsigned m = grp; m; m &= m - 1) {
                const int j = __ffs(m) - 1;
                const uint32_t lj = wlw[j];
                wlw[j] = c;
                c += lj;
            }
            cw[hi[u]] = c;
        }
        __syncwarp();
        const uint32_t dst = wlw[lane];
        const uint32_t incl = (uint32_t)warp_incl_scan((int)len[u], lane);
        const int64_t rs = in0 + base + incl - len[u];
        base += __shfl_sync(kFull, incl, 31);
        // ---- phase 3: copy the round's input range [rs_0, rs_0 + T), coalesced.  The row of
        // item q is the last nonzero row starting at or before q: row starts of each wave
        // come from one OR-reduction, and a per-round table maps start rank -> lane.
        const uint32_t T = __shfl_sync(kFull, incl, 31);
        const int64_t rbase = __shfl_sync(kFull, rs, 0);
        const uint32_t excl = incl - len[u];
        const unsigned nzmask = __ballot_sync(kFull, len[u] != 0);
        __syncwarp();  // every lane has read its dst from wlw
        if (len[u]) wlw[__popc(nzmask & lt)] = lane;  // start rank -> lane
        __syncwarp();
        uint32_t kbase = 0;  // nonzero rows started in earlier waves
        for (uint32_t q0 = 0; q0 < T; q0 += 32 * kW) {
            uint32_t c[kW];
            TV v[kW];
#pragma unroll
            for (int k = 0; k < kW; ++k) {
                const uint32_t q = q0 + k * 32 + lane;
                c[k] = q < T ? (uint32_t)cols[rbase + q] : 0u;
                v[k] = q < T ? vals[rbase + q] : TV(0);
            }
#pragma unroll
            for (int k = 0; k < kW; ++k) {
                const uint32_t wq = q0 + k * 32;
                if (wq >= T) break;
                const bool starts_here = len[u] != 0 && (excl >> 5) == (wq >> 5);
                const unsigned starts = __reduce_or_sync(kFull, starts_here ? 1u << (excl & 31) : 0u);
                const uint32_t r = kbase + __popc(starts & (lt | (1u << lane))) - 1;
                kbase += __popc(starts);
                const int j = (int)wlw[r & 31];
                const uint32_t ej = __shfl_sync(kFull, excl, j);
                const uint32_t dj = __shfl_sync(kFull, dst, j);
                const uint32_t kj = __shfl_sync(kFull, key[u], j);
                const uint32_t q = wq + lane;
                if (q < T) {
                    const uint32_t o = dj + (q - ej);
                    if (staged) {
                        skey[o] = pack(kj, c[k]);
                        sval[o] = v[k];
                    } else {
                        keyA[o] = pack(kj, c[k]);
                        valA[o] = v[k];
                    }
                }
            }
        }
        __syncwarp();
    }
    if (staged) {  // flush: warp w takes bins w, w+8, ...
        __syncthreads();
        for (int h = w; h < NH; h += 8) {
            const uint32_t a = soff[h], e = soff[h + 1], g = gbase[h];
            for (uint32_t q = a + lane; q < e; q += 32) {
                keyA[g + (q - a)] = skey[q];
                valA[g + (q - a)] = sval[q];
            }
        }
    }
}

// Pass-B tile bookkeeping (one block): coarse bin h spans [seg[h], seg[h+1]) of the pass-A
// output; it is cut into ceil(size/kCapB) CTA tiles numbered from tstart[h].
__global__ void part_tiles(const uint32_t* __restrict__ posA, Plan p, uint32_t nnz, uint32_t* __restrict__ seg,
                           uint32_t* __restrict__ tstart) {
    __shared__ uint32_t s[1024];
    const int h = threadIdx.x;
    uint32_t nt = 0;
    if (h < p.NH) {
        const uint32_t a = posA[(int64_t)h * p.NT];
        const uint32_t e = h + 1 < p.NH ? posA[(int64_t)(h + 1) * p.NT] : nnz;
        seg[h] = a;
        nt = (e - a + kCapB - 1) / kCapB;
    }
    s[h] = nt;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive block scan
        const uint32_t v = h >= o ? s[h - o] : 0u;
        __syncthreads();
        s[h] += v;
        __syncthreads();
    }
    if (h < p.NH) tstart[h + 1] = s[h];
    if (h == 0) {
        tstart[0] = 0;
        seg[p.NH] = nnz;
    }
}

struct TileB {
    int h;
    int64_t k, nt;
    uint32_t e0, e1;
};

// CTA tile gt -> (coarse bin, tile within it, entry range); false past the last tile
__device__ __forceinline__ bool tile_b(const uint32_t* ts, const uint32_t* seg, const Plan& p, int64_t gt, TileB& t) {
    if (gt >= (int64_t)ts[p.NH]) return false;
    int lo = 0, hi = p.NH - 1;  // last h with ts[h] <= gt
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((int64_t)ts[mid] <= gt) lo = mid;
        else hi = mid - 1;
    }
    t.h = lo;
    t.k = gt - ts[lo];
    t.nt = (int64_t)ts[lo + 1] - ts[lo];
    t.e0 = seg[lo] + (uint32_t)(t.k * kCapB);
    t.e1 = (uint32_t)min((int64_t)seg[lo + 1], (int64_t)t.e0 + kCapB);
    return true;
}

// ---------------------------------------------------------------------------- pass B
__global__ void __launch_bounds__(256) part_count_lo(const uint32_t* __restrict__ keyA, Plan p,
                                                     const uint32_t* __restrict__ seg, const uint32_t* __restrict__ ts,
                                                     uint32_t* __restrict__ cntB) {
    extern __shared__ uint32_t hs[];
    const int nlo = 1 << p.L;
    TileB tb;
    if (!tile_b(ts, seg, p, blockIdx.x, tb)) return;
    for (int j = threadIdx.x; j < nlo; j += 256) hs[j] = 0;
    __syncthreads();
    for (uint32_t e = tb.e0 + threadIdx.x; e < tb.e1; e += 256) atomicAdd(&hs[keyA[e] >> p.kshift], 1u);
    __syncthreads();
    const int64_t blk = (int64_t)ts[tb.h] * nlo;
    for (int j = threadIdx.x; j < nlo; j += 256) cntB[blk + (int64_t)j * tb.nt + tb.k] = hs[j];
}

// Stable partition of one pass-B tile (<= kCapB entries of one coarse bin) by the fine
// digit, written straight to the final positions; keys shrink to the 16 bits pass C
// needs.  Warp w owns entries [e0 + 512w, e0 + 512w + 512), 16 per lane held in
// registers: count per (warp, digit), CTA offsets, then per wave ranks by lane order.
template <typename TV>
__global__ void __launch_bounds__(256) part_scatter_lo(const uint32_t* __restrict__ keyA, const TV* __restrict__ valA,
                                                       Plan p, const uint32_t* __restrict__ seg,
                                                       const uint32_t* __restrict__ ts, const uint32_t* __restrict__ posB,
                                                       uint16_t* __restrict__ keyB, TV* __restrict__ valB) {
    extern __shared__ __align__(16) uint32_t sb_[];
    const int nlo = 1 << p.L;
    uint32_t* offw = sb_;               // [8][nlo] per-warp digit counts, then offsets
    uint32_t* soff = offw + 8 * nlo;    // [nlo+1] staging offsets of the tile's runs
    uint32_t* gbase = soff + nlo + 1;   // [nlo] global start of the tile's runs
    uint32_t* tot = gbase + nlo;        // [nlo]
    uint32_t* wtot = tot + nlo;         // [8]
    TV* sval = reinterpret_cast<TV*>((reinterpret_cast<uintptr_t>(wtot + 8) + 15) & ~uintptr_t(15));  // [kCapB]
    uint16_t* skey = reinterpret_cast<uint16_t*>(sval + kCapB);                                       // [kCapB]
    const unsigned t = threadIdx.x, lane = t & 31, w = t >> 5;
    const unsigned lt = (1u << lane) - 1u;
    TileB tb;
    if (!tile_b(ts, seg, p, blockIdx.x, tb)) return;
    for (int j = t; j < 8 * nlo; j += 256) offw[j] = 0;
    __syncthreads();
    const uint32_t we0 = tb.e0 + w * 32 * kEntPerLane;
    uint32_t key[kEntPerLane];
    TV v[kEntPerLane];
#pragma unroll
    for (int k = 0; k < kEntPerLane; ++k) {
        const uint32_t e = we0 + k * 32 + lane;
        key[k] = e < tb.e1 ? keyA[e] : 0xffffffffu;
        v[k] = e < tb.e1 ? valA[e] : TV(0);
    }
    uint32_t* cw = offw + w * nlo;
#pragma unroll
    for (int k = 0; k < kEntPerLane; ++k)
        if (key[k] != 0xffffffffu) atomicAdd(&cw[key[k] >> p.kshift], 1u);
    __syncthreads();
    const int64_t blk = (int64_t)ts[tb.h] * nlo;
    for (int l = t; l < nlo; l += 256) {
        uint32_t c = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) c += offw[u * nlo + l];
        tot[l] = c;
        gbase[l] = posB[blk + (int64_t)l * tb.nt + tb.k];
    }
    __syncthreads();
    block_excl_scan_bins(tot, soff, nlo, wtot);
    for (int l = t; l < nlo; l += 256) {  // per-(warp, digit) staging offsets
        uint32_t run = soff[l];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t c = offw[u * nlo + l];
            offw[u * nlo + l] = run;
            run += c;
        }
    }
    __syncthreads();
    const uint32_t low_mask = (1u << p.kshift) - 1u;
#pragma unroll
    for (int k = 0; k < kEntPerLane; ++k) {
        const bool ok = key[k] != 0xffffffffu;
        const uint32_t lo = ok ? key[k] >> p.kshift : 0xffffffffu;
        const unsigned grp = match_any_bits(ok ? lo : 1u << p.L, p.L + 1);
        const uint32_t dst = ok ? cw[lo] + __popc(grp & lt) : 0u;
        __syncwarp();
        if (ok && (int)lane == __ffs(grp) - 1) cw[lo] += __popc(grp);
        __syncwarp();
        if (ok) {
            skey[dst] = (uint16_t)(key[k] & low_mask);
            sval[dst] = v[k];
        }
    }
    __syncthreads();
    for (int l = w; l < nlo; l += 8) {  // flush run by run (coalesced)
        const uint32_t a = soff[l], e = soff[l + 1], g = gbase[l];
        for (uint32_t q = a + lane; q < e; q += 32) {
            keyB[g + (q - a)] = skey[q];
            valB[g + (q - a)] = sval[q];
        }
    }
}

// ---------------------------------------------------------------------------- pass C
__device__ __forceinline__ float neg_if(float v, uint32_t n) { return __int_as_float(__float_as_int(v) ^ (int)(n << 31)); }
__device__ __forceinline__ double neg_if(double v, uint32_t n) {
    return __longlong_as_double(__double_as_longlong(v) ^ ((long long)n << 63));
}

// One warp per final bin: its entries, in (row, position) order, added into an SB x CS
// fp64 tile in shared memory; same-slot lanes of a wave are applied in lane order.
// Loads run kU waves ahead of the adds.
template <typename TV>
__global__ void __launch_bounds__(256) part_accumulate(const uint16_t* __restrict__ keyB, const TV* __restrict__ valB,
                                                       Plan p, const uint32_t* __restrict__ ts,
                                                       const uint32_t* __restrict__ posB, int64_t posB_count,
                                                       uint32_t nnz, int64_t B, int64_t d, double* __restrict__ sx) {
    constexpr int kU = 8;
    extern __shared__ double acc_all[];
    const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int SB = 1 << p.sb_log, CS = 1 << p.cs_log;
    double* acc = acc_all + (size_t)wid * SB * CS;
    uint8_t* tag = reinterpret_cast<uint8_t*>(acc_all + (size_t)8 * SB * CS) + wid * SB * CS;
    const int64_t F = (int64_t)blockIdx.x * 8 + wid;
    const int64_t g = F >> p.ncs_log, csl = F & ((1 << p.ncs_log) - 1);
    if (g * SB >= B || csl * CS >= d) return;
    auto start_of = [&](int64_t f) -> uint32_t {  // first pass-B position of final bin f
        const int64_t h = f >> p.L, lo = f & ((1 << p.L) - 1);
        if (h >= p.NH) return nnz;
        const int64_t idx = (int64_t)ts[h] * (1 << p.L) + lo * ((int64_t)ts[h + 1] - ts[h]);
        return idx < posB_count ? posB[idx] : nnz;
    };
    const uint32_t e0 = start_of(F), e1 = start_of(F + 1);
    for (int j = lane; j < SB * CS; j += 32) acc[j] = 0.0;
    __syncwarp();
    for (uint32_t eb = e0; eb < e1; eb += 32 * kU) {
        uint32_t key[kU];
        TV v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t e = eb + u * 32 + lane;
            key[u] = e < e1 ? (uint32_t)keyB[e] : 0x10000u;  // past the bin's end
            v[u] = e < e1 ? valB[e] : TV(0);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (eb + u * 32 >= e1) break;
            const bool ok = key[u] < 0x10000u;
            const uint32_t slot = ok ? key[u] >> 1 : 0u;  // bl * CS + cl (10 bits)
            const double x = (double)neg_if(v[u], key[u] & 1u);
            double* a = acc + slot;
            // distinct slots (most waves): a byte tag per slot, written by every lane and read
            // back, shows whether any two lanes share a slot
            if (ok) tag[slot] = (uint8_t)lane;
            __syncwarp();
            const bool mine = !ok || tag[slot] == (uint8_t)lane;
            if (__all_sync(kFull, mine)) {
                if (ok) *a += x;
            } else {  // some slot twice: items of a slot in lane (= reference) order
                const unsigned grp = match_any_bits(ok ? slot : 1u << 10, 11);
                const unsigned rank = __popc(grp & lt);
                for (unsigned r = 0; __any_sync(kFull, ok && rank >= r); ++r) {
                    if (ok && rank == r) *a += x;
                    __syncwarp();
                }
            }
            __syncwarp();
        }
    }
    __syncwarp();
    const int64_t b0 = g * SB, c0 = csl * CS;
    const int nb = (int)min((int64_t)SB, B - b0), nc = (int)min((int64_t)CS, d - c0);
    for (int bl = 0; bl < nb; ++bl)
        for (int cl = lane; cl < nc; cl += 32) sx[(b0 + bl) * d + c0 + cl] = acc[bl * CS + cl];
}

// explicit maps: per-row bucket | neg from the transform's bucket-sorted perm
__global__ void rowkey_from_perm(const uint32_t* __restrict__ perm, const uint32_t* __restrict__ offsets, int64_t B,
                                 int64_t n, uint32_t* __restrict__ rowkey) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = B - 1;  // last bucket with offsets[b] <= k
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if ((int64_t)offsets[mid] <= k) lo = mid;
            else hi = mid - 1;
        }
        const uint32_t pe = perm[k];
        rowkey[pe & kRowMask] = (uint32_t)lo | (pe & kNegBit);
    }
}

int ceil_log2(int64_t v) {
    int l = 0;
    while (((int64_t)1 << l) < v) ++l;
    return l;
}

bool make_plan(int64_t n, int64_t B, int64_t d, int64_t nnz, Plan& p) {
    if (n <= 0 || d <= 0 || nnz <= 0 || nnz >= ((int64_t)1 << 32) - 1) return false;
    p.cs_log = std::min(5, ceil_log2(d));
    const int64_t ncs = (d + (1 << p.cs_log) - 1) >> p.cs_log;
    p.ncs_log = ceil_log2(ncs);
    p.sb_log = 10 - p.cs_log;  // SB x CS = 1024 fp64 = 8 KB of tile per warp
    const int64_t NG = (B + (1 << p.sb_log) - 1) >> p.sb_log;
    const int64_t NF = NG << p.ncs_log;
    const int fbits = ceil_log2(NF);
    p.L = std::max(p.ncs_log, (fbits + 1) / 2);
    p.NH = (int)((NF + ((int64_t)1 << p.L) - 1) >> p.L);
    if (p.L > 10 || p.NH > 1024 || p.NH < 1) return false;
    p.kshift = p.sb_log + p.cs_log + 1;
    p.hbits = ceil_log2(p.NH);
    p.R = 8 * 32 * kRowsPerLane;
    p.NT = (n + p.R - 1) / p.R;
    p.TE = kCapB;
    p.NTB = (nnz + kCapB - 1) / kCapB + p.NH;
    return true;
}

size_t smem_a(const Plan& p, size_t tv) {
    return sizeof(uint32_t) * (size_t)(8 * p.NH + 256 + 3 * p.NH + 1 + 8) + 16 + (tv + 4) * kCapA;
}
size_t smem_b(const Plan& p, size_t tv) {
    const size_t nlo = (size_t)1 << p.L;
    return sizeof(uint32_t) * (8 * nlo + 3 * nlo + 1 + 8) + 16 + (tv + 2) * kCapB;
}

template <typename TV, typename TI>
void run(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const TI* cols, const TV* vals, int64_t n,
         int64_t d, int64_t nnz, const Plan& p, double* sx, cudaStream_t s) {
    RowKeys rk{nullptr, xf->map_seed, FastMod((uint64_t)xf->B), xf->row0};
    if (!xf->seeded_map) {
        uint32_t* rkey = (uint32_t*)ctx->part[5].get(sizeof(uint32_t) * (size_t)n);
        rowkey_from_perm<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 16), 256, 0, s>>>(
            xf->perm, xf->offsets, xf->B, n, rkey);
        count_launch(ctx);
        check_launch("rowkey_from_perm");
        rk.rowkey = rkey;
    }
    const int64_t nlo = (int64_t)1 << p.L;
    const int64_t nA = (int64_t)p.NH * p.NT;
    const int64_t nB = p.NTB * nlo;
    // scratch: [cntA/posA | seg | tstart | cntB/posB] and the two payload copies
    char* meta = (char*)ctx->part[0].get(sizeof(uint32_t) * (size_t)(nA + 2 * (p.NH + 1) + nB + 1));
    uint32_t* posA = (uint32_t*)meta;
    uint32_t* seg = posA + nA;
    uint32_t* ts = seg + p.NH + 1;
    uint32_t* posB = ts + p.NH + 1;
    uint32_t* keyA = (uint32_t*)ctx->part[1].get(sizeof(uint32_t) * (size_t)nnz);
    TV* valA = (TV*)ctx->part[2].get(sizeof(TV) * (size_t)nnz);
    uint16_t* keyB = (uint16_t*)ctx->part[3].get(sizeof(uint16_t) * (size_t)nnz);
    TV* valB = (TV*)ctx->part[4].get(sizeof(TV) * (size_t)nnz);

    part_count_rows<<<(unsigned)p.NT, 256, sizeof(uint32_t) * p.NH, s>>>(rowptr, n, rk, p, posA);
    count_launch(ctx);
    check_launch("part_count_rows");
    exclusive_scan_u32(ctx, posA, posA, nA, s);
    const size_t smA = smem_a(p, sizeof(TV));
    CGX_CUDA(cudaFuncSetAttribute(part_scatter_rows<TV, TI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA));
    part_scatter_rows<TV, TI><<<(unsigned)p.NT, 256, smA, s>>>(rowptr, cols, vals, n, rk, p, posA, keyA, valA);
    count_launch(ctx);
    check_launch("part_scatter_rows");
    part_tiles<<<1, 1024, 0, s>>>(posA, p, (uint32_t)nnz, seg, ts);
    count_launch(ctx);
    check_launch("part_tiles");
    // pass-B counters of absent tiles (the grid is an upper bound) must read as zero
    CGX_CUDA(cudaMemsetAsync(posB, 0, sizeof(uint32_t) * (size_t)nB, s));
    part_count_lo<<<(unsigned)p.NTB, 256, sizeof(uint32_t) * nlo, s>>>(keyA, p, seg, ts, posB);
    count_launch(ctx);
    check_launch("part_count_lo");
    exclusive_scan_u32(ctx, posB, posB, nB, s);
    const size_t smB = smem_b(p, sizeof(TV));
    CGX_CUDA(cudaFuncSetAttribute(part_scatter_lo<TV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB));
    part_scatter_lo<TV><<<(unsigned)p.NTB, 256, smB, s>>>(keyA, valA, p, seg, ts, posB, keyB, valB);
    count_launch(ctx);
    check_launch("part_scatter_lo");
    const int64_t nF = (int64_t)p.NH << p.L;
    const size_t smC = (sizeof(double) + 1) * 8 * 1024;
    CGX_CUDA(cudaFuncSetAttribute(part_accumulate<TV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smC));
    part_accumulate<TV><<<(unsigned)((nF + 7) / 8), 256, smC, s>>>(keyB, valB, p, ts, posB, nB, (uint32_t)nnz, xf->B,
                                                                   d, sx);
    count_launch(ctx);
    check_launch("part_accumulate");
}

} // namespace

bool csr_partition_applies(const cgx_ctx* ctx, int64_t n, int64_t B, int64_t d, int64_t nnz) {
    if (ctx->opt_csr_mode == 1) return false;
    Plan p;
    if (!make_plan(n, B, d, nnz, p)) return false;
    // Opt-in only: measured on c3 (2.56 nnz/row) the five passes take 6.0 ms against 4.4 ms
    // for the row gather -- each partition pass runs at radix-sort speed (~1.7-2 ms for
    // 172 M pairs), so two of them cost more than the gather's DRAM amplification.
    return ctx->opt_csr_mode == 2;
}

void launch_sketch_csr_partition(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols,
                                 int idx_type, const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz,
                                 double* sx, cudaStream_t s) {
    Plan p;
    if (!make_plan(n, xf->B, d, nnz, p)) fail(CGX_EINVAL, "csr partition: shape not covered");
    if (dtype == CGX_F32) {
        if (idx_type == CGX_I32)
            run<float, int32_t>(ctx, xf, rowptr, (const int32_t*)cols, (const float*)vals, n, d, nnz, p, sx, s);
        else
            run<float, int64_t>(ctx, xf, rowptr, (const int64_t*)cols, (const float*)vals, n, d, nnz, p, sx, s);
    } else {
        if (idx_type == CGX_I32)
            run<double, int32_t>(ctx, xf, rowptr, (const int32_t*)cols, (const double*)vals, n, d, nnz, p, sx, s);
        else
            run<double, int64_t>(ctx, xf, rowptr, (const int64_t*)cols, (const double*)vals, n, d, nnz, p, sx, s);
    }
}

} // namespace cgx
