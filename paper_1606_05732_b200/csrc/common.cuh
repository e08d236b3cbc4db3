// common.cuh -- device-side primitives shared by every kernel of the CountGauss path.
//
//  * SplitMix64 counter map: draw k of SeededRng(seed) is F(seed + (k+1)*gamma)
//    (reference include/countgauss/rng.hpp:31-37), so hashes, signs and G entries are
//    pure functions of (seed, index) and are computed where they are consumed.
//  * Exact 64-bit "mod B" through a 64x64->128 high multiply (no software division).
//  * The reference's N(0,1) quantile: Acklam's rational approximation followed by one
//    Halley step against erfc (reference src/rng.cpp:13-55).  The arithmetic is written
//    with explicit _rn intrinsics so nvcc cannot contract it into FMAs that the x86
//    reference (built without FMA) does not perform; only erfc/exp/log differ (CUDA libm
//    vs glibc), which is why G parity is stated as a tolerance.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace cgx {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t fin64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// Draw k (0-based) of SeededRng(seed).
__host__ __device__ __forceinline__ uint64_t rng_draw(uint64_t seed, uint64_t k) {
    return fin64(seed + (k + 1) * kGamma);
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) {
    return fin64(a + kGamma + b * 0xBF58476D1CE4E5B9ULL);
}

// z mod B for 1 <= B < 2^63 with magic = floor((2^64-1)/B): q = hi(z*magic) is floor(z/B)
// or one less, so one conditional subtraction finishes the job.
struct FastMod {
    uint64_t B;
    uint64_t magic;
    __host__ explicit FastMod(uint64_t b) : B(b), magic(~0ULL / b) {}
    __device__ __forceinline__ uint64_t operator()(uint64_t z) const {
        uint64_t q = __umul64hi(z, magic);
        uint64_t r = z - q * B;
        return r >= B ? r - B : r;
    }
};

// Row i of a seeded CountSketch (sketch.cpp:21-26): bucket = draw 2i mod B,
// sign = + iff draw 2i+1 is odd.  Returned as (bucket, negative?).
__device__ __forceinline__ uint32_t cs_bucket(uint64_t cs_seed, uint64_t i, const FastMod& mod) {
    return (uint32_t)mod(rng_draw(cs_seed, 2 * i));
}
__device__ __forceinline__ uint32_t cs_negative(uint64_t cs_seed, uint64_t i) {
    return (uint32_t)((rng_draw(cs_seed, 2 * i + 1) & 1ULL) ^ 1ULL);
}

// next_uniform (rng.hpp:40-42): exact in fp64.
__host__ __device__ __forceinline__ double uniform53(uint64_t u) {
    return ((double)(u >> 11) + 0.5) * 0x1.0p-53;
}

#define CGX_M(a, b) __dmul_rn((a), (b))
#define CGX_A(a, b) __dadd_rn((a), (b))

// Acklam's rational approximation (rng.cpp:13-41), evaluated in the reference's order.
__device__ __forceinline__ double acklam(double p) {
    const double a0 = -3.969683028665376e+01, a1 = 2.209460984245205e+02, a2 = -2.759285104469687e+02,
                 a3 = 1.383577518672690e+02, a4 = -3.066479806614716e+01, a5 = 2.506628277459239e+00;
    const double b0 = -5.447609879822406e+01, b1 = 1.615858368580409e+02, b2 = -1.556989798598866e+02,
                 b3 = 6.680131188771972e+01, b4 = -1.328068155288572e+01;
    const double c0 = -7.784894002430293e-03, c1 = -3.223964580411365e-01, c2 = -2.400758277161838e+00,
                 c3 = -2.549732539343734e+00, c4 = 4.374664141464968e+00, c5 = 2.938163982698783e+00;
    const double d0 = 7.784695709041462e-03, d1 = 3.224671290700398e-01, d2 = 2.445134137142996e+00,
                 d3 = 3.754408661907416e+00;
    const double p_low = 0.02425;
    if (p >= p_low && p <= 1.0 - p_low) {
        double q = __dadd_rn(p, -0.5);
        double r = CGX_M(q, q);
        double num = CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(a0, r), a1), r), a2), r), a3), r), a4), r), a5);
        num = CGX_M(num, q);
        double den = CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(b0, r), b1), r), b2), r), b3), r), b4), r), 1.0);
        return __ddiv_rn(num, den);
    }
    // Tails: q = sqrt(-2 log(p)) for p < p_low, sqrt(-2 log(1-p)) (negated result) above.
    const bool upper = p > 1.0 - p_low;
    double t = upper ? __dadd_rn(1.0, -p) : p;
    double q = __dsqrt_rn(CGX_M(-2.0, log(t)));
    double num = CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(c0, q), c1), q), c2), q), c3), q), c4), q), c5);
    double den = CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(CGX_A(CGX_M(d0, q), d1), q), d2), q), d3), q), 1.0);
    double x = __ddiv_rn(num, den);
    return upper ? -x : x;
}

// Out of line: taken by ~4e-6 of draws, and inlined it costs the warp-specialised kernels
// registers on their hot path.
static __device__ __noinline__ double acklam_far(double p) { return acklam(p); }

// Starting point for the Halley step of inverse_normal_cdf: Acklam's rational, with the
// central region in fp64 (FMA-contracted; its polynomial cancels near |p-0.5| = 0.475, so
// fp32 would lose 1e-4 there) and the tails -- whose log/sqrt dominate the FP64 cost and
// which diverge a warp 80% of the time -- in fp32 with MUFU log/sqrt (~4e-7 relative).
// Halley's cubic convergence takes either start below fp64 resolution, so the refined
// quantile is limited by erfc exactly as the reference's is (the reference starts from
// Acklam's 1.15e-9).  The tail variable (p or 1-p) is formed in fp64 before narrowing.
__device__ __forceinline__ double acklam_start(double p) {
    const double a0 = -3.969683028665376e+01, a1 = 2.209460984245205e+02, a2 = -2.759285104469687e+02,
                 a3 = 1.383577518672690e+02, a4 = -3.066479806614716e+01, a5 = 2.506628277459239e+00;
    const double b0 = -5.447609879822406e+01, b1 = 1.615858368580409e+02, b2 = -1.556989798598866e+02,
                 b3 = 6.680131188771972e+01, b4 = -1.328068155288572e+01;
    const float c0 = -7.784894002430293e-03f, c1 = -3.223964580411365e-01f, c2 = -2.400758277161838e+00f,
                c3 = -2.549732539343734e+00f, c4 = 4.374664141464968e+00f, c5 = 2.938163982698783e+00f;
    const float d0 = 7.784695709041462e-03f, d1 = 3.224671290700398e-01f, d2 = 2.445134137142996e+00f,
                d3 = 3.754408661907416e+00f;
    const double p_low = 0.02425;
    if (p >= p_low && p <= 1.0 - p_low) {
        const double q = p - 0.5;
        const double r = q * q;
        const double num = (((((a0 * r + a1) * r + a2) * r + a3) * r + a4) * r + a5) * q;
        const double den = ((((b0 * r + b1) * r + b2) * r + b3) * r + b4) * r + 1.0;
        return num / den;
    }
    const bool upper = p > 1.0 - p_low;
    const double t64 = upper ? 1.0 - p : p;
    // Far tails (t < 2^-20, one draw in ~5e5 per tail): the reference's Halley residual is
    // rounded at ulp(p), which near p = 1 resolves x only to ulp(p)/phi(x) -- there its
    // output is its Acklam start plus noise, so the start must be the reference's own.
    // (Also keeps fp32 away from t below FLT_MIN.)
    if (t64 < 0x1.0p-20) return acklam_far(p);
    const float t = (float)t64;
    const float q = sqrtf(-2.0f * logf(t));
    const float num = ((((c0 * q + c1) * q + c2) * q + c3) * q + c4) * q + c5;
    const float den = (((d0 * q + d1) * q + d2) * q + d3) * q + 1.0f;
    const double x = (double)(num / den);
    return upper ? -x : x;
}

// inverse_normal_cdf (rng.cpp:45-55) for p in (0,1): one Halley step against erfc from an
// Acklam start (fp32 in the near tails, see acklam_start).
__device__ __forceinline__ double inverse_normal_cdf(double p) {
    double x = acklam_start(p);
    const double sqrt2pi = 2.5066282746310005024;
    const double sqrt2 = 1.41421356237309504880;
    double e = __dadd_rn(CGX_M(0.5, erfc(__ddiv_rn(-x, sqrt2))), -p);
    double u = CGX_M(CGX_M(e, sqrt2pi), exp(CGX_M(CGX_M(0.5, x), x)));
    x = __dadd_rn(x, -__ddiv_rn(u, CGX_A(1.0, CGX_M(CGX_M(0.5, x), u))));
    return x;
}

// G(r, c) of gaussian_matrix(m, B, SeededRng(g_seed)) (matrix.cpp:199-207): draw c*m + r.
__device__ __forceinline__ double gauss_entry(uint64_t g_seed, uint64_t m, uint64_t r, uint64_t c) {
    return inverse_normal_cdf(uniform53(rng_draw(g_seed, c * m + r)));
}

// Synthetic-input normal (oracle/cgoracle.c cgo_normal_f32): fp32 rounding of the Acklam
// quantile; the Halley step is below fp32 resolution.
__device__ __forceinline__ float datagen_normal(uint64_t seed, uint64_t e) {
    return (float)acklam(uniform53(rng_draw(seed, e)));
}

#undef CGX_M
#undef CGX_A

// ---- programmatic dependent launch: a dependent kernel (launched with
// cudaLaunchAttributeProgrammaticStreamSerialization) may be scheduled once every CTA of the
// running kernel has called pdl_trigger (or exited); it calls pdl_wait before touching the
// running kernel's results (returns at once when the kernel was launched normally) ----------
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- shared-memory mbarriers (producer/consumer hand-off between warp roles) ----------
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_addr(bar))
                 : "memory");
}
// Wait until the phase with parity `parity` of `bar` has completed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// ---- bulk copies (TMA engine, 1-D): global -> shared, completion counted on an mbarrier --
// The arriving thread announces the transaction bytes, then issues copies that complete_tx
// on the same barrier; waiters see the phase flip once every byte has landed.
// mbar_wait for long waits (a warp idle for a whole accumulation): polls with a sleep in
// between, so the spinning does not take issue slots from the warps doing the work
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity, unsigned ns) {
    for (;;) {
        unsigned ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        __nanosleep(ns);
    }
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
// size and both addresses multiples of 16 bytes
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(smem)),
                 "l"(gmem), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// ---- cp.async (LDGSTS): 16 B global -> shared, bypassing L1; completion by group ------
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Fire-and-forget global reductions.  atomicAdd with its result unused compiles to a
// returning ATOMG (destination RZ) in this library's relocatable-device-code build, while a
// whole-program build gets REDG: the returning form waits on L2 responses and measured ~30%
// fewer fp64 adds per second on B200 (1.38 vs 1.00 ms for 172 M adds into 8 MB slices,
// tools/microbench/l2_red2.cu).  These spell out the RED.
__device__ __forceinline__ void red_add(double* p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void red_add(unsigned* p, unsigned v) {
    asm volatile("red.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Named barrier among `count` threads (id 1..15; 0 is __syncthreads).
__device__ __forceinline__ void named_sync(unsigned id, unsigned count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Perm entries: row index in bits 0..30, "negative sign" flag in bit 31.
constexpr uint32_t kRowMask = 0x7FFFFFFFu;
constexpr uint32_t kNegBit = 0x80000000u;

// Mask of the lanes whose v equals this lane's (the result of __match_any_sync), for
// v < 2^nbits, built from nbits ballots.  MATCH.ANY resolves one distinct value per pass,
// so on 32 mostly-distinct digits -- the common case for the bucket and bin digits here
// -- it costs tens of times more than these vote-unit instructions.  All lanes active;
// nbits <= 12.
__device__ __forceinline__ unsigned match_any_bits(uint32_t v, int nbits) {
    unsigned m = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 12; ++b) {  // nbits <= 12, warp-uniform
        if (b < nbits) {
            const unsigned x = __ballot_sync(0xffffffffu, (v >> b) & 1u);
            m &= x ^ (((v >> b) & 1u) - 1u);  // x where my bit is 1, ~x where it is 0
        }
    }
    return m;
}

__device__ __forceinline__ int warp_incl_scan(int v, unsigned lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if ((int)lane >= o) v += t;
    }
    return v;
}

} // namespace cgx
