// internal.h -- host-side structures and kernel launchers behind the cgx C-ABI.
#pragma once

#include <cstdint>
#include <cstddef>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/cgx.h"

namespace cgx {

// Status-carrying error used inside the library; converted to a CGX_* code at the ABI.
struct Error {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void set_last_error(const std::string& msg);  // the thread's cgx_last_error() text
void check_cuda(cudaError_t e, const char* what);
#define CGX_CUDA(call) ::cgx::check_cuda((call), #call)

// A grow-only device buffer owned by a context.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need);
    void release();
};

struct HostPool;

// Where a sketch kernel's finished S.X rows land when a device group combines the partial
// sketches over peer memory (group.cu, CGX_COMBINE_P2P): bucket b's row is stored at
// base[b / per] + (b % per) * d -- base[q] is this rank's slot in the landing buffer of the
// rank that owns buckets [q*per, (q+1)*per), a peer-mapped pointer (NVLink / NVSwitch).
constexpr int kMaxSegs = 8;
struct OutSegs {
    double* base[kMaxSegs];
    uint32_t per;
};

struct Profile {
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[2];
    size_t used[2] = {0, 0};
    void begin(int stage, cudaStream_t s);
    void end(int stage, cudaStream_t s);
};

} // namespace cgx

struct cgx_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;        // last call's completion, for cross-stream scratch reuse
    std::recursive_mutex mu;
    uint64_t launches = 0;
    cgx::DevBuf sx, zpart, xstage, tmp;     // scratch (tmp: scan.cu only)
    cgx::DevBuf sort_k[2], sort_v[2], sort_hist, counts;  // transform construction
    cgx::DevBuf hstage_dev;                 // device landing zone for host inputs
    cgx::DevBuf sched;                      // small per-call flags (construct.cu)
    // Work queue of the persistent kernels: one 64-bit counter that is never reset.  A
    // launch handing `ntasks` tasks to `warps` persistent warps advances it by exactly
    // ntasks + warps (every warp's last fetch fails), so the host knows each launch's base
    // and no memset precedes the launch.
    unsigned long long* task_ctr = nullptr;
    unsigned long long task_base = 0;
    cgx::DevBuf gen_tables;                 // synthetic-input generator tables
    cgx::DevBuf gfull;                      // rows of G for the split-over-m stage 2 (gen_gauss_rows)
    cgx::DevBuf gchunk;                     // G super-chunk of the chunked stage 2 (dgemm.cu)
    char* small_pin = nullptr;              // pinned bounce buffer for small results read back by the host
    void* pinned = nullptr;                 // pinned staging for pageable host inputs
    size_t pinned_bytes = 0;
    cgx::Profile prof;
    // host-input staging (hoststage.cu): worker pool, pinned chunk ring, device landing
    // buffers (full / narrowed width) for up to three arrays of one call
    cgx::HostPool* hpool = nullptr;
    char* ring = nullptr;
    cudaEvent_t ring_ev[4] = {};
    uint64_t ring_next = 0;
    cgx::DevBuf hin[6];
    // Caching pool for per-transform device arrays: transforms are built and dropped at
    // high rates by Monte-Carlo callers (distcheck), and cudaMalloc/cudaFree cost more
    // than a small sketch.  Blocks are size-classed (powers of two) and reused.
    std::map<size_t, std::vector<void*>> pool_free;
    std::unordered_map<void*, size_t> pool_class;
    bool no_fuse = false;                  // option "fuse"=0: always run the two stages
    bool force_fuse = false;               // option "fuse"=2: one-pass kernel even when G is in memory
    int fuse_mode = 2;                      // option "fuse_mode": 1 all-warps one-pass, 2 warp-specialized
    int64_t opt_rows_per_task = 1024;       // option "rows_per_task": dense stream-kernel task size
    int64_t opt_tail_tasks = 2;             // option "tail_tasks": single-bucket tasks per warp at the end
    int64_t opt_grid_waves = 1;             // option "grid_waves": stream-kernel blocks = resident x waves
    int64_t opt_ws_gw = 0;                  // option "ws_gw": buckets per sketch warp per tile (0 = auto)
    int64_t opt_async = 2;                  // option "async_stages": cp.async row-gather ring depth (0 = register loads)
    int64_t opt_csr_mode = 0;               // option "csr_mode": 0 auto, 1 row gather, 3 records + L2 atomics
    int64_t opt_csr_slice_mb = 8;           // option "csr_slice_mb": S.X slice per partition of the record path
    int64_t opt_gather_sms = 0;             // option "gather_sms": SMs the CSR gather's persistent grid spans (0 = all)
    int64_t opt_csr_zero = 1;               // option "csr_zero": 1 S.X slices zeroed in the accumulate queue, 0 memset first
    int64_t opt_gemm_tile = 0;              // option "gemm_tile": 1 = 8-warp 64x128/128x64 large-Z tiles
    int64_t opt_gemm_chunks = 0;            // option "gemm_chunks": 1 = 48 MB K-chunks even when G is in memory
    int64_t opt_g_resident = 1;             // option "g_resident": materialize seeded G at construction (<= 4 GiB)
    cgx::DevBuf part[6];                    // csr_atomic.cu scratch: counters, records, row hashes
    int64_t opt_pdl = 1;                    // option "pdl": stage-2 kernels launched as programmatic dependents
    int64_t opt_oz_slices = 7;              // option "oz_slices": stage 2 on tcgen05 int8 with S digit planes (0 = DMMA)
    int64_t opt_oz_min_z = 16384;           // option "oz_min_z": smallest m*d that takes the tcgen05 stage 2
    int64_t opt_oz_cluster = 2;             // option "oz_cluster": CTAs sharing G's planes by multicast (1, 2, 4, 8)
    int64_t opt_oz_st = 0, opt_oz_rs = 4;   // options "oz_st"/"oz_rs": ring depths of the tcgen05 stage 2 (0 = auto)
    int64_t opt_oz_staged = 1;              // option "oz_staged": S.X rows reach the converters by bulk copy (0 = loads)
    int64_t opt_oz_mpair = 1;               // option "oz_mpair": M-tile pairs share the S.X conversion over DSMEM
    cgx::DevBuf oz_max, oz_a, oz_b;         // (oz_b: column maxima of S.X)
    // Set by group.cu around a stage-1 call: S.X rows go to the owners' landing slots instead of
    // `sx`.  The gather kernels store there directly (sketch_dense_async, sketch_csr_lean);
    // every other sketch path writes seg_local and push_segs copies the bucket ranges out.
    const cgx::OutSegs* out_segs = nullptr;
    cgx::DevBuf seg_local;
    int64_t seg_fused = 0, seg_copied = 0;  // stage-1 calls of each kind (cgx_group_stats)
    // Set by group.cu around a CSR call on a row shard: the shard's row offsets are passed as
    // they stand in the caller's array (rowptr + row0), i.e. they index the caller's whole
    // cols/vals arrays, of which the call receives the part starting at element csr_base.
    int64_t csr_base = 0;
    const double* oz_colmax_for = nullptr;  // S.X whose column maxima the sketch left in oz_b
    int64_t oz_colmax_d = 0;         // ozgemm.cu scratch: scales, digit images of G and S.X
};

struct cgx_xform {
    cgx_ctx* ctx = nullptr;
    int64_t B = 0, n = 0, m = 0;
    int64_t row0 = 0;              // global index of local row 0 (row shards, multi-GPU)
    uint64_t t_seed = 0, map_seed = 0, g_seed = 0;
    bool seeded_map = true;        // hash/sign are the index functions of map_seed
    bool has_g = false;
    bool g_explicit = false;
    double* g_dev = nullptr;       // G in memory (m x B col-major): explicit, or resident seeded G
    bool g_pool = false;           // g_dev is a resident copy from the pool (else cudaMalloc'd explicit G)
    uint32_t* perm = nullptr;      // n entries: row | neg<<31, sorted by (bucket, row)
    uint32_t* offsets = nullptr;   // B+1 bucket boundaries into perm
    uint32_t* grows = nullptr;     // bucket-shard transforms: global row index of each local row
    bool view = false;             // a stack copy over borrowed G (no caches may attach to it)
    int8_t* oz_gimg = nullptr;     // ozgemm.cu: G's int8 digit image (oz_gS planes), built on first use
    unsigned long long* oz_gmax = nullptr;
    int oz_gS = 0;
};

namespace cgx {

// Base of a persistent-kernel launch's tasks on ctx->task_ctr (see cgx_ctx::task_ctr).
inline unsigned long long take_tasks(cgx_ctx* ctx, int64_t ntasks, int64_t warps) {
    const unsigned long long b = ctx->task_base;
    ctx->task_base += (unsigned long long)(ntasks + warps);
    return b;
}
// After a persistent-kernel launch: if the launch was rejected the counter did not advance,
// so restart the queue at zero before reporting the error (a stale base would make every
// later launch see its tasks as taken).
inline void tasks_launched(cgx_ctx* ctx, cudaStream_t s) {
    if (cudaPeekAtLastError() != cudaSuccess) {
        cudaMemsetAsync(ctx->task_ctr, 0, sizeof(unsigned long long), s);
        ctx->task_base = 0;
    }
}

// construct.cu
void build_perm_seeded(cgx_ctx* ctx, cgx_xform* xf, cudaStream_t s);
void build_perm_explicit(cgx_ctx* ctx, cgx_xform* xf, const uint32_t* keys_dev, const uint32_t* vals_dev,
                         cudaStream_t s);
bool prep_explicit(cgx_ctx* ctx, const int64_t* hash, const double* sign, int64_t n, int64_t B, uint32_t* keys,
                   uint32_t* vals, cudaStream_t s);
void launch_fill_hash_sign(cgx_ctx* ctx, const cgx_xform* xf, int64_t* hash, double* sign, cudaStream_t s);
// Buckets [b0, b0+nb) of `full` as their own transform: local rows = the full transform's
// rows of those buckets in (bucket, row) order, so local perm is the identity (+ signs).
// global row index of each local row (bucket shards: grows; row shards: row0 + k)
void launch_xform_rows(cgx_ctx* ctx, const cgx_xform* xf, int64_t* rows, cudaStream_t s);
void launch_bucket_shard(cgx_ctx* ctx, const cgx_xform* full, int64_t b0, int64_t nb, uint32_t o0, cgx_xform* local,
                         cudaStream_t s);

// sketch_dense.cu: SX (row-major B x d, fp64) from row-major X.
void launch_sketch_dense(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int64_t ld, int64_t n,
                         int64_t d, double* sx, cudaStream_t s);
// Whole countgauss_apply in one kernel (+ the partial reduction) for row-major X with
// wide rows; false when the shape is not covered (caller runs the two stages).
bool launch_countgauss_dense_fused(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int64_t ld,
                                   int64_t d, double* z, cudaStream_t s);
// Deterministic sum of `splits` column-major partials (gauss_gemm.cu).
void launch_reduce_splits(cgx_ctx* ctx, const double* zpart, int64_t splits, int64_t md, double* z, cudaStream_t s);
// col-major -> row-major copy of X (any dtype) into dst
void launch_transpose_x(cgx_ctx* ctx, const void* x, int dtype, int64_t ld, int64_t n, int64_t d, void* dst,
                        cudaStream_t s);
// row-major B x d (fp64) -> col-major
void launch_transpose_sx(cgx_ctx* ctx, const double* src, int64_t B, int64_t d, double* dst, cudaStream_t s);

// sketch_dense.cu / sketch_csr.cu: whether the launch below stores straight into ctx->out_segs
bool sketch_dense_fuses_segs(const cgx_ctx* ctx, const void* x, int dtype, int64_t ld, int64_t d);
bool sketch_csr_fuses_segs(const cgx_ctx* ctx, int64_t d, int64_t chunk_rows);
// group.cu: out[i] = ((slot_0[i] + slot_1[i]) + ...) for i < count, slots `stride` doubles apart
void launch_sum_slots(cgx_ctx* c, const double* slots, int P, int64_t stride, int64_t count, double* out,
                      cudaStream_t st);
// capi.cu: rows [q*per, (q+1)*per) of a local row-major S.X -> segs.base[q] (device-to-device copies)
void push_segs(cgx_ctx* ctx, const double* sx, int64_t B, int64_t d, const OutSegs& segs, cudaStream_t s);

// sketch_csr.cu
void launch_sketch_csr(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols, int idx_type,
                       const void* vals, int dtype, int64_t n, int64_t d, double* sx, int64_t chunk_rows,
                       cudaStream_t s);

// csr_atomic.cu: bucket-range partitioned records + L2-resident fp64 RED (short-row CSR)
bool csr_atomic_applies(const cgx_ctx* ctx, const cgx_xform* xf, int64_t n, int64_t d, int64_t nnz, int dtype);
void launch_sketch_csr_atomic(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols, int idx_type,
                              const void* vals, int64_t n, int64_t d, int64_t nnz, double* sx, cudaStream_t s);

// gauss_gemm.cu: z (col-major m x d) = G . sx (row-major B x d)
// Buckets [b0, b1) only: sx points at row b0 (split-K across ranks).
void launch_gauss_gemm(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t b0, int64_t b1, int64_t d,
                       double* z, cudaStream_t s);
void launch_fill_gaussian(cgx_ctx* ctx, const cgx_xform* xf, double* g, cudaStream_t s);
// gauss_gemm.cu: T = G . S, m x n column-major
void launch_materialize_t(cgx_ctx* ctx, const cgx_xform* xf, double* t, cudaStream_t s);
// dgemm.cu: G columns [c0, c0+cols) of the transform -> out (m x cols, col-major)
void launch_gen_gauss(cgx_ctx* ctx, const cgx_xform* xf, int64_t c0, int64_t cols, double* out, cudaStream_t s);
// dgemm.cu: rows [r0, r1) of Z = G[r0:r1, :] . sx (the multi-GPU split of G's m rows)
void launch_gauss_gemm_rows(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t d, int64_t r0, int64_t r1,
                            double* z, cudaStream_t s);
// dgemm.cu: Z within one CTA tile (ceil(m/32) x ceil(d/32) <= 8 warps), G in memory or
// generated in L2-resident chunks; false when not applicable
bool launch_gemm_small_g_ready(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t b0, int64_t b1,
                               int64_t d, double* z, cudaStream_t s);
// dgemm.cu: G super-chunks + pipelined DMMA GEMM; false when Z is small (not used)
bool launch_gauss_gemm_chunked(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t b0, int64_t b1,
                               int64_t d, double* z, cudaStream_t s, bool force = false);
// ozgemm.cu: z (col-major m x d) = g (m x K col-major) . sx (row-major K x d) on tcgen05 kind::i8
// with FP64 emulated by S = opt_oz_slices digit slices; false when the option is off
// (buckets [b0, b1): sx points at row b0; G's digit image is cached on the transform)
bool launch_gemm_ozaki(cgx_ctx* ctx, const cgx_xform* xf, int64_t b0, int64_t b1, const double* sx, int64_t d,
                       double* z, cudaStream_t s);
void oz_drop_image(cgx_xform* xf);  // whenever G changes or goes
bool oz_stage2_applies(const cgx_ctx* ctx, const cgx_xform* xf, int64_t d);
// dgemm.cu: row-major fp32 (pitch ld) -> contiguous row-major fp64
void launch_widen_f32(cgx_ctx* ctx, const float* src, int64_t ld, int64_t n, int64_t d, double* dst, cudaStream_t s);
void launch_inverse_normal_cdf(cgx_ctx* ctx, const double* p, double* out, int64_t count, int* bad,
                               cudaStream_t s);

// extremes.cu
void launch_select_extremes(cgx_ctx* ctx, const double* z, int64_t m, int64_t d, int64_t* amax, int64_t* amin,
                            int64_t* tie_flags, cudaStream_t s);

// datagen.cu
void launch_gen_dense(cgx_ctx* ctx, uint64_t seed, int64_t row0, const int64_t* rows, int64_t n, int64_t d, int dtype,
                      int layout, void* x,
                      cudaStream_t s);
// config 4: H = Dirichlet(alpha) mixing weights (r x cols column-major, host) and the
// near-separable X = max(A.[I_r | H] + sigma*N(0,1), 0), rows [row0, row0+n)
void separable_mixing(uint64_t seed, int64_t r, int64_t cols, double alpha, double* h);
void launch_gen_separable(cgx_ctx* ctx, uint64_t seed, int64_t row0, int64_t n, int64_t d, int64_t r, double alpha,
                          double sigma, int dtype, int layout, void* x, cudaStream_t s);
struct CsrGenSpec {
    bool zipf = false;
    double density = 0.0;                      // Bernoulli
    double s_len = 1.5, s_col = 1.1;           // Zipf exponents (row length, column popularity)
    int cap = 512;                             // row-length cap
};
void launch_gen_csr_counts(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, const CsrGenSpec& spec,
                           int64_t* rowptr, cudaStream_t s);
void launch_gen_csr_fill(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, const CsrGenSpec& spec,
                         const int64_t* rowptr, int32_t* cols, float* vals, cudaStream_t s);

// gproject.cu: dense-Gaussian baseline Z = G~.X for CSR X, G~(r, i) = draw i*m + r of g_seed
void launch_gproject_csr(cgx_ctx* ctx, uint64_t g_seed, int64_t m, const int64_t* rowptr, const void* cols,
                         int idx_type, const void* vals, int dtype, int64_t n, int64_t d, double* z, cudaStream_t s);

// csr_io.cu: binary CSR container (CGXCSR1) and the streamed file -> pinned -> HBM loader
void csr_save(const char* path, const int64_t* rowptr, const void* cols, int idx_type, const void* vals, int dtype,
              int64_t n, int64_t d, int64_t nnz);
void csr_info(const char* path, int64_t* n, int64_t* d, int64_t* nnz, int* idx_type, int* dtype);
void csr_load(cgx_ctx* ctx, const char* path, int64_t* rowptr, void* cols, void* vals, int mem, cudaStream_t s);

// batch.cu: distcheck's trial loop -- su = S_t.U and gram(su) for trials [t0, t0+trials)
void launch_batch_sketch_gram(cgx_ctx* ctx, uint64_t master, int64_t t0, int64_t trials, int64_t B, const double* u,
                              int64_t ld, int64_t n, int64_t d, double* su_out, double* gram_out, cudaStream_t s);

// scan.cu: exclusive scans (in place allowed), total written to out[count] when requested
void exclusive_scan_u32(cgx_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t count, cudaStream_t s);
void exclusive_scan_i64(cgx_ctx* ctx, const int64_t* in, int64_t* out, int64_t count, cudaStream_t s);

// hoststage.cu: pipelined pinned staging of a host array with lossless narrowing (kind 1:
// fp64 -> fp32, kind 2: int64 -> int32); *narrowed when the whole array arrived narrowed
// (seg, sld): the source is count/seg segments of seg elements, sld elements apart (a
// column-major row block), landing contiguous on the device; 0 = one contiguous array
const void* stage_in(cgx_ctx* ctx, DevBuf& full, DevBuf& half, const void* src, size_t count, size_t esize, int kind,
                     bool* narrowed, cudaStream_t s, size_t seg = 0, size_t sld = 0);
uint64_t host_checksum(cgx_ctx* ctx, const void* p, size_t bytes);
void host_pool_free(cgx_ctx* ctx);

// Rows per task of the persistent gather kernels: the option's ~1K rows, fewer when the
// input is small (a row shard) so that every one of the ~num_sms * 32 resident warps gets at
// least two tasks -- with fewer tasks than warps, each warp walked one long task with one
// chunk in flight and c2's sketch at n/8 rows took 90 us against ~45 us of streaming.
inline int64_t rows_per_task(const cgx_ctx* ctx, int64_t n) {
    const int64_t fair = n / ((int64_t)ctx->num_sms * 32 * 2);
    int64_t r = ctx->opt_rows_per_task < fair ? ctx->opt_rows_per_task : fair;
    return r < 64 ? 64 : r;
}

inline void count_launch(cgx_ctx* ctx, int k = 1) { ctx->launches += (uint64_t)k; }
// Launch as a programmatic dependent of the previous kernel in the stream (option "pdl"): its
// CTAs start while that kernel's last CTAs drain and wait in pdl_wait for its results.
template <typename... KArgs, typename... Args>
inline void launch_pdl(cgx_ctx* ctx, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ctx->opt_pdl ? 1 : 0;
    CGX_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
}
void* pool_alloc(cgx_ctx* ctx, size_t bytes);
void pool_free(cgx_ctx* ctx, void* p);
void check_launch(const char* what);

} // namespace cgx
