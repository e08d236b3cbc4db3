/* cgx.h -- C-ABI of the B200-native CountGauss path (T.X = G.(S.X), arXiv 1606.05732).
 *
 * Drop-in boundary for the reference library's hot path
 * (/root/reference/proj/include/countgauss/sketch.hpp:25-54, nmf.hpp:51-52).  The
 * reference has no C ABI; each entry point below names the C++ symbol it replaces.
 * Plain pointers and sizes only -- no C++ or torch types cross this boundary, and no
 * exception escapes it: every function returns a CGX_* status and sets a thread-local
 * message readable with cgx_last_error().  The C++ shim maps
 * CGX_EINVAL to std::invalid_argument with the reference's own messages.
 *
 * Memory: every array argument carries a `mem` flag.  CGX_MEM_HOST arrays are ordinary
 * (pageable or pinned) host memory and the call is synchronous, exactly like the
 * reference.  CGX_MEM_DEVICE arrays are device pointers on the context's GPU; such a
 * call is stream-ordered on `stream` (NULL = the context's own stream) and returns
 * without waiting for the GPU when every array is device-resident.  Inputs are
 * borrowed for the duration of the call; outputs are caller-owned.
 *
 * Threading: a context may be shared by threads (the reference's functions are called
 * from inside OpenMP regions, distcheck.cpp:107-111); calls on one context serialize.
 *
 * Results: hashes, signs, per-row extremes and S.X are bit-identical to the reference
 * (S.X accumulates every (bucket, column) in ascending row order, as sketch.cpp:52-113
 * does, including the 8192-row chunked CSR branch).  G is the reference's
 * SplitMix64 + Acklam/Halley quantile evaluated with CUDA's libm (tolerance parity),
 * and Z = G.(S.X) is within a relative Frobenius tolerance of the reference.
 */
#ifndef CGX_H
#define CGX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    CGX_OK = 0,
    CGX_EINVAL = 1,  /* std::invalid_argument in the reference */
    CGX_ENOMEM = 2,  /* device or pinned-host allocation failed */
    CGX_ECUDA = 3,   /* CUDA runtime / launch error */
    CGX_ENCCL = 4,   /* reserved: collective failure */
    CGX_ERANGE = 5   /* std::length_error in the reference (size overflow) */
};
enum { CGX_F64 = 0, CGX_F32 = 1 };            /* value dtype */
enum { CGX_I64 = 0, CGX_I32 = 1 };            /* CSR column-index dtype */
enum { CGX_COL_MAJOR = 0, CGX_ROW_MAJOR = 1 }; /* dense layout */
enum { CGX_MEM_HOST = 0, CGX_MEM_DEVICE = 1 };

typedef struct cgx_ctx cgx_ctx;     /* one GPU: stream, scratch, counters */
typedef struct cgx_xform cgx_xform; /* a CountSketch map, optionally with its Gaussian G */

/* ---- library / context ------------------------------------------------------------- */
const char* cgx_last_error(void);
const char* cgx_version(void);
int cgx_init(int device, cgx_ctx** out);
int cgx_free(cgx_ctx* ctx);
int cgx_synchronize(cgx_ctx* ctx, void* stream);
/* Release the device memory the context keeps between calls -- per-call scratch buffers and
 * the free lists of the transform-array pool (live transforms keep theirs) -- after
 * waiting for the context's work.  No reference counterpart (the CPU library has no
 * device memory); for long-lived callers that alternate large and small problems. */
int cgx_trim(cgx_ctx* ctx);
/* Device allocations owned by the context's GPU (for callers without an allocator). */
int cgx_device_alloc(cgx_ctx* ctx, size_t bytes, void** out);
int cgx_device_free(cgx_ctx* ctx, void* p);
int cgx_host_alloc(cgx_ctx* ctx, size_t bytes, void** out); /* pinned */
int cgx_host_free(cgx_ctx* ctx, void* p);
int cgx_memcpy(cgx_ctx* ctx, void* dst, const void* src, size_t bytes, void* stream);

/* ---- seed plumbing (pure host functions; rng.hpp:12-37) ---------------------------- */
/* mix64(a, b)  -- include/countgauss/rng.hpp:12-17 */
uint64_t cgx_mix64(uint64_t a, uint64_t b);
/* draw k (0-based) of SeededRng(seed)  -- rng.hpp:31-37 */
uint64_t cgx_rng_draw(uint64_t seed, uint64_t k);

/* ---- construction ------------------------------------------------------------------- */
/* countsketch_new(buckets, input_dim, rng)  -- sketch.cpp:12-28.  `map_seed` is the
 * value the reference stores in map.seed, i.e. the caller's rng.next_u64(). */
int cgx_countsketch_new(cgx_ctx* ctx, uint64_t map_seed, int64_t buckets, int64_t input_dim,
                        cgx_xform** out);
/* countsketch_injective(buckets, input_dim, rng)  -- sketch.cpp:30-50 (Fisher-Yates on
 * the host: its hashes are not an index function of the seed). */
int cgx_countsketch_injective(cgx_ctx* ctx, uint64_t map_seed, int64_t buckets, int64_t input_dim,
                              cgx_xform** out);
/* A hand-built CountSketchMap (CountSketchMap fields, sketch.hpp:15-21): hash[i] in
 * [0, buckets), sign[i] in {-1, +1}. */
int cgx_countsketch_explicit(cgx_ctx* ctx, int64_t buckets, int64_t input_dim, const int64_t* hash,
                             const double* sign, int mem, cgx_xform** out);
/* countgauss_new(m, buckets, input_dim, rng)  -- sketch.cpp:115-126.  `t_seed` is the
 * caller's rng.next_u64() (the reference's t.seed); S and G derive from it.  The
 * two-argument overload (sketch.cpp:128-130) is buckets = 5*m. */
int cgx_countgauss_new(cgx_ctx* ctx, uint64_t t_seed, int64_t m, int64_t buckets, int64_t input_dim,
                       cgx_xform** out);
/* Row shard [row0, row0+rows) of the same transform (multi-GPU row sharding; no
 * reference counterpart -- the paper's seed-sharing): hashes and signs
 * are those of the shard's *global* rows, applied to an X holding only the shard's rows.
 * Sum over shards of countsketch_apply == the full S.X up to fp reassociation. */
int cgx_countgauss_new_shard(cgx_ctx* ctx, uint64_t t_seed, int64_t m, int64_t buckets, int64_t input_dim,
                             int64_t row0, int64_t rows, cgx_xform** out);
/* Attach G to a map: seeded (G column-major draw order of SeededRng(g_seed),
 * matrix.cpp:199-207) or explicit (m x buckets, column-major). */
int cgx_xform_set_gaussian_seeded(cgx_ctx* ctx, cgx_xform* xf, int64_t m, uint64_t g_seed);
int cgx_xform_set_gaussian_explicit(cgx_ctx* ctx, cgx_xform* xf, int64_t m, const double* g, int mem);
int cgx_xform_info(const cgx_xform* xf, uint64_t* t_seed, uint64_t* map_seed, uint64_t* g_seed,
                   int64_t* m, int64_t* buckets, int64_t* input_dim);
int cgx_xform_free(cgx_xform* xf);

/* ---- materializers (the transform structs' public fields) -------------------------- */
/* cs.hash / cs.sign  (sketch.hpp:18-19) */
int cgx_fill_hash_sign(cgx_ctx* ctx, const cgx_xform* xf, int64_t* hash, double* sign, int mem,
                       void* stream);
/* g, m x buckets column-major  (sketch.hpp:45) */
int cgx_fill_gaussian(cgx_ctx* ctx, const cgx_xform* xf, double* g, int mem, void* stream);
/* inverse_normal_cdf elementwise  (rng.hpp:62, rng.cpp:45-55); p outside (0,1) -> CGX_EINVAL */
int cgx_inverse_normal_cdf(cgx_ctx* ctx, const double* p, double* out, int64_t count, int mem,
                           void* stream);

/* ---- apply -------------------------------------------------------------------------- */
/* countsketch_apply(map, DenseMatrix)  -- sketch.cpp:52-66.  X is n x d with leading
 * dimension ld (elements) in `layout`; sx receives S.X, buckets x d, in `sx_layout`
 * (CGX_COL_MAJOR = the reference DenseMatrix). */
int cgx_countsketch_apply_dense(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype,
                                int layout, int64_t ld, int64_t n, int64_t d, int x_mem, double* sx,
                                int sx_layout, int sx_mem, void* stream);
/* countsketch_apply(map, SparseMatrix)  -- sketch.cpp:68-113.  CSR with int64 row offsets
 * (n+1), column indices (int32/int64, strictly increasing per row), values (f32/f64). */
int cgx_countsketch_apply_csr(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr,
                              const void* cols, int idx_type, const void* vals, int dtype, int64_t n,
                              int64_t d, int64_t nnz, int x_mem, double* sx, int sx_layout, int sx_mem,
                              void* stream);
/* countgauss_apply(t, DenseMatrix)  -- sketch.cpp:132-134.  z: m x d, column-major. */
int cgx_countgauss_apply_dense(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int layout,
                               int64_t ld, int64_t n, int64_t d, int x_mem, double* z, int z_mem,
                               void* stream);
/* countgauss_apply(t, SparseMatrix)  -- sketch.cpp:136-138. */
int cgx_countgauss_apply_csr(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols,
                             int idx_type, const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz,
                             int x_mem, double* z, int z_mem, void* stream);
/* Stage 2 alone: z = G . sx  (gemm(t.g, SX), matrix.cpp:111-129) with G regenerated
 * inside the kernel from the transform's seed (never materialized). */
int cgx_gauss_gemm(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int sx_layout, int64_t d,
                   int sx_mem, double* z, int z_mem, void* stream);
/* Split-K piece of stage 2: z = G[:, b0:b1) . sx_rows, where sx_rows is the row-major
 * (b1-b0) x d slice of S.X for buckets [b0, b1) (a reduce-scatter's output). */
int cgx_gauss_gemm_range(cgx_ctx* ctx, const cgx_xform* xf, const double* sx_rows, int64_t b0, int64_t b1,
                         int64_t d, int sx_mem, double* z, int z_mem, void* stream);

/* Large CSR ingestion, replacing the text Matrix Market / CSV readers
 * (io.cpp:72-136, 159-214): a binary container "CGXCSR1" -- 64-byte header, then row
 * offsets int64[n+1], column indices (CGX_I32/CGX_I64) [nnz], values (CGX_F32/CGX_F64)
 * [nnz] -- holding the arrays exactly as the apply entry points take them.
 * cgx_csr_load with mem = CGX_MEM_DEVICE streams the file through two pinned 32 MiB
 * buffers, overlapping the disk read of chunk k+1 with the H2D copy of chunk k; the
 * caller provides arrays sized from cgx_csr_info.  With mem = CGX_MEM_HOST it is a plain
 * read and ctx may be null. */
int cgx_csr_save(const char* path, const int64_t* rowptr, const void* cols, int idx_type, const void* vals, int dtype,
                 int64_t n, int64_t d, int64_t nnz);
int cgx_csr_info(const char* path, int64_t* n, int64_t* d, int64_t* nnz, int* idx_type, int* dtype);
int cgx_csr_load(cgx_ctx* ctx, const char* path, int64_t* rowptr, void* cols, void* vals, int mem, void* stream);

/* T = G . S  (m x n, column-major): the CountGauss projection matrix that svm-check builds as
 * gemm(t.g, reference::materialize(t.cs)) (tools/countgauss_main.cpp:660-668, svm.cpp:128-150).
 * Column i is sign_i * G(:, hash_i), bit-identical to that gemm (which skips S's zeros). */
int cgx_countgauss_materialize(cgx_ctx* ctx, const cgx_xform* xf, double* t, int mem, void* stream);

/* Dense-Gaussian baseline for CSR X (the config-5 ablation): z = G~ . X with
 * G~ = gaussian_matrix(m, n, rng) at the rng state `rng_state` -- the reference bench's
 * naive O(nnz * m) loop (tools/countgauss_main.cpp:535-547, acceptance.cpp:365-377).
 * G~ is generated where it is used and never stored.  Z matches to rounding (fp64
 * atomics), not bitwise; the caller's rng advances by m*n draws. */
int cgx_gaussian_project_csr(cgx_ctx* ctx, uint64_t rng_state, int64_t m, const int64_t* rowptr, const void* cols,
                             int idx_type, const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz, int x_mem,
                             double* z, int z_mem, void* stream);

/* Batched tiny sketches -- distcheck's Monte-Carlo loop (distcheck.cpp:107-113): for each
 * trial t in [t0, t0+trials): map = countsketch_new(buckets, n, SeededRng(mix64(master, t)))
 * (sketch.cpp:12-28), su = countsketch_apply(map, U) (sketch.cpp:52-66), gram(su)
 * (matrix.cpp:149-165).  U: n x d fp64 column-major (leading dimension ld).  Outputs, each
 * optional (null to skip): su, trials blocks of buckets x d column-major; gram, trials
 * blocks of d x d column-major.  Both bit-identical to the reference.  One launch. */
int cgx_countsketch_batch_gram(cgx_ctx* ctx, uint64_t master, int64_t t0, int64_t trials, int64_t buckets,
                               const double* u, int64_t ld, int64_t n, int64_t d, int u_mem, double* su,
                               double* gram, int out_mem, void* stream);

/* Hash-partitioned row placement (SURVEY 8e ablation C): buckets [b0, b1) of
 * countgauss_new(t_seed, m, buckets, input_dim) as a transform of their own.  Its rows are
 * the full transform's rows hashing into [b0, b1), in (bucket, global row) order -- a rank
 * that holds exactly those rows, in that order, sketches them with a sequential read and
 * no reduction: S.X of the shard = rows [b0, b1) of the full S.X (bit-identical), and its
 * G is G[:, b0:b1), so countgauss_apply gives the split-K partial Z_p (sum over ranks = Z).
 * cgx_xform_info reports buckets = b1-b0 and input_dim = the shard's row count. */
int cgx_countgauss_bucket_shard(cgx_ctx* ctx, uint64_t t_seed, int64_t m, int64_t buckets, int64_t input_dim,
                                int64_t b0, int64_t b1, cgx_xform** out);
/* Global row index of each local row of a transform (input_dim entries): a bucket shard's
 * row list, or row0 + k for row shards and ordinary transforms. */
int cgx_xform_rows(cgx_ctx* ctx, const cgx_xform* xf, int64_t* rows, int mem, void* stream);

/* Split of G's m rows across ranks (north star's multi-GPU final product):
 * z = G[r0:r1, :] . sx -- (r1-r0) x d column-major -- with sx the full row-major B x d S.X
 * (e.g. after an all-reduce of the partial sketches). */
int cgx_gauss_gemm_rows(cgx_ctx* ctx, const cgx_xform* xf, const double* sx, int64_t d, int64_t r0, int64_t r1,
                        int sx_mem, double* z, int z_mem, void* stream);

/* Dense-Gaussian baseline (SURVEY 8f, config-5 ablation): z = G~ . X with G~ the m x n
 * i.i.d. N(0,1) matrix gaussian_matrix(m, n, rng) would draw (matrix.cpp:199-207) from a
 * SeededRng whose current state is `rng_state` -- the product gp_nmf computes
 * (nmf.cpp:155-159).  G~ is generated in L2-resident chunks, never stored whole.  The
 * caller advances its rng by m*n draws. */
int cgx_gaussian_project_dense(cgx_ctx* ctx, uint64_t rng_state, int64_t m, const void* x, int dtype, int layout,
                               int64_t ld, int64_t n, int64_t d, int x_mem, double* z, int z_mem, void* stream);

/* select_extremes(Z)  -- nmf.cpp:99-118: per row argmax/argmin of an m x d column-major
 * Z, strict compares (ties to the lowest column), tie_rows = rows whose max or min is
 * attained more than once.  amax/amin: m entries each (unsorted, per row). */
int cgx_select_extremes(cgx_ctx* ctx, const double* z, int64_t m, int64_t d, int mem, int64_t* amax,
                        int64_t* amin, int64_t* tie_rows, void* stream);

/* ---- synthetic inputs (device generators; the oracle shares their definition) ------ */
/* Dense n x d, entry (i,j) = fp32 N(0,1) quantile of draw i*d+j of SeededRng(seed)
 * (oracle/cgoracle.c cgo_normal_f32); dtype F64 stores the exact widening. */
int cgx_gen_dense_normal(cgx_ctx* ctx, uint64_t seed, int64_t row0, int64_t n, int64_t d, int dtype,
                         int layout, void* x_dev, void* stream); /* rows [row0, row0+n) */
/* The same values for an arbitrary list of n global rows (device int64 array): the rows of
 * a bucket-shard transform (cgx_xform_rows). */
int cgx_gen_dense_normal_rows(cgx_ctx* ctx, uint64_t seed, const int64_t* rows_dev, int64_t n, int64_t d,
                              int dtype, int layout, void* x_dev, void* stream);
/* CSR n x d with Bernoulli(density) entries (int32 cols, fp32 N(0,1) values).  Call once
 * with cols/vals NULL to get row offsets and *nnz_out, then again with buffers. */
int cgx_gen_csr_bernoulli(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, double density,
                          int64_t* rowptr_dev, int32_t* cols_dev, float* vals_dev, int64_t* nnz_out,
                          void* stream);

/* Config-5 style heavy-tailed CSR: row i draws a target length L from Zipf(s_len) on
 * [1, cap]; column j is kept with probability min(1, c_L * w_j), w_j ~ (j+1)^-s_col
 * normalized and c_L solved so that a row's expected length is L (Zipf-skewed columns,
 * sorted and distinct).  Same two-phase protocol. */
int cgx_gen_csr_zipf(cgx_ctx* ctx, uint64_t seed, int64_t n, int64_t d, double s_len, int64_t cap, double s_col,
                     int64_t* rowptr_dev, int32_t* cols_dev, float* vals_dev, int64_t* nnz_out, void* stream);

/* Config 4 (BASELINE configs[3]): near-separable nonnegative X for NMF anchor selection,
 * X = max(A.[I_r | H] + sigma*N(0,1), 0) with A (n x r) uniform on [0,1) and the columns of
 * H (r x (d-r)) drawn from Dirichlet(alpha): every non-anchor column of X is a convex
 * combination of the r anchor columns 0..r-1, plus clipped noise.  Rows [row0, row0+n) of
 * the matrix defined by `seed`; fp32 arithmetic without FMA (CPU twin in
 * oracle/cgoracle.c).  No reference counterpart: generate_separable (nmf.cpp:12-44) mixes
 * with normalized uniforms and has no noise. */
int cgx_gen_separable(cgx_ctx* ctx, uint64_t seed, int64_t row0, int64_t n, int64_t d, int64_t r, double alpha,
                      double sigma, int dtype, int layout, void* x_dev, void* stream);
/* The mixing weights H of cgx_gen_separable (r x cols, column-major, fp64, host): column c
 * is Dirichlet(alpha), the normalized Marsaglia-Tsang Gamma(alpha) draws of
 * SeededRng(mix64(seed, 13)).  Pure host function (no context, no GPU). */
int cgx_separable_mixing(uint64_t seed, int64_t r, int64_t cols, double alpha, double* h);

/* 64-bit content checksum of a host array (bytes of it), computed with the context's host
 * worker threads (ctx may be null: one thread).  The drop-in shim uses it to verify that a
 * transform's public fields still hold what construction wrote before taking the cached
 * device transform ("seeded fast path"). */
int cgx_host_checksum(cgx_ctx* ctx, const void* p, size_t bytes, uint64_t* out);

/* ---- device groups: one process, several GPUs of a node (the north star's
 * multi-GPU split; no reference counterpart -- the reference has no distributed code, the
 * scheme is the paper's seed sharing) ----------------------------------
 * A group holds one context per device and one NCCL communicator per device
 * (ncclCommInitAll over NVLink/NVSwitch; NCCL is loaded with dlopen on first use --
 * CGX_ENCCL if it cannot be).  A group transform gives rank p the rows
 * [row0_p, row0_p + rows_p) of countgauss_new(t_seed, m, buckets, input_dim) (contiguous
 * shards, sizes differing by at most one); rank p builds its part of S from the shared seed
 * for its global rows, so no map is exchanged.  The apply runs every rank on its own host
 * thread and combines the partials over NCCL:
 *   CGX_COMBINE_G  all-reduce of the B x d partial S.X; rank p computes rows
 *                  [p*ceil(m/P), ...) of Z = G.S.X (G's m rows split); row blocks all-gathered
 *   CGX_COMBINE_SX reduce-scatter of S.X by bucket range (ceil(B/P) buckets per rank);
 *                  split-K stage 2 on the owned slice; all-reduce of Z
 *   CGX_COMBINE_Z  both stages per rank on its shard; all-reduce of Z
 *   CGX_COMBINE_P2P no NCCL: the reduce-scatter of S.X is fused into the sketch kernels, whose
 *                  finished bucket rows are stored straight into the owning rank's landing
 *                  buffer over peer-mapped memory (NVLink / NVSwitch); owners sum their P slots
 *                  and the partial Z's in rank order, so every rank gets the same bits and the
 *                  result does not depend on timing.  Needs peer access between all devices
 *                  (else CGX_EINVAL) and at most 8 ranks.  A device may be listed twice in
 *                  cgx_group_init (two ranks on one GPU); such a group supports only this mode.
 * Z equals the single-GPU result up to floating-point reassociation across ranks. */
enum { CGX_COMBINE_Z = 0, CGX_COMBINE_G = 1, CGX_COMBINE_SX = 2, CGX_COMBINE_P2P = 3 };
typedef struct cgx_group cgx_group;
typedef struct cgx_gxform cgx_gxform;
int cgx_group_init(int ndev, const int* devs, cgx_group** out);
int cgx_group_free(cgx_group* g);
int cgx_group_size(const cgx_group* g);
int cgx_group_context(cgx_group* g, int rank, cgx_ctx** out); /* rank's context (owned by the group) */
/* 1 if the group can run this combine mode (NCCL modes: distinct devices; CGX_COMBINE_P2P: peer
 * access between all of them and at most 8 ranks), else 0. */
int cgx_group_supports(const cgx_group* g, int combine);
/* CGX_COMBINE_P2P bookkeeping, summed over ranks: stage-1 calls whose gather kernel stored its
 * rows straight into the owners' landing slots, and calls that sketched locally and copied the
 * bucket ranges out (the kernels without segmented stores: narrow dense X, the chunked CSR
 * branch, the record path). */
int cgx_group_stats(const cgx_group* g, int64_t* fused_sketches, int64_t* copied_sketches);
int cgx_group_countgauss_new(cgx_group* g, uint64_t t_seed, int64_t m, int64_t buckets, int64_t input_dim,
                             cgx_gxform** out);
int cgx_gxform_free(cgx_gxform* t);
int cgx_gxform_shard(const cgx_gxform* t, int rank, int64_t* row0, int64_t* rows);
/* countgauss_apply(t, DenseMatrix) over the group.  x_mem CGX_MEM_HOST: x is the whole
 * n x d matrix on the host (layout, ld as in cgx_countgauss_apply_dense); each rank stages its
 * row block.  x_mem CGX_MEM_DEVICE: x is an array of P device pointers, rank p's shard
 * (rows_p x d, same layout and ld) on device p.  z_mem CGX_MEM_HOST: z is the m x d
 * column-major result; CGX_MEM_DEVICE: z is an array of P device pointers, each receiving Z. */
int cgx_group_countgauss_apply_dense(cgx_group* g, const cgx_gxform* t, const void* x, int dtype, int layout,
                                     int64_t ld, int64_t n, int64_t d, int x_mem, double* z, int z_mem, int combine);
/* countgauss_apply(t, SparseMatrix) over the group; CSR in host memory (rowptr[0] = 0). */
int cgx_group_countgauss_apply_csr(cgx_group* g, const cgx_gxform* t, const int64_t* rowptr, const void* cols,
                                   int idx_type, const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz,
                                   double* z, int z_mem, int combine);

/* ---- the peer-memory combine for one process per GPU (torchrun-style launches; no reference
 * counterpart -- the reference has no distributed code, PAPER.md:274-275 only names seed sharing)
 * The pieces of CGX_COMBINE_P2P as separate calls, for callers whose ranks are processes: each
 * rank allocates its landing buffer (cgx_device_alloc), exports it (cgx_ipc_export: a 64-byte
 * CUDA IPC handle to pass to the other ranks by any host channel), opens the others'
 * (cgx_ipc_open; on NVLink-connected GPUs the mapping is a peer mapping), and runs its sketch
 * with cgx_countsketch_apply_*_to: bucket b's finished row goes to bases[b / per] +
 * (b % per) * d -- the kernels that can, store there directly; the others sketch locally and
 * copy the ranges (as in CGX_COMBINE_P2P).  After the ranks have synchronized on the host, each
 * sums its slots in rank order with cgx_sum_slots and runs cgx_gauss_gemm_range on the result
 * (paper_1606_05732_b200/distributed.py, combine "p2p"). */
#define CGX_IPC_HANDLE_BYTES 64
int cgx_ipc_export(cgx_ctx* ctx, const void* dev_ptr, unsigned char* handle /* [CGX_IPC_HANDLE_BYTES] */);
int cgx_ipc_open(cgx_ctx* ctx, const unsigned char* handle, void** dev_ptr);
int cgx_ipc_close(cgx_ctx* ctx, void* dev_ptr);
int cgx_countsketch_apply_dense_to(cgx_ctx* ctx, const cgx_xform* xf, const void* x, int dtype, int layout, int64_t ld,
                                   int64_t n, int64_t d, int x_mem, double* const* bases, int nseg, int64_t per,
                                   void* stream);
int cgx_countsketch_apply_csr_to(cgx_ctx* ctx, const cgx_xform* xf, const int64_t* rowptr, const void* cols,
                                 int idx_type, const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz, int x_mem,
                                 double* const* bases, int nseg, int64_t per, void* stream);
/* out[i] = ((slot_0[i] + slot_1[i]) + ...) for i < count; slot q starts at slots + q * stride. */
int cgx_sum_slots(cgx_ctx* ctx, const double* slots, int nslots, int64_t stride, int64_t count, double* out,
                  void* stream);

/* ---- instrumentation ---------------------------------------------------------------- */
/* Context options (kernel variants for A/B runs; every variant gives the same S.X bits and
 * Z to rounding -- "oz_slices" below 7 trades Z accuracy for speed, as stated):
 *   "g_resident"   1 (default): countgauss_new materializes G (<= 4 GiB) and applies read
 *                  it; 0: G is generated inside the apply kernels.  Set before construction.
 *   "fuse"         1 (default): the one-pass dense kernel (sketch + G + contraction) when G
 *                  is not resident; 2: also when it is; 0: always the two stages.
 *   "fuse_mode"    one-pass variant: 2 (default) warp-specialized, 1 all-warps.
 *   "async_stages" dense row-gather ring depth: 2 (default), 3, 4; 0 = register batches.
 *   "csr_mode"     0 (default): the record path for short-row CSR (fp32 values, < 8 nnz/row,
 *                  >= 4M nnz, B*d >= 2^22; S.X to fp64 rounding), else the gather; 1: always
 *                  the bucket-ordered row gather (S.X bit-identical to the reference); 3: the
 *                  record path whenever it applies (csr_atomic.cu).
 *   "csr_slice_mb", "csr_sc": the record path's S.X slice per partition (8 MB default) and
 *                  scatter variant.
 *   "oz_slices"    stage 2 (gemm, matrix.cpp:111-129) on the tcgen05 int8 tensor cores with
 *                  FP64 emulated by S planes of 8-bit digits (ozgemm.cu): 7 (default; Z within
 *                  ~1e-14 of fp64), 6 (~7e-13), 5 (~1.5e-10), 3-4; 0 = always the FP64 DMMA
 *                  stage 2.  Used when G is in memory and m*d >= "oz_min_z" (16384 default;
 *                  smaller Z streams faster through the split-K DMMA kernel).
 *   "oz_staged"    1 (default): S.X tiles reach the converter warps by TMA; 0: direct loads.
 *   "pdl"          1 (default): stage-2 kernels are programmatic dependent launches (their
 *                  CTAs start while the sketch drains); 0: ordinary stream order.
 *   "oz_cluster"   2 (default), 1, 4, 8: CTAs (N tiles) sharing G's digit planes by multicast.
 *   "oz_st", "oz_rs": ring depths of the tensor-core stage 2 (MMA ring: 0 = automatic; raw
 *                  S.X ring: 2 default -- deeper prefetch measured slower, c5 4.76 vs 5.10 ms).
 *   "gemm_tile", "gemm_chunks": DMMA stage-2 tiling (128x128 one-pass default; 1 = 8-warp
 *                  tiles / 48 MB G chunks).
 *   "rows_per_task", "grid_waves", "ws_gw", "tail_tasks": scheduling knobs of the sketch
 *                  kernels. */
int cgx_set_option(cgx_ctx* ctx, const char* key, int64_t value);
/* Number of kernels this context has launched so far. */
uint64_t cgx_launch_count(const cgx_ctx* ctx);
/* When enabled, the sketch (stage 1) and gemm (stage 2) kernels of every apply are
 * bracketed with CUDA events on their launch stream; cgx_profile_read synchronizes and
 * returns total milliseconds and launches per stage (0 = sketch, 1 = gemm), then resets. */
int cgx_profile_enable(cgx_ctx* ctx, int on);
int cgx_profile_read(cgx_ctx* ctx, int stage, double* total_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* CGX_H */
