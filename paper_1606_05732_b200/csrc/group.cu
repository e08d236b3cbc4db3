// group.cu -- multi-GPU CountGauss behind the C ABI (include/cgx.h, "device groups"): one
// process drives several GPUs of a node, for C++ callers of the drop-in (the
// north star's split).  The reference has no distributed code; the scheme is the paper's
// seed sharing: rank p holds rows shard_range(n, P, p) of X and builds
// its part of S from the shared seed for its *global* rows, so no map is exchanged.  The
// partials combine over NCCL (ncclCommInitAll: one communicator per device, NVLink /
// NVSwitch inside the node):
//   CGX_COMBINE_G  (default, dense): all-reduce of the B x d partial S.X, then rank p
//                  computes rows [p*ceil(m/P), ...) of Z = G[r0:r1, :].S.X -- G's m rows
//                  split across ranks -- and the row blocks are gathered;
//   CGX_COMBINE_SX (CSR):  reduce-scatter of S.X by bucket range, split-K stage 2 on the
//                  owned slice, all-reduce of Z;
//   CGX_COMBINE_Z:         every rank runs both stages on its shard, all-reduce of Z.
// and, without NCCL, over peer memory:
//   CGX_COMBINE_P2P: the reduce-scatter of S.X is fused into the sketch kernels.  Every rank
//                  owns a bucket range and a landing buffer of P slots; rank p's gather
//                  kernel stores each finished bucket row straight into slot p of the
//                  owner's buffer (peer-mapped pointers, NVLink stores: OutSegs in
//                  internal.h), so the transfer rides under the whole sketch instead of
//                  following it.  The owner then sums its P slots in rank order
//                  (`sum_slots`: a fixed order, so the result does not depend on timing),
//                  runs the split-K stage 2 on its range, writes its m x d partial Z into
//                  every rank's Z slots, and each rank sums those in rank order: every
//                  rank ends with the same bits.  Ranks order their streams with events
//                  (record, host join, wait): no kernel ever waits on another GPU's kernel.
// Each device is driven by its own host thread (host-input staging blocks the host; the
// threads are started with the group and parked between calls), its kernels and collectives
// ordered on its context's stream.  NCCL is loaded with dlopen on
// first use, so libcgx has no link-time NCCL dependency.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nccl.h>

#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

struct Nccl {
    bool ok = false;
    std::string why;
    decltype(&ncclCommInitAll) CommInitAll = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclReduceScatter) ReduceScatter = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl r;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            r.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return r;
        }
#define CGX_SYM(f)                                                      \
    r.f = (decltype(r.f))dlsym(h, "nccl" #f);                           \
    if (!r.f) {                                                         \
        r.why = "libnccl.so.2 lacks nccl" #f;                           \
        return r;                                                       \
    }
        CGX_SYM(CommInitAll)
        CGX_SYM(CommDestroy)
        CGX_SYM(AllReduce)
        CGX_SYM(ReduceScatter)
        CGX_SYM(AllGather)
        CGX_SYM(GroupStart)
        CGX_SYM(GroupEnd)
        CGX_SYM(GetErrorString)
#undef CGX_SYM
        r.ok = true;
        return r;
    }();
    return n;
}

void check_nccl(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    fail(CGX_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

void shard(int64_t n, int P, int p, int64_t* a, int64_t* b) {  // distributed.shard_range
    const int64_t base = n / P, extra = n % P;
    *a = p * base + std::min<int64_t>(p, extra);
    *b = *a + base + (p < extra ? 1 : 0);
}

// The group's rank threads: one per device, started once (a thread start per rank and call
// cost ~40 us of every apply) and parked on a condition variable between calls.  run(f) hands
// f(p) to every rank's thread, waits for all of them and rethrows the first failure.
class RankThreads {
public:
    explicit RankThreads(int P) : P_(P), errs_((size_t)P), bad_((size_t)P, 0) {
        for (int p = 0; p < P; ++p) th_.emplace_back([this, p] { loop(p); });
    }
    ~RankThreads() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void run(const std::function<void(int)>& f) {
        std::lock_guard<std::mutex> call(call_);  // one job at a time per group
        {
            std::lock_guard<std::mutex> lk(m_);
            job_ = &f;
            left_ = P_;
            std::fill(bad_.begin(), bad_.end(), 0);
            ++gen_;
        }
        cv_.notify_all();
        {
            std::unique_lock<std::mutex> lk(m_);
            done_.wait(lk, [&] { return left_ == 0; });
            job_ = nullptr;
        }
        for (int p = 0; p < P_; ++p)
            if (bad_[(size_t)p]) throw errs_[(size_t)p];
    }

private:
    void loop(int p) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* job;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                job = job_;
            }
            try {
                (*job)(p);
            } catch (const Error& e) {
                errs_[(size_t)p] = e;
                bad_[(size_t)p] = 1;
            } catch (const std::exception& e) {
                errs_[(size_t)p] = Error{CGX_ECUDA, e.what()};
                bad_[(size_t)p] = 1;
            }
            {
                std::lock_guard<std::mutex> lk(m_);
                if (--left_ == 0) done_.notify_all();
            }
        }
    }
    int P_;
    std::vector<std::thread> th_;
    std::vector<Error> errs_;
    std::vector<char> bad_;
    std::mutex m_, call_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* job_ = nullptr;
    int left_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

void ok_or_throw(int rc) {
    if (rc != CGX_OK) fail(rc, cgx_last_error());
}

// Phase boundary of the rank threads inside one each_rank (the peer-memory combine): a rank
// that failed keeps arriving, so nobody is left waiting, and everyone skips the later phases.
struct PhaseBarrier {
    explicit PhaseBarrier(int n) : n_(n) {}
    void arrive_and_wait() {
        std::unique_lock<std::mutex> lk(m_);
        const uint64_t g = gen_;
        if (++count_ == n_) {
            count_ = 0;
            ++gen_;
            cv_.notify_all();
        } else {
            cv_.wait(lk, [&] { return gen_ != g; });
        }
    }
    std::atomic<bool> failed{false};

private:
    std::mutex m_;
    std::condition_variable cv_;
    int n_, count_ = 0;
    uint64_t gen_ = 0;
};

} // namespace

// out[i] = ((slot_0[i] + slot_1[i]) + slot_2[i]) + ... for i < count; slots `stride` apart.
__global__ void sum_slots_kernel(const double* __restrict__ slots, int P, int64_t stride, int64_t count,
                          double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        double a = slots[i];
        for (int q = 1; q < P; ++q) a += slots[(int64_t)q * stride + i];
        out[i] = a;
    }
}

void launch_sum_slots(cgx_ctx* c, const double* slots, int P, int64_t stride, int64_t count, double* out,
                      cudaStream_t st) {
    if (count <= 0) return;
    const int64_t blocks = std::min<int64_t>((count + 255) / 256, (int64_t)c->num_sms * 16);
    sum_slots_kernel<<<(unsigned)blocks, 256, 0, st>>>(slots, P, stride, count, out);
    c->launches++;
    CGX_CUDA(cudaGetLastError());
}
} // namespace cgx

struct cgx_group {
    int P = 0;
    std::vector<int> dev;
    std::vector<cgx_ctx*> ctx;
    std::vector<ncclComm_t> comm;
    std::vector<cgx::DevBuf> sx, slice, zp, zg, rp;  // per-rank scratch (rp: Z row blocks)
    // CGX_COMBINE_P2P: per-rank landing buffers (P slots of ceil(B/P) x d, and of m x d) that
    // the other ranks' kernels and copies write, and the events ordering the ranks' streams
    std::vector<cgx::DevBuf> land, zslot;
    std::vector<cudaEvent_t> ev_sx, ev_z;
    bool have_nccl = false, p2p = false;
    std::string nccl_why, p2p_why;
    std::unique_ptr<cgx::RankThreads> threads;
    std::mutex mu;  // one group call at a time (the ranks' scratch and landing buffers are per group)
};

namespace cgx {
namespace {
template <class F>
void each_rank(cgx_group* g, F&& f) {
    g->threads->run(std::function<void(int)>(std::forward<F>(f)));
}
} // namespace
} // namespace cgx

struct cgx_gxform {
    cgx_group* g = nullptr;
    int64_t m = 0, B = 0, n = 0;
    std::vector<cgx_xform*> xf;
    std::vector<int64_t> r0, r1;
};

using namespace cgx;

namespace {

template <class F>
int gguard(F&& f) {
    try {
        f();
        return CGX_OK;
    } catch (const Error& e) {
        set_last_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return CGX_ENOMEM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return CGX_ECUDA;
    }
}

// The combine step of rank p, on its context's stream, once rank p's stage 1 (or both
// stages, for CGX_COMBINE_Z) is queued.  The NCCL calls of all ranks run concurrently from
// their threads (one communicator per device).
void combine_rank(cgx_group* g, const cgx_gxform* t, int p, int64_t d, int mode, double* z_host, int z_mem,
                  double* const* z_dev) {
    cgx_ctx* c = g->ctx[(size_t)p];
    const Nccl& N = nccl();
    const int P = g->P;
    const int64_t m = t->m, B = t->B;
    cudaStream_t st = c->stream;
    CGX_CUDA(cudaSetDevice(c->device));
    double* zfull = (double*)g->zg[(size_t)p].get(sizeof(double) * (size_t)(m * d));
    if (mode == CGX_COMBINE_Z) {
        double* zp = (double*)g->zp[(size_t)p].p;
        check_nccl(N.AllReduce(zp, zfull, (size_t)(m * d), ncclDouble, ncclSum, g->comm[(size_t)p], st), "ncclAllReduce(Z)");
    } else if (mode == CGX_COMBINE_SX) {
        const int64_t per = (B + P - 1) / P;
        double* sx = (double*)g->sx[(size_t)p].p;  // (per*P) x d row-major, zero-padded past B
        double* sl = (double*)g->slice[(size_t)p].get(sizeof(double) * (size_t)(per * d));
        check_nccl(N.ReduceScatter(sx, sl, (size_t)(per * d), ncclDouble, ncclSum, g->comm[(size_t)p], st),
                   "ncclReduceScatter(S.X)");
        const int64_t b0 = std::min(B, p * per), b1 = std::min(B, b0 + per);
        double* zp = (double*)g->zp[(size_t)p].get(sizeof(double) * (size_t)(m * d));
        if (b1 > b0)
            ok_or_throw(cgx_gauss_gemm_range(c, t->xf[(size_t)p], sl, b0, b1, d, CGX_MEM_DEVICE, zp, CGX_MEM_DEVICE, st));
        else
            CGX_CUDA(cudaMemsetAsync(zp, 0, sizeof(double) * (size_t)(m * d), st));
        check_nccl(N.AllReduce(zp, zfull, (size_t)(m * d), ncclDouble, ncclSum, g->comm[(size_t)p], st), "ncclAllReduce(Z)");
    } else {  // CGX_COMBINE_G
        double* sx = (double*)g->sx[(size_t)p].p;  // B x d row-major
        check_nccl(N.AllReduce(sx, sx, (size_t)(B * d), ncclDouble, ncclSum, g->comm[(size_t)p], st), "ncclAllReduce(S.X)");
        const int64_t per = (m + P - 1) / P;
        const int64_t r0 = std::min(m, p * per), r1 = std::min(m, r0 + per);
        // rank p's rows as a zero-padded per x d column-major block; blocks are all-gathered
        double* blk = (double*)g->zp[(size_t)p].get(sizeof(double) * (size_t)(per * d));
        double* all = (double*)g->slice[(size_t)p].get(sizeof(double) * (size_t)(per * P * d));
        CGX_CUDA(cudaMemsetAsync(blk, 0, sizeof(double) * (size_t)(per * d), st));
        if (r1 > r0) {
            double* rows = (double*)g->rp[(size_t)p].get(sizeof(double) * (size_t)((r1 - r0) * d));
            ok_or_throw(cgx_gauss_gemm_rows(c, t->xf[(size_t)p], sx, d, r0, r1, CGX_MEM_DEVICE, rows, CGX_MEM_DEVICE, st));
            CGX_CUDA(cudaMemcpy2DAsync(blk, sizeof(double) * per, rows, sizeof(double) * (r1 - r0),
                                       sizeof(double) * (r1 - r0), d, cudaMemcpyDeviceToDevice, st));
        }
        check_nccl(N.AllGather(blk, all, (size_t)(per * d), ncclDouble, g->comm[(size_t)p], st), "ncclAllGather(Z rows)");
        for (int q = 0; q < P; ++q) {  // block q -> rows [q*per, ...) of the m x d column-major Z
            const int64_t a = std::min(m, q * per), b = std::min(m, a + per);
            if (b > a)
                CGX_CUDA(cudaMemcpy2DAsync(zfull + a, sizeof(double) * m, all + q * per * d, sizeof(double) * per,
                                           sizeof(double) * (b - a), d, cudaMemcpyDeviceToDevice, st));
        }
    }
    if (z_mem == CGX_MEM_DEVICE) {
        CGX_CUDA(cudaMemcpyAsync(z_dev[p], zfull, sizeof(double) * (size_t)(m * d), cudaMemcpyDeviceToDevice, st));
    } else if (p == 0) {
        CGX_CUDA(cudaMemcpyAsync(z_host, zfull, sizeof(double) * (size_t)(m * d), cudaMemcpyDeviceToHost, st));
    }
    CGX_CUDA(cudaStreamSynchronize(st));
}

// Stage 1 of rank p into the combine mode's landing buffer (or both stages for Z).
void partial_rank(cgx_group* g, const cgx_gxform* t, int p, int64_t d, int mode,
                  const std::function<void(cgx_ctx*, cgx_xform*, double*, bool)>& apply) {
    cgx_ctx* c = g->ctx[(size_t)p];
    CGX_CUDA(cudaSetDevice(c->device));
    if (mode == CGX_COMBINE_Z) {
        double* zp = (double*)g->zp[(size_t)p].get(sizeof(double) * (size_t)(t->m * d));
        apply(c, t->xf[(size_t)p], zp, true);
        return;
    }
    const int P = g->P;
    const int64_t rows = mode == CGX_COMBINE_SX ? (t->B + P - 1) / P * P : t->B;
    double* sx = (double*)g->sx[(size_t)p].get(sizeof(double) * (size_t)(rows * d));
    if (rows > t->B)
        CGX_CUDA(cudaMemsetAsync(sx + t->B * d, 0, sizeof(double) * (size_t)((rows - t->B) * d), c->stream));
    apply(c, t->xf[(size_t)p], sx, false);
}

void check_mode(const cgx_group* g, int mode) {
    if (mode == CGX_COMBINE_P2P) {
        if (!g->p2p) fail(CGX_EINVAL, "cgx_group: CGX_COMBINE_P2P unavailable: " + g->p2p_why);
        return;
    }
    if (mode != CGX_COMBINE_Z && mode != CGX_COMBINE_G && mode != CGX_COMBINE_SX)
        fail(CGX_EINVAL, "cgx_group: combine must be CGX_COMBINE_Z, _G, _SX or _P2P");
    if (!g->have_nccl) fail(CGX_ENCCL, "cgx_group: " + g->nccl_why);
}

// CGX_COMBINE_P2P.  stage1(p, ctx, xform, out) queues rank p's countsketch_apply with `out` as
// its (device, row-major) destination; ctx->out_segs redirects the rows to the owners' slots.
void apply_p2p(cgx_group* g, const cgx_gxform* t, int64_t d,
               const std::function<void(int, cgx_ctx*, cgx_xform*, double*)>& stage1, double* z_host, int z_mem,
               double* const* z_dev) {
    const int P = g->P;
    const int64_t m = t->m, B = t->B, per = (B + P - 1) / P;
    const int64_t slot = per * d, zn = m * d;
    // every rank's kernels store into every rank's landing buffer: allocate them all first
    for (int p = 0; p < P; ++p) {
        CGX_CUDA(cudaSetDevice(g->dev[(size_t)p]));
        g->land[(size_t)p].get(sizeof(double) * (size_t)(slot * P));
        g->zslot[(size_t)p].get(sizeof(double) * (size_t)(zn * P));
    }
    // One thread per rank, three phases separated by host barriers (an event must have been
    // recorded before another rank's stream can be made to wait on it).
    PhaseBarrier bar(P);
    each_rank(g, [&](int p) {
        cgx_ctx* c = g->ctx[(size_t)p];
        cudaStream_t st = c->stream;
        Error err{CGX_OK, ""};
        auto phase = [&](auto&& body) {
            if (bar.failed.load()) return;
            try {
                body();
            } catch (const Error& e) {
                err = e;
                bar.failed.store(true);
            } catch (const std::exception& e) {
                err = Error{CGX_ECUDA, e.what()};
                bar.failed.store(true);
            }
        };
        // A: the sketch, storing (or copying) bucket range q into slot p of rank q
        phase([&] {
            CGX_CUDA(cudaSetDevice(c->device));
            OutSegs segs{};
            for (int q = 0; q < P; ++q) segs.base[q] = (double*)g->land[(size_t)q].p + (int64_t)p * slot;
            segs.per = (uint32_t)per;
            c->out_segs = &segs;
            try {
                stage1(p, c, t->xf[(size_t)p], segs.base[p]);
            } catch (...) {
                c->out_segs = nullptr;
                throw;
            }
            c->out_segs = nullptr;
            CGX_CUDA(cudaEventRecord(g->ev_sx[(size_t)p], st));
        });
        bar.arrive_and_wait();
        // B: rank p sums its slots, runs stage 2 on its bucket range, hands its partial Z to everyone
        phase([&] {
            for (int q = 0; q < P; ++q)
                if (q != p) CGX_CUDA(cudaStreamWaitEvent(st, g->ev_sx[(size_t)q], 0));
            const int64_t b0 = std::min(B, p * per), b1 = std::min(B, b0 + per);
            double* sl = (double*)g->slice[(size_t)p].get(sizeof(double) * (size_t)slot);
            double* zp = (double*)g->zp[(size_t)p].get(sizeof(double) * (size_t)zn);
            const double* mine = (const double*)g->land[(size_t)p].p;
            if (P > 1) launch_sum_slots(c, mine, P, slot, (b1 - b0) * d, sl, st);
            if (b1 > b0)
                ok_or_throw(cgx_gauss_gemm_range(c, t->xf[(size_t)p], P > 1 ? sl : mine, b0, b1, d, CGX_MEM_DEVICE, zp,
                                                 CGX_MEM_DEVICE, st));
            else
                CGX_CUDA(cudaMemsetAsync(zp, 0, sizeof(double) * (size_t)zn, st));
            for (int q = 0; q < P; ++q)
                CGX_CUDA(cudaMemcpyAsync((double*)g->zslot[(size_t)q].p + (int64_t)p * zn, zp,
                                         sizeof(double) * (size_t)zn, cudaMemcpyDeviceToDevice, st));
            CGX_CUDA(cudaEventRecord(g->ev_z[(size_t)p], st));
        });
        bar.arrive_and_wait();
        // C: Z = the partials in rank order, on every rank
        phase([&] {
            for (int q = 0; q < P; ++q)
                if (q != p) CGX_CUDA(cudaStreamWaitEvent(st, g->ev_z[(size_t)q], 0));
            const double* zsl = (const double*)g->zslot[(size_t)p].p;
            double* zfull = (double*)g->zg[(size_t)p].get(sizeof(double) * (size_t)zn);
            if (P > 1) launch_sum_slots(c, zsl, P, zn, zn, zfull, st);
            const double* zres = P > 1 ? zfull : zsl;
            if (z_mem == CGX_MEM_DEVICE)
                CGX_CUDA(cudaMemcpyAsync(z_dev[p], zres, sizeof(double) * (size_t)zn, cudaMemcpyDeviceToDevice, st));
            else if (p == 0)
                CGX_CUDA(cudaMemcpyAsync(z_host, zres, sizeof(double) * (size_t)zn, cudaMemcpyDeviceToHost, st));
        });
        // (a failed rank may have left work queued that reads peers' buffers: always drain)
        cudaStreamSynchronize(st);
        if (err.code != CGX_OK) throw err;
    });
}

} // namespace

extern "C" {

int cgx_group_init(int ndev, const int* devs, cgx_group** out) {
    return gguard([&] {
        if (!out || ndev < 1 || !devs) fail(CGX_EINVAL, "cgx_group_init: need ndev >= 1 devices");
        // A device listed twice gives two ranks on one GPU: NCCL refuses that, the peer-memory
        // combine does not (its "peer" pointers are then local) -- which is also how the P2P path
        // is tested on a one-GPU box.
        std::vector<int> uniq(devs, devs + ndev);
        std::sort(uniq.begin(), uniq.end());
        const bool distinct = std::adjacent_find(uniq.begin(), uniq.end()) == uniq.end();
        const Nccl& N = nccl();
        if (distinct && !N.ok) fail(CGX_ENCCL, "cgx_group_init: " + N.why);
        auto* g = new cgx_group;
        g->P = ndev;
        g->dev.assign(devs, devs + ndev);
        g->ctx.assign((size_t)ndev, nullptr);
        g->comm.assign((size_t)ndev, nullptr);
        g->ev_sx.assign((size_t)ndev, nullptr);
        g->ev_z.assign((size_t)ndev, nullptr);
        for (auto* v : {&g->sx, &g->slice, &g->zp, &g->zg, &g->rp, &g->land, &g->zslot}) v->resize((size_t)ndev);
        try {
            for (int p = 0; p < ndev; ++p) ok_or_throw(cgx_init(devs[p], &g->ctx[(size_t)p]));
            g->threads.reset(new RankThreads(ndev));
            if (distinct) {
                check_nccl(N.CommInitAll(g->comm.data(), ndev, devs), "ncclCommInitAll");
                g->have_nccl = true;
            } else {
                g->nccl_why = "a device appears twice in the group: only CGX_COMBINE_P2P applies";
            }
            // peer access, both ways, between every pair of distinct devices
            g->p2p = ndev <= kMaxSegs;
            if (!g->p2p) g->p2p_why = "more than " + std::to_string(kMaxSegs) + " ranks";
            for (int p = 0; p < ndev && g->p2p; ++p) {
                CGX_CUDA(cudaSetDevice(devs[p]));
                for (int q = 0; q < ndev && g->p2p; ++q) {
                    if (devs[q] == devs[p]) continue;
                    int can = 0;
                    CGX_CUDA(cudaDeviceCanAccessPeer(&can, devs[p], devs[q]));
                    if (!can) {
                        g->p2p = false;
                        g->p2p_why = "device " + std::to_string(devs[p]) + " cannot map device " + std::to_string(devs[q]);
                        break;
                    }
                    const cudaError_t e = cudaDeviceEnablePeerAccess(devs[q], 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled)
                        cudaGetLastError();
                    else
                        CGX_CUDA(e);
                }
            }
            for (int p = 0; p < ndev; ++p) {
                CGX_CUDA(cudaSetDevice(devs[p]));
                CGX_CUDA(cudaEventCreateWithFlags(&g->ev_sx[(size_t)p], cudaEventDisableTiming));
                CGX_CUDA(cudaEventCreateWithFlags(&g->ev_z[(size_t)p], cudaEventDisableTiming));
            }
        } catch (...) {
            for (int p = 0; p < ndev; ++p) {
                if (g->ev_sx[(size_t)p]) cudaEventDestroy(g->ev_sx[(size_t)p]);
                if (g->ev_z[(size_t)p]) cudaEventDestroy(g->ev_z[(size_t)p]);
                if (g->comm[(size_t)p]) N.CommDestroy(g->comm[(size_t)p]);
            }
            for (auto* c : g->ctx)
                if (c) cgx_free(c);
            delete g;
            throw;
        }
        *out = g;
    });
}

int cgx_group_free(cgx_group* g) {
    return gguard([&] {
        if (!g) return;
        g->threads.reset();
        for (int p = 0; p < g->P; ++p) {  // (peers write each other's buffers: quiesce all first)
            cudaSetDevice(g->dev[(size_t)p]);
            cudaDeviceSynchronize();
        }
        for (int p = 0; p < g->P; ++p) {
            cudaSetDevice(g->dev[(size_t)p]);
            for (auto* b : {&g->sx[(size_t)p], &g->slice[(size_t)p], &g->zp[(size_t)p], &g->zg[(size_t)p],
                            &g->rp[(size_t)p], &g->land[(size_t)p], &g->zslot[(size_t)p]})
                b->release();
            cudaEventDestroy(g->ev_sx[(size_t)p]);
            cudaEventDestroy(g->ev_z[(size_t)p]);
            if (g->comm[(size_t)p]) nccl().CommDestroy(g->comm[(size_t)p]);
            cgx_free(g->ctx[(size_t)p]);
        }
        delete g;
    });
}

int cgx_group_size(const cgx_group* g) { return g ? g->P : 0; }

int cgx_group_supports(const cgx_group* g, int combine) {
    if (!g) return 0;
    if (combine == CGX_COMBINE_P2P) return g->p2p ? 1 : 0;
    if (combine == CGX_COMBINE_Z || combine == CGX_COMBINE_G || combine == CGX_COMBINE_SX) return g->have_nccl ? 1 : 0;
    return 0;
}

int cgx_group_stats(const cgx_group* g, int64_t* fused_sketches, int64_t* copied_sketches) {
    return gguard([&] {
        if (!g) fail(CGX_EINVAL, "cgx_group_stats: null group");
        int64_t f = 0, c = 0;
        for (const cgx_ctx* x : g->ctx) {
            f += x->seg_fused;
            c += x->seg_copied;
        }
        if (fused_sketches) *fused_sketches = f;
        if (copied_sketches) *copied_sketches = c;
    });
}

int cgx_group_context(cgx_group* g, int rank, cgx_ctx** out) {
    return gguard([&] {
        if (!g || !out || rank < 0 || rank >= g->P) fail(CGX_EINVAL, "cgx_group_context: bad rank");
        *out = g->ctx[(size_t)rank];
    });
}

int cgx_group_countgauss_new(cgx_group* g, uint64_t t_seed, int64_t m, int64_t buckets, int64_t input_dim,
                             cgx_gxform** out) {
    return gguard([&] {
        if (!g || !out) fail(CGX_EINVAL, "cgx_group_countgauss_new: null argument");
        std::lock_guard<std::mutex> group_lock(g->mu);
        if (m < 1 || buckets < 1 || input_dim < 1)
            fail(CGX_EINVAL, "countgauss_new: m, buckets and input_dim must be >= 1");
        auto* t = new cgx_gxform;
        t->g = g;
        t->m = m;
        t->B = buckets;
        t->n = input_dim;
        t->xf.assign((size_t)g->P, nullptr);
        t->r0.assign((size_t)g->P, 0);
        t->r1.assign((size_t)g->P, 0);
        try {
            each_rank(g, [&](int p) {
                shard(input_dim, g->P, p, &t->r0[(size_t)p], &t->r1[(size_t)p]);
                ok_or_throw(cgx_countgauss_new_shard(g->ctx[(size_t)p], t_seed, m, buckets, input_dim, t->r0[(size_t)p],
                                                     t->r1[(size_t)p] - t->r0[(size_t)p], &t->xf[(size_t)p]));
                ok_or_throw(cgx_synchronize(g->ctx[(size_t)p], nullptr));
            });
        } catch (...) {
            for (auto* x : t->xf)
                if (x) cgx_xform_free(x);
            delete t;
            throw;
        }
        *out = t;
    });
}

int cgx_gxform_free(cgx_gxform* t) {
    return gguard([&] {
        if (!t) return;
        for (auto* x : t->xf)
            if (x) cgx_xform_free(x);
        delete t;
    });
}

int cgx_gxform_shard(const cgx_gxform* t, int rank, int64_t* row0, int64_t* rows) {
    return gguard([&] {
        if (!t || rank < 0 || rank >= t->g->P) fail(CGX_EINVAL, "cgx_gxform_shard: bad rank");
        if (row0) *row0 = t->r0[(size_t)rank];
        if (rows) *rows = t->r1[(size_t)rank] - t->r0[(size_t)rank];
    });
}

int cgx_group_countgauss_apply_dense(cgx_group* g, const cgx_gxform* t, const void* x, int dtype, int layout,
                                     int64_t ld, int64_t n, int64_t d, int x_mem, double* z, int z_mem, int combine) {
    return gguard([&] {
        if (!g || !t || t->g != g) fail(CGX_EINVAL, "cgx_group: null group or transform of another group");
        std::lock_guard<std::mutex> group_lock(g->mu);
        check_mode(g, combine);
        if (n != t->n)
            fail(CGX_EINVAL, "countsketch_apply: X has " + std::to_string(n) + " rows, sketch expects " +
                                 std::to_string(t->n));
        if (d < 1) fail(CGX_EINVAL, "cgx_group: X must have at least one column");
        if (layout != CGX_COL_MAJOR && layout != CGX_ROW_MAJOR) fail(CGX_EINVAL, "cgx: bad layout");
        const size_t es = dtype == CGX_F32 ? 4 : 8;
        auto shard_of = [&](int p, int64_t* rows) -> const void* {
            const int64_t r0 = t->r0[(size_t)p];
            *rows = t->r1[(size_t)p] - r0;
            if (x_mem == CGX_MEM_DEVICE) return ((const void* const*)x)[p];  // rank p's shard on its device
            return (const char*)x + es * (size_t)(layout == CGX_COL_MAJOR ? r0 : r0 * ld);
        };
        if (combine == CGX_COMBINE_P2P) {
            apply_p2p(g, t, d, [&](int p, cgx_ctx* c, cgx_xform* xf, double* out) {
                int64_t rows = 0;
                const void* xp = shard_of(p, &rows);
                ok_or_throw(cgx_countsketch_apply_dense(c, xf, xp, dtype, layout, ld, rows, d, x_mem, out, CGX_ROW_MAJOR,
                                                        CGX_MEM_DEVICE, nullptr));
            }, z, z_mem, (double* const*)z);
            return;
        }
        each_rank(g, [&](int p) {
            int64_t rows = 0;
            const void* xp = shard_of(p, &rows);
            const int64_t lp = ld;
            partial_rank(g, t, p, d, combine, [&](cgx_ctx* c, cgx_xform* xf, double* out, bool both) {
                if (both)
                    ok_or_throw(cgx_countgauss_apply_dense(c, xf, xp, dtype, layout, lp, rows, d, x_mem, out,
                                                           CGX_MEM_DEVICE, nullptr));
                else
                    ok_or_throw(cgx_countsketch_apply_dense(c, xf, xp, dtype, layout, lp, rows, d, x_mem, out,
                                                            CGX_ROW_MAJOR, CGX_MEM_DEVICE, nullptr));
            });
            combine_rank(g, t, p, d, combine, z, z_mem, (double* const*)z);
        });
    });
}

int cgx_group_countgauss_apply_csr(cgx_group* g, const cgx_gxform* t, const int64_t* rowptr, const void* cols,
                                   int idx_type, const void* vals, int dtype, int64_t n, int64_t d, int64_t nnz,
                                   double* z, int z_mem, int combine) {
    return gguard([&] {
        if (!g || !t || t->g != g) fail(CGX_EINVAL, "cgx_group: null group or transform of another group");
        std::lock_guard<std::mutex> group_lock(g->mu);
        check_mode(g, combine);
        if (n != t->n)
            fail(CGX_EINVAL, "countsketch_apply: X has " + std::to_string(n) + " rows, sketch expects " +
                                 std::to_string(t->n));
        if (d < 1 || nnz < 0) fail(CGX_EINVAL, "cgx_group: bad CSR sizes");
        if (!rowptr || rowptr[0] != 0 || rowptr[n] != nnz) fail(CGX_EINVAL, "cgx_group: row offsets must run 0..nnz");
        const size_t is = idx_type == CGX_I32 ? 4 : 8, vs = dtype == CGX_F32 ? 4 : 8;
        // Rank p's shard: its row offsets as they stand in the caller's array (ctx->csr_base tells
        // the kernels they count from the caller's element 0 -- copying and rebasing 8 B per row
        // on the host cost c3 more than its whole apply), its nonzeros the part of cols / vals
        // from rowptr[r0] on; all staged by the apply (pipelined, narrowed).
        struct Base {  // csr_base only around this rank's call
            cgx_ctx* c;
            Base(cgx_ctx* cc, int64_t b) : c(cc) { c->csr_base = b; }
            ~Base() { c->csr_base = 0; }
        };
        if (combine == CGX_COMBINE_P2P) {
            apply_p2p(g, t, d, [&](int p, cgx_ctx* c, cgx_xform* xf, double* out) {
                const int64_t r0 = t->r0[(size_t)p], rows = t->r1[(size_t)p] - r0;
                const int64_t q0 = rowptr[r0], q1 = rowptr[r0 + rows];
                Base base(c, q0);
                ok_or_throw(cgx_countsketch_apply_csr(c, xf, rowptr + r0, (const char*)cols + is * (size_t)q0, idx_type,
                                                      (const char*)vals + vs * (size_t)q0, dtype, rows, d, q1 - q0,
                                                      CGX_MEM_HOST, out, CGX_ROW_MAJOR, CGX_MEM_DEVICE, nullptr));
            }, z, z_mem, (double* const*)z);
            return;
        }
        each_rank(g, [&](int p) {
            const int64_t r0 = t->r0[(size_t)p], rows = t->r1[(size_t)p] - r0;
            const int64_t q0 = rowptr[r0], q1 = rowptr[r0 + rows];
            const int64_t* rpp = rowptr + r0;
            const void* cp = (const char*)cols + is * (size_t)q0;
            const void* vp = (const char*)vals + vs * (size_t)q0;
            Base base(g->ctx[(size_t)p], q0);
            partial_rank(g, t, p, d, combine, [&](cgx_ctx* c, cgx_xform* xf, double* out, bool both) {
                if (both)
                    ok_or_throw(cgx_countgauss_apply_csr(c, xf, rpp, cp, idx_type, vp, dtype, rows, d, q1 - q0,
                                                         CGX_MEM_HOST, out, CGX_MEM_DEVICE, nullptr));
                else
                    ok_or_throw(cgx_countsketch_apply_csr(c, xf, rpp, cp, idx_type, vp, dtype, rows, d, q1 - q0,
                                                          CGX_MEM_HOST, out, CGX_ROW_MAJOR, CGX_MEM_DEVICE, nullptr));
            });
            combine_rank(g, t, p, d, combine, z, z_mem, (double* const*)z);
        });
    });
}

} // extern "C"
