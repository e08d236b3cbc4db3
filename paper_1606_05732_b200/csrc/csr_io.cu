// csr_io.cu -- large CSR ingestion: a binary CSR container and a
// streamed file -> pinned host -> HBM loader, replacing the reference's text Matrix
// Market / CSV readers (src/io.cpp:72-136, 159-214), whose triplet sort
// (SparseMatrix::from_triplets, matrix.cpp:33-64) is O(nnz log nnz).
//
// File layout (little endian):  CsrFileHeader (64 B) | row_offsets int64[n+1] |
// col_indices int32/int64[nnz] | values f32/f64[nnz].  A file holds the CSR arrays exactly
// as the apply entry points take them, so loading is a straight copy.
//
// Device loads stream the three arrays in 64 MiB chunks through two pinned staging buffers:
// the read of chunk k+1 overlaps the H2D copy of chunk k (each buffer is reused only after
// its copy's event has completed), and each chunk is read by 8 threads (pread of 8 MiB
// slices) -- one thread copying out of the page cache tops out near 6-8 GB/s, below PCIe.
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace cgx {
namespace {

struct CsrFileHeader {
    char magic[8];  // "CGXCSR1\0"
    uint32_t version;
    int32_t idx_type;  // CGX_I32 / CGX_I64
    int32_t dtype;     // CGX_F32 / CGX_F64
    int32_t reserved0;
    int64_t n, d, nnz;
    int64_t reserved[2];
};
static_assert(sizeof(CsrFileHeader) == 64, "header is 64 bytes");

constexpr char kMagic[8] = {'C', 'G', 'X', 'C', 'S', 'R', '1', 0};
constexpr size_t kChunk = (size_t)64 << 20;
constexpr int kReaders = 8;

size_t idx_size(int t) { return t == CGX_I32 ? 4 : 8; }
size_t val_size(int t) { return t == CGX_F32 ? 4 : 8; }

struct File {
    FILE* f = nullptr;
    explicit File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

CsrFileHeader read_header(FILE* f, const char* path) {
    CsrFileHeader h;
    if (std::fread(&h, sizeof(h), 1, f) != 1 || std::memcmp(h.magic, kMagic, 8) != 0 || h.version != 1)
        fail(CGX_EINVAL, std::string("cgx_csr: not a CGXCSR1 file: ") + path);
    if ((h.idx_type != CGX_I32 && h.idx_type != CGX_I64) || (h.dtype != CGX_F32 && h.dtype != CGX_F64) || h.n < 0 ||
        h.d < 0 || h.nnz < 0)
        fail(CGX_EINVAL, std::string("cgx_csr: corrupt header: ") + path);
    return h;
}

} // namespace

void csr_save(const char* path, const int64_t* rowptr, const void* cols, int idx_type, const void* vals, int dtype,
              int64_t n, int64_t d, int64_t nnz) {
    if (idx_type != CGX_I32 && idx_type != CGX_I64) fail(CGX_EINVAL, "cgx_csr_save: idx_type must be CGX_I32 or CGX_I64");
    if (dtype != CGX_F32 && dtype != CGX_F64) fail(CGX_EINVAL, "cgx_csr_save: dtype must be CGX_F32 or CGX_F64");
    if (n < 0 || d < 0 || nnz < 0) fail(CGX_EINVAL, "cgx_csr_save: negative size");
    File out(path, "wb");
    if (!out.f) fail(CGX_EINVAL, std::string("cgx_csr_save: cannot open ") + path);
    CsrFileHeader h{};
    std::memcpy(h.magic, kMagic, 8);
    h.version = 1;
    h.idx_type = idx_type;
    h.dtype = dtype;
    h.n = n;
    h.d = d;
    h.nnz = nnz;
    bool ok = std::fwrite(&h, sizeof(h), 1, out.f) == 1;
    ok = ok && std::fwrite(rowptr, sizeof(int64_t), (size_t)(n + 1), out.f) == (size_t)(n + 1);
    if (nnz) {
        ok = ok && std::fwrite(cols, idx_size(idx_type), (size_t)nnz, out.f) == (size_t)nnz;
        ok = ok && std::fwrite(vals, val_size(dtype), (size_t)nnz, out.f) == (size_t)nnz;
    }
    if (!ok) fail(CGX_EINVAL, std::string("cgx_csr_save: write failed: ") + path);
}

void csr_info(const char* path, int64_t* n, int64_t* d, int64_t* nnz, int* idx_type, int* dtype) {
    File in(path, "rb");
    if (!in.f) fail(CGX_EINVAL, std::string("cgx_csr_info: cannot open ") + path);
    const CsrFileHeader h = read_header(in.f, path);
    if (n) *n = h.n;
    if (d) *d = h.d;
    if (nnz) *nnz = h.nnz;
    if (idx_type) *idx_type = h.idx_type;
    if (dtype) *dtype = h.dtype;
}

void csr_load(cgx_ctx* ctx, const char* path, int64_t* rowptr, void* cols, void* vals, int mem, cudaStream_t s) {
    File in(path, "rb");
    if (!in.f) fail(CGX_EINVAL, std::string("cgx_csr_load: cannot open ") + path);
    const CsrFileHeader h = read_header(in.f, path);
    struct Part {
        void* dst;
        size_t bytes;
    } parts[3] = {{rowptr, sizeof(int64_t) * (size_t)(h.n + 1)},
                  {cols, idx_size(h.idx_type) * (size_t)h.nnz},
                  {vals, val_size(h.dtype) * (size_t)h.nnz}};
    if (mem == CGX_MEM_HOST) {  // plain reads straight into the caller's arrays
        for (const Part& p : parts)
            if (p.bytes && std::fread(p.dst, 1, p.bytes, in.f) != p.bytes)
                fail(CGX_EINVAL, std::string("cgx_csr_load: truncated file: ") + path);
        return;
    }
    const int fd = fileno(in.f);
    // pread `len` bytes at file offset `pos` into buf with kReaders threads
    auto read_chunk = [&](char* buf, size_t len, off_t pos) {
        const size_t slice = (len + kReaders - 1) / kReaders;
        std::vector<std::thread> th;
        std::vector<int> ok(kReaders, 1);
        for (int t = 0; t < kReaders; ++t) {
            const size_t a = (size_t)t * slice;
            if (a >= len) break;
            const size_t b = std::min(len, a + slice);
            th.emplace_back([&, t, a, b] {
                size_t done = a;
                while (done < b) {
                    const ssize_t r = pread(fd, buf + done, b - done, pos + (off_t)done);
                    if (r <= 0) {
                        ok[t] = 0;
                        return;
                    }
                    done += (size_t)r;
                }
            });
        }
        for (auto& x : th) x.join();
        return std::all_of(ok.begin(), ok.end(), [](int v) { return v != 0; });
    };
    // two pinned staging buffers; buffer k is refilled only after its previous H2D completed
    if (ctx->pinned_bytes < 2 * kChunk) {
        if (ctx->pinned) CGX_CUDA(cudaFreeHost(ctx->pinned));
        ctx->pinned = nullptr;
        ctx->pinned_bytes = 0;
        CGX_CUDA(cudaMallocHost(&ctx->pinned, 2 * kChunk));
        ctx->pinned_bytes = 2 * kChunk;
    }
    cudaEvent_t ev[2];
    CGX_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CGX_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    bool used[2] = {false, false};
    int k = 0;
    off_t pos = (off_t)sizeof(CsrFileHeader);
    try {
        for (const Part& p : parts) {
            for (size_t off = 0; off < p.bytes; off += kChunk) {
                const size_t len = p.bytes - off < kChunk ? p.bytes - off : kChunk;
                char* buf = (char*)ctx->pinned + (size_t)k * kChunk;
                if (used[k]) CGX_CUDA(cudaEventSynchronize(ev[k]));
                if (!read_chunk(buf, len, pos)) fail(CGX_EINVAL, std::string("cgx_csr_load: truncated file: ") + path);
                pos += (off_t)len;
                CGX_CUDA(cudaMemcpyAsync((char*)p.dst + off, buf, len, cudaMemcpyHostToDevice, s));
                CGX_CUDA(cudaEventRecord(ev[k], s));
                used[k] = true;
                k ^= 1;
            }
        }
        CGX_CUDA(cudaStreamSynchronize(s));  // the staging buffers are reused by later calls
    } catch (...) {
        cudaStreamSynchronize(s);
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        throw;
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
}

} // namespace cgx
