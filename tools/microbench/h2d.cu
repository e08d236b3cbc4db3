// h2d.cu -- measurement tool (not product code): ways to move a caller's PAGEABLE host
// array (the reference's std::vector-backed DenseMatrix) into HBM, for the drop-in's
// as-is-API path.  Prints GB/s for: plain cudaMemcpy from pageable memory; from pinned
// memory; cudaHostRegister + copy + unregister of the pageable array; and a pipeline that
// stages pageable -> pinned chunks with T host threads while the DMA engine drains the
// previous chunks.
// Build: make -C tools/microbench h2d
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
    const size_t bytes = (size_t)(argc > 1 ? atof(argv[1]) : 4.0) * (1ull << 30);
    char* host = (char*)malloc(bytes);
    for (size_t i = 0; i < bytes; i += 4096) host[i] = (char)i;  // fault the pages in
    memset(host, 1, bytes);
    char* dev;
    cudaMalloc(&dev, bytes);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    double t;
    for (int rep = 0; rep < 2; ++rep) {
        t = now();
        cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice);
        t = now() - t;
    }
    printf("pageable cudaMemcpy: %.1f GB/s (%.1f ms)\n", bytes / t / 1e9, t * 1e3);

    char* pin;
    cudaMallocHost(&pin, bytes);
    memset(pin, 1, bytes);
    for (int rep = 0; rep < 2; ++rep) {
        t = now();
        cudaMemcpy(dev, pin, bytes, cudaMemcpyHostToDevice);
        t = now() - t;
    }
    printf("pinned cudaMemcpy: %.1f GB/s (%.1f ms)\n", bytes / t / 1e9, t * 1e3);
    cudaFreeHost(pin);

    for (int rep = 0; rep < 2; ++rep) {
        t = now();
        double t0 = now();
        cudaHostRegister(host, bytes, cudaHostRegisterReadOnly);
        double treg = now() - t0;
        cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice);
        t0 = now();
        cudaHostUnregister(host);
        double tun = now() - t0;
        t = now() - t;
        printf("register+copy+unregister: %.1f GB/s (%.1f ms; register %.1f ms, unregister %.1f ms)\n", bytes / t / 1e9,
               t * 1e3, treg * 1e3, tun * 1e3);
    }

    // staged pipeline: chunk c is memcpy'd by T threads into pinned slot c % S, then DMA'd
    for (size_t chunk : {(size_t)8 << 20, (size_t)32 << 20}) {
        const int S = 4;
        char* slots;
        cudaMallocHost(&slots, chunk * S);
        cudaEvent_t ev[S];
        for (int s = 0; s < S; ++s) cudaEventCreateWithFlags(&ev[s], cudaEventDisableTiming);
        for (int T : {1, 2, 4, 8, 12}) {
            for (int rep = 0; rep < 2; ++rep) {
                t = now();
                const size_t nchunks = (bytes + chunk - 1) / chunk;
                for (size_t c = 0; c < nchunks; ++c) {
                    const int s = (int)(c % S);
                    if (c >= (size_t)S) cudaEventSynchronize(ev[s]);
                    const size_t off = c * chunk, len = std::min(chunk, bytes - off);
                    std::vector<std::thread> th;
                    const size_t per = (len + T - 1) / T;
                    for (int k = 0; k < T; ++k) {
                        const size_t a = k * per, b = std::min(len, a + per);
                        if (a < b) th.emplace_back([=] { memcpy(slots + s * chunk + a, host + off + a, b - a); });
                    }
                    for (auto& x : th) x.join();
                    cudaMemcpyAsync(dev + off, slots + s * chunk, len, cudaMemcpyHostToDevice, st);
                    cudaEventRecord(ev[s], st);
                }
                cudaStreamSynchronize(st);
                t = now() - t;
            }
            printf("staged %zu MB chunks, %d threads: %.1f GB/s (%.1f ms)\n", chunk >> 20, T, bytes / t / 1e9, t * 1e3);
        }
        cudaFreeHost(slots);
    }
    // raw host memcpy bandwidth with T threads (pageable -> pageable)
    char* h2 = (char*)malloc(bytes);
    memset(h2, 0, bytes);
    for (int T : {1, 4, 8, 16}) {
        t = now();
        std::vector<std::thread> th;
        const size_t per = (bytes + T - 1) / T;
        for (int k = 0; k < T; ++k) {
            const size_t a = k * per, b = std::min(bytes, a + per);
            th.emplace_back([=] { memcpy(h2 + a, host + a, b - a); });
        }
        for (auto& x : th) x.join();
        t = now() - t;
        printf("host memcpy %d threads: %.1f GB/s\n", T, bytes / t / 1e9);
    }
    return 0;
}
