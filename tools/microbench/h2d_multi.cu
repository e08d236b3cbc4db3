// h2d_multi.cu -- measurement tool (not product code): pinned host -> HBM copy rate of one
// 2 GB cudaMemcpyAsync against the same bytes split into chunks over 1, 2 or 4 streams
// (does a second copy engine lift the e2e path's H2D rate?).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

int main() {
    const size_t bytes = (size_t)2 << 30;
    char *pin, *dev;
    cudaMallocHost(&pin, bytes);
    memset(pin, 1, bytes);
    cudaMalloc(&dev, bytes);
    cudaStream_t st[4];
    for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int nst : {1, 2, 4})
        for (int chunks : {1, 8, 32}) {
            if (chunks < nst) continue;
            double best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                cudaDeviceSynchronize();
                auto t0 = std::chrono::steady_clock::now();
                const size_t cb = bytes / chunks;
                for (int c = 0; c < chunks; ++c)
                    cudaMemcpyAsync(dev + c * cb, pin + c * cb, cb, cudaMemcpyHostToDevice, st[c % nst]);
                cudaDeviceSynchronize();
                const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                best = t < best ? t : best;
            }
            printf("streams %d chunks %2d: %.1f GB/s (%.2f ms)\n", nst, chunks, bytes / best / 1e9, best * 1e3);
        }
    return 0;
}
