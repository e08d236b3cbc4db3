// l2_red2.cu -- measurement tool (not product code): why the CSR record path's accumulate
// (csr_atomic.cu) reaches ~119 G fp64 REDs/s while l2_red.cu's random REDs into one fixed
// region reach 167-197 G/s.  Records (u32 address, f32 value) are streamed in partition
// order -- partition p's addresses uniform in an S-MB slice p of a 537 MB target -- and
// added with RED.ADD.F64 by a grid-stride kernel, with the target (a) memset beforehand,
// (b) zero-stored slice by slice just ahead of the REDs in the same kernel (queue order), (c)
// one fixed slice reused for every partition (addresses mod S MB: the l2_red.cu case).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void make(uint32_t* key, float* val, int64_t n, int64_t per_part, uint64_t slice_words, int fixed,
                     int randval) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = e / per_part;
        const uint64_t h = mix((uint64_t)e);
        key[e] = (uint32_t)((fixed ? 0 : p * slice_words) + h % slice_words);
        // constant 1.0 (l2_red.cu's records) or a full-mantissa value in (-1, 1)
        val[e] = randval ? (float)((double)(mix(h) >> 11) * 0x1.0p-52 - 1.0) : 1.0f;
    }
}

__global__ void red(const uint32_t* __restrict__ key, const float* __restrict__ val, int64_t n, double* acc) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(acc + __ldcs(key + e), (double)__ldcs(val + e));
}

// items of 4096 records in order, claimed from a counter (the accumulate kernel's queue
// without its zero items)
__global__ void red_queue(const uint32_t* __restrict__ key, const float* __restrict__ val, int64_t n, double* acc,
                          unsigned* ctr) {
    __shared__ unsigned s_it;
    for (;;) {
        if (threadIdx.x == 0) s_it = atomicAdd(ctr, 1u);
        __syncthreads();
        const int64_t base = (int64_t)s_it * 4096;
        __syncthreads();
        if (base >= n) break;
        uint32_t k[16];
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int64_t e = base + u * 256 + threadIdx.x;
            k[u] = e < n ? __ldcs(key + e) : 0xffffffffu;
            v[u] = e < n ? __ldcs(val + e) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u)
            if (k[u] != 0xffffffffu) atomicAdd(acc + k[u], (double)v[u]);
    }
}

int main(int argc, char** argv) {
    // optional ballast: allocate (and touch) this many GB first, as a process holding the
    // bench's inputs does
    const double ballast_gb = argc > 1 ? atof(argv[1]) : 0.0;
    if (ballast_gb > 0) {
        void* p;
        cudaMalloc(&p, (size_t)(ballast_gb * (1ull << 30)));
        cudaMemset(p, 1, (size_t)(ballast_gb * (1ull << 30)));
    }
    const int64_t n = 171798691;
    const int64_t total_words = (int64_t)537 << 17;  // 537 MB of doubles
    uint32_t* key;
    float* val;
    double* acc;
    unsigned* ctr;
    cudaMalloc(&key, 4 * n);
    cudaMalloc(&val, 4 * n);
    cudaMalloc(&acc, 8 * total_words);
    cudaMalloc(&ctr, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mb : {8}) {
        const uint64_t slice_words = (uint64_t)mb << 17;
        const int64_t parts = total_words / (int64_t)slice_words;
        const int64_t per_part = (n + parts - 1) / parts;
        for (int fixed : {0, 1, 2}) {
            make<<<148 * 8, 256>>>(key, val, n, per_part, slice_words, fixed == 1, fixed == 2);
            float ms_grid = 0, ms_q = 0;
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(acc, 0, 8 * total_words);
                cudaEventRecord(a);
                red<<<148 * 4, 256>>>(key, val, n, acc);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms_grid, a, b);
                cudaMemset(acc, 0, 8 * total_words);
                cudaMemset(ctr, 0, 4);
                cudaEventRecord(a);
                red_queue<<<148 * 4, 256>>>(key, val, n, acc, ctr);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms_q, a, b);
            }
            printf("slice %2d MB %s: grid-stride %.3f ms (%.0f G/s), queue %.3f ms (%.0f G/s)\n", mb,
                   fixed == 1 ? "fixed " : fixed == 2 ? "moving, random values" : "moving", ms_grid, n / ms_grid / 1e6, ms_q, n / ms_q / 1e6);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
