// dY slab streaming as the wgrad A loaders do it: 144 CTAs x 4 warps; CTA = one 128-column
// tile x a range of 32-row slabs; thread = one column, B=32 loads per slab, NSET slabs in flight.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__device__ __forceinline__ uint32_t ld(const float *p) {
    uint32_t v;
    if (MODE == 0) asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    else if (MODE == 1) asm volatile("ld.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
    else if (MODE == 2) asm volatile("ld.global.cs.b32 %0, [%1];" : "=r"(v) : "l"(p));
    else asm volatile("ld.global.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
template <int MODE, int NSET>
__global__ void __launch_bounds__(128, 1) k(const float *dY, int M, int N, int rows_per_cta, float *sink) {
    const int ntn = N / 128;
    const int nt = blockIdx.x % ntn, split = blockIdx.x / ntn;
    const float *col = dY + nt * 128 + threadIdx.x;
    const int r0 = split * rows_per_cta;
    uint32_t v[NSET][32];
    uint32_t acc = 0;
    int j = 0;
#pragma unroll
    for (int u = 0; u < NSET - 1; ++u)
#pragma unroll
        for (int kk = 0; kk < 32; ++kk) v[u][kk] = ld<MODE>(col + (size_t)((r0 + u) * 32 + kk) * N);
    for (j = 0; j < rows_per_cta; j += NSET) {
#pragma unroll
        for (int u = 0; u < NSET; ++u) {
            const int jn = j + u + NSET - 1;
            if (jn < rows_per_cta) {
#pragma unroll
                for (int kk = 0; kk < 32; ++kk) v[(u + NSET - 1) % NSET][kk] = ld<MODE>(col + (size_t)((r0 + jn) * 32 + kk) * N);
            }
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) acc ^= v[u][kk];
        }
    }
    if (acc == 0x12345678u) sink[0] = 1.f;
}
template <int MODE, int NSET>
void run(const float *dY, int M, int N, float *sink, const char *name) {
    const int ntn = N / 128, nsplit = 12, rows = M / 32 / nsplit;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k<MODE, NSET><<<ntn * nsplit, 128>>>(dY, M, N, rows, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
    }
    const double bytes = (double)ntn * nsplit * rows * 32 * 128 * 4;
    printf("%-22s NSET=%d: %.1f us  %.0f GB/s  (%s)\n", name, NSET, best * 1e3, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    const int M = 25088, N = 1536;
    float *dY, *sink; cudaMalloc(&dY, (size_t)M * N * 4); cudaMemset(dY, 1, (size_t)M * N * 4); cudaMalloc(&sink, 4);
    run<0, 2>(dY, M, N, sink, "nc.L1::no_allocate"); run<0, 3>(dY, M, N, sink, "nc.L1::no_allocate"); run<0, 4>(dY, M, N, sink, "nc.L1::no_allocate");
    run<1, 3>(dY, M, N, sink, "plain"); run<2, 3>(dY, M, N, sink, "cs"); run<3, 3>(dY, M, N, sink, "L1::no_allocate");
    return 0;
}
