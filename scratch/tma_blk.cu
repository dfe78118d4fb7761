// Micro-benchmark: per-SM TMA throughput for the span-kernel pattern -- per "row"
// one dY slab box (3-D, 16 KB) and/or NB boxes of G 4-KB blocks (4-D map over a
// block array, SW128_32B), ring of S stages, one producer thread, one consumer
// thread that only waits and releases.  148 CTAs.  Reports GB/s and cycles/row.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}
struct Maps { CUtensorMap m[4]; };
__global__ void kern(const __grid_constant__ CUtensorMap tdy, const __grid_constant__ Maps mv, int rows, int nb, int G,
                     int S, int stage_bytes, int use_dy, int nmaps, int nblocks_total, int nt, long long *cyc) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + S * stage_bytes);
    uint64_t *empty = full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t bytes = (use_dy ? 16384u : 0u) + (uint32_t)(nb * G * 4096);
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        int stage = 0; uint32_t ph = 0;
        unsigned h = blockIdx.x * 2654435761u;
        for (int r = 0; r < rows; ++r) {
            mbar_wait(empty + stage, ph ^ 1);
            uint32_t bar = smem_u32(full + stage);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            uint32_t dst = smem_u32(smem + stage * stage_bytes);
            if (use_dy) {
                int row = (blockIdx.x / nt) * rows + r;
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                             ::"r"(dst), "l"((uint64_t)&tdy), "r"(0), "r"(row * 32), "r"((int)(blockIdx.x % nt) * 4), "r"(bar) : "memory");
                dst += 16384;
            }
            for (int i = 0; i < nb; ++i) {
                h = h * 1664525u + 1013904223u;
                int blk = (int)(h % (unsigned)(nblocks_total - G));
                const CUtensorMap *m = &mv.m[i % nmaps];
                asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {0, 0, 0, %2}], [%3];"
                             ::"r"(dst), "l"((uint64_t)m), "r"(blk), "r"(bar) : "memory");
                dst += G * 4096;
            }
            if (++stage == S) { stage = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int stage = 0; uint32_t ph = 0;
        for (int r = 0; r < rows; ++r) {
            mbar_wait(full + stage, ph);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + stage)) : "memory");
            if (++stage == S) { stage = 0; ph ^= 1; }
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
}

int main(int argc, char **argv) {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const int M = 25088, N = 1536, NBLK = 4704 * 2;
    float *dy, *vals; long long *cyc;
    cudaMalloc(&dy, (size_t)M * N * 4); cudaMalloc(&vals, (size_t)NBLK * 4096); cudaMalloc(&cyc, 160 * 8);
    cudaMemset(dy, 0, (size_t)M * N * 4); cudaMemset(vals, 0, (size_t)NBLK * 4096);
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUtensorMap tdy;
    cuuint64_t dd[3] = {32, (cuuint64_t)M, (cuuint64_t)N / 32}, ds[2] = {(cuuint64_t)N * 4, 128};
    cuuint32_t db[3] = {32, 32, 4};
    enc(&tdy, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dy, dd, ds, db, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    struct Case { int nb, G, use_dy, nmaps, S; const char *name; } cases[] = {
        {0, 1, 1, 1, 5, "dY 16KB only"},
        {3, 1, 0, 1, 5, "3 x 4KB blocks, 1 map"},
        {3, 1, 0, 3, 5, "3 x 4KB blocks, 3 maps"},
        {1, 4, 0, 1, 5, "1 x 16KB (G=4)"},
        {3, 1, 1, 1, 5, "dY + 3 x 4KB"},
        {3, 1, 1, 3, 5, "dY + 3 x 4KB, 3 maps"},
        {6, 1, 1, 1, 3, "dY + 6 x 4KB (S=3)"},
        {1, 2, 1, 1, 5, "dY + 1 x 8KB"},
        {8, 1, 0, 1, 5, "8 x 4KB"},
    };
    const int rows = 65, nt = 12, ctas = 144;
    for (auto &c : cases) {
        Maps mv;
        for (int i = 0; i < 4; ++i) {
            cuuint64_t vd[4] = {32, 32, 1, (cuuint64_t)NBLK}, vs[3] = {128, 128, 4096};
            cuuint32_t vb[4] = {32, 32, 1, (cuuint32_t)c.G};
            enc(&mv.m[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, vals, vd, vs, vb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        int sb = ((c.use_dy ? 16384 : 0) + c.nb * c.G * 4096 + 1023) & ~1023;
        int smem = c.S * sb + 2048;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int w = 0; w < 2; ++w) kern<<<ctas, 64, smem>>>(tdy, mv, rows, c.nb, c.G, c.S, sb, c.use_dy, c.nmaps, NBLK, nt, cyc);
        cudaEventRecord(e0);
        const int R = 10;
        for (int w = 0; w < R; ++w) kern<<<ctas, 64, smem>>>(tdy, mv, rows, c.nb, c.G, c.S, sb, c.use_dy, c.nmaps, NBLK, nt, cyc);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long hc[160]; cudaMemcpy(hc, cyc, ctas * 8, cudaMemcpyDeviceToHost);
        double us = ms * 1e3 / R;
        double bytes = (double)ctas * rows * ((c.use_dy ? 16384 : 0) + c.nb * c.G * 4096);
        printf("%-28s %7.1f us  %6.0f GB/s  %6.0f cyc/row  err=%s\n", c.name, us, bytes / us / 1e3, (double)hc[0] / rows,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
