// B-operand load pattern micro-benchmark: 144 CTAs = 12 groups x 12 "n-tiles"; the 12 CTAs of a
// group stream the SAME sequence of 4 KB blocks (values array, L2-resident) with 4-D TMA boxes of G
// blocks into a ring of S slots.  Reports aggregate delivered bytes/s (L2 -> SM).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__global__ void kb(const __grid_constant__ CUtensorMap tm, int nblocks_per_cta, int G, int S, int slot_bytes, int groups) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + S * slot_bytes);
    uint64_t *empty = full + S;
    const int grp = blockIdx.x % groups;  // CTAs with the same grp read the same blocks
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(full + s)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(empty + s)));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int iters = nblocks_per_cta / G;
    if (threadIdx.x == 0) {
        int st = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(empty + st, ph ^ 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + st)), "r"(G * 4096) : "memory");
            const int blk = grp * nblocks_per_cta + i * G;
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                ::"r"(smem_u32(smem + st * slot_bytes)), "l"((uint64_t)&tm), "r"(0), "r"(0), "r"(0), "r"(blk), "r"(smem_u32(full + st)) : "memory");
            if (++st == S) { st = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int st = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(full + st, ph);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + st)) : "memory");
            if (++st == S) { st = 0; ph ^= 1; }
        }
    }
}
int main() {
    const int nnzb = 4704;  // C2: 19.3 MB of fp32 32x32 blocks
    float *d; cudaMalloc(&d, (size_t)nnzb * 4096); cudaMemset(d, 0, (size_t)nnzb * 4096);
    void *f = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    for (int G : {1, 2, 4, 8}) for (int S : {4, 8, 16}) for (int groups : {12, 144}) {
        CUtensorMap tm;
        cuuint64_t dims[4] = {32, 32, 1, (cuuint64_t)nnzb};
        cuuint64_t str[3] = {128, 128, 4096};
        cuuint32_t box[4] = {32, 32, 1, (cuuint32_t)G};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) { printf("enc fail\n"); continue; }
        const int per_cta = (nnzb / groups) / G * G;  // groups of CTAs partition the blocks
        const int slot = G * 4096;
        const int smem = S * slot + 1024 + 512;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(e0);
            kb<<<144, 64, smem>>>(tm, per_cta, G, S, slot, groups);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep && ms < best) best = ms;
        }
        double bytes = 144.0 * per_cta * 4096;
        printf("G=%d S=%2d groups=%3d: %.1f us  %.0f GB/s delivered (%s)\n", G, S, groups, best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
