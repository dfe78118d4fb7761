// Micro-benchmark: TMA streaming of an M x N fp32 row-major matrix in boxes of
// (bw bytes wide) x (rows) with a ring of S stages; a consumer warp only waits and
// releases.  Measures achievable HBM bandwidth for the wgrad dY access pattern.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap *tm, uint64_t *bar, void *dst, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}

// CTA c handles column tile (c % ntn) of width tile_cols, rows [r0, r1) in steps of `rows`.
__device__ __forceinline__ void tma_load_3d(const CUtensorMap *tm, uint64_t *bar, void *dst, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)) : "memory");
}
__global__ void stream_kernel(const __grid_constant__ CUtensorMap tm, int ntn, int tile_cols, int box_cols, int rows,
                              int M, int nsplit, int S, int stage_bytes, int use3d) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + S * stage_bytes);
    uint64_t *empty = full + S;
    int nt = blockIdx.x % ntn, split = blockIdx.x / ntn;
    int nrb = M / rows;
    int Ib = (int)((int64_t)split * nrb / nsplit), Ie = (int)((int64_t)(split + 1) * nrb / nsplit);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nbox = tile_cols / box_cols;
    if (threadIdx.x == 0) {
        int st = 0; uint32_t ph = 0;
        for (int I = Ib; I < Ie; ++I) {
            mbar_wait(empty + st, ph ^ 1);
            mbar_arrive_expect_tx(full + st, stage_bytes);
            if (use3d & 1) tma_load_3d(&tm, full + st, smem + st * stage_bytes, 0, I * rows, nt * nbox);
            else
            for (int a = 0; a < nbox; ++a)
                tma_load_2d(&tm, full + st, smem + st * stage_bytes + a * (box_cols * 4 * rows), nt * tile_cols + a * box_cols, I * rows);
            if (++st == S) { st = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int st = 0; uint32_t ph = 0;
        for (int I = Ib; I < Ie; ++I) {
            mbar_wait(full + st, ph);
            if (use3d & 2)
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(empty + st)) : "memory");
            else
                mbar_arrive(empty + st);
            if (++st == S) { st = 0; ph ^= 1; }
        }
    }
}

int main() {
    const int M = 25088, N = 1536;
    float *d;
    cudaMalloc(&d, (size_t)M * N * 4 * 3);
    cudaMemset(d, 0, (size_t)M * N * 4 * 3);
    void *f = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    struct Cfg { int tile_cols, box_cols, rows, S, swz, use3d = 0; };
    std::vector<Cfg> cfgs = {
        {128, 32, 32, 4, 4, 1}, {128, 32, 32, 4, 4, 3}, {128, 32, 32, 8, 4, 1}, {128, 32, 32, 8, 4, 3},
        {128, 32, 32, 3, 4}, {128, 32, 32, 6, 4}, {128, 32, 32, 12, 4}, {128, 32, 32, 12, 0},
        {128, 32, 64, 6, 4}, {128, 32, 128, 3, 4}, {256, 32, 32, 6, 4}, {512, 32, 32, 4, 4},
        {1536, 32, 8, 4, 4}, {1536, 32, 16, 4, 4}, {128, 128, 32, 6, 0}, {128, 64, 32, 6, 0},
    };
    for (auto c : cfgs) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M * 3};
        cuuint64_t str[1] = {(cuuint64_t)N * 4};
        cuuint32_t box[2] = {(cuuint32_t)c.box_cols, (cuuint32_t)c.rows};
        cuuint32_t es[3] = {1, 1, 1};
        cuuint64_t dims3[3] = {(cuuint64_t)c.box_cols, (cuuint64_t)M * 3, (cuuint64_t)N / c.box_cols};
        cuuint64_t str3[2] = {(cuuint64_t)N * 4, (cuuint64_t)c.box_cols * 4};
        cuuint32_t box3[3] = {(cuuint32_t)c.box_cols, (cuuint32_t)c.rows, (cuuint32_t)(c.tile_cols / c.box_cols)};
        CUresult r = (c.use3d & 1) ? enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims3, str3, box3, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         c.swz == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) :
            enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         c.swz == 4 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); continue; }
        int ntn = N / c.tile_cols;
        int nsplit = sms / ntn; if (nsplit < 1) nsplit = 1;
        int stage_bytes = c.tile_cols * 4 * c.rows;
        int smem = c.S * stage_bytes + 1024 + 256;
        if (smem > 227 * 1024) { printf("skip smem %d\n", smem); continue; }
        cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        float best = 1e9;
        for (int rep = 0; rep < 6; ++rep) {
            int base = (rep % 3);
            CUtensorMap tm2 = tm;  // use the same map, shifted rows not needed: region size 3M; use M rows at offset
            (void)base;
            cudaEventRecord(e0);
            stream_kernel<<<ntn * nsplit, 64, smem>>>(tm2, ntn, c.tile_cols, c.box_cols, c.rows, M, nsplit, c.S, stage_bytes, c.use3d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        double gb = (double)M * N * 4 / 1e9;
        printf("3d=%d tile %4d box %3dx%3d S=%2d swz=%d grid=%d: %.1f us  %.0f GB/s  %s\n", c.use3d, c.tile_cols, c.box_cols, c.rows, c.S,
               c.swz, ntn * nsplit, best * 1e3, gb / (best * 1e-3), cudaGetErrorString(err));
    }
    return 0;
}
