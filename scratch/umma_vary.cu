// tcgen05.mma (A in TMEM, B MN-major tf32 from smem) issue cost when N and/or the
// B address change from one MMA to the next (as in the BSR wgrad main loop).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint32_t blo, uint32_t bhi, uint32_t idesc) {
    asm volatile("{\n.reg .pred p;\n.reg .b64 b;\nmov.b64 b, {%2, %3};\nelect.sync _|p, 0xffffffff;\n"
                 "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], b, %4, 1;\n}\n" ::"r"(d), "r"(a), "r"(blo), "r"(bhi), "r"(idesc));
}
// mode bit0: vary N (32/64/96/...); bit1: vary B address; bit2: vary D; bit3: words from smem via redux (like the kernel)
__global__ void k(int mode, int nmma, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    __shared__ uint32_t words[64];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 65536 / 4; i += blockDim.x) ((float *)sm)[i] = 0.f;
    if (tid < 64) {
        const uint32_t len = 1 + (tid * 7 % 3);          // 1..3 blocks
        const uint32_t col = (tid * 5 % 9) * 32;        // TMEM column
        const uint32_t slot = tid * 3 % 12;             // B slot
        words[tid] = col | (slot << 10) | (len << 22);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (warp == 1) {
        const uint64_t bd = smem_desc(smem_u32(sm), 4096, 512, 1);
        const uint32_t blo0 = (uint32_t)bd, bhi = (uint32_t)(bd >> 32);
        const uint32_t idesc0 = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((128u >> 4) << 24);
        const uint32_t a = tmem + 384;
        long long t0 = clock64();
        uint32_t wl = words[lane];
        for (int i = 0; i < nmma; i += 4) {
            uint32_t rw = __reduce_or_sync(0xffffffffu, lane == ((i >> 2) & 31) ? wl : 0u);
            if (!(mode & 8)) rw = (1u << 22);
            uint32_t d = tmem + ((mode & 4) ? (rw & 0x3FFu) : 0u);
            uint32_t blo = blo0 + ((mode & 2) ? ((rw >> 10) & 0xFFFu) * 256u : 0u);
            uint32_t idesc = idesc0 | (((mode & 1) ? ((rw >> 22) & 0x3Fu) * 32u : 32u) >> 3 << 17);
#pragma unroll
            for (int s = 0; s < 4; ++s) mma_ts(d, a + 8 * s, blo + s * 64, bhi, idesc);
        }
        long long t1 = clock64();
        __syncwarp();
        if (lane == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
        long long t2 = clock64();
        if (lane == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}
int main() {
    unsigned long long *d, h[2];
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    const int nm = 1024;
    const char *names[] = {"const", "vary N", "vary B", "vary N+B", "vary D", "vary N+D", "vary B+D", "vary all"};
    for (int mode = 8; mode < 16; ++mode) {
        k<<<1, 128, 65536 + 1024>>>(mode, nm, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%-9s: issue %.1f cyc/mma, complete %.1f cyc/mma  %s\n", names[mode & 7], (double)h[0] / nm, (double)h[1] / nm, cudaGetErrorString(e));
    }
    return 0;
}
