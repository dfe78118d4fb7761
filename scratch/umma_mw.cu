// tcgen05.mma issue/throughput micro-benchmark: one thread issues NMMA MMAs
// (M=128, N=n, K=one k-step) from shared memory (MN-major, 128B swizzle variants),
// commits and waits; reports cycles per MMA.
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

template <int KIND, int TS>
__global__ void rate(int n, int nmma, int spread, int amaj, int bmaj, unsigned long long *out, int mdim) {
    __shared__ __align__(1024) uint8_t sA[16384];
    __shared__ __align__(1024) uint8_t sB[16384];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 16384 / 4; i += blockDim.x) { ((float *)sA)[i] = 0.f; ((float *)sB)[i] = 0.f; }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(spread ? spread : 1) : "memory");
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
    const int nw_issue = spread ? spread : 1;
    if ((tid & 31) == 0 && warp < nw_issue) {
        const uint32_t fmt = KIND == 1 ? 1u : 2u;
        const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
                               (((uint32_t)n >> 3) << 17) | (((uint32_t)mdim >> 4) << 24);
        const uint32_t lt = (KIND == 0 && amaj) ? 1u : 2u;
        const uint32_t sbo = (KIND == 0 && amaj) ? 512u : 1024u;
        const uint32_t lbo = KIND == 0 ? 1024u : 2048u;
        uint64_t ad = smem_desc(smem_u32(sA), lbo, sbo, lt);
        uint64_t bd = smem_desc(smem_u32(sB), lbo, sbo, lt);
        long long t0 = clock64();
        const uint32_t d0 = tmem + warp * 64u, d1 = d0, d2 = d0, d3 = d0;
        const uint32_t at = tmem + 384u;
#define MMA1(D)                                                                                                                              \
    do {                                                                                                                                   \
        if (TS) {                                                                                                                          \
            if (KIND == 1)                                                                                                                 \
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(D), "r"(at), "l"(bd), "r"(idesc), "r"(1)); \
            else                                                                                                                           \
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(D), "r"(at), "l"(bd), "r"(idesc), "r"(1)); \
        } else if (KIND == 1)                                                                                                              \
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(D), "l"(ad), "l"(bd), "r"(idesc), "r"(1)); \
        else                                                                                                                               \
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(D), "l"(ad), "l"(bd), "r"(idesc), "r"(1)); \
    } while (0)
        if (!TS && KIND == 0) {
            for (int i = 0; i < nmma / nw_issue; i += 8)
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %5, %6, %7, p;\n"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%1], %5, %6, %7, p;\n"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%2], %5, %6, %7, p;\n"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%3], %5, %6, %7, p;\n"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%0], %5, %6, %7, p;\n"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%1], %5, %6, %7, p;\n"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%2], %5, %6, %7, p;\n"
                             "tcgen05.mma.cta_group::1.kind::tf32 [%3], %5, %6, %7, p;\n}\n"
                             ::"r"(d0), "r"(d1), "r"(d2), "r"(d3), "r"(1), "l"(ad), "l"(bd), "r"(idesc));
        } else
        for (int i = 0; i < nmma / nw_issue; i += 4) {
            MMA1(d0); MMA1(d1); MMA1(d2); MMA1(d3);
        }
        long long t1 = clock64();
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
        long long t2 = clock64();
        if (warp == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
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
    const int nm = 512;
    for (int ts = 0; ts < 2; ++ts)
    for (int kind = 0; kind < 2; ++kind)
        for (int mdim : {128})
            for (int n : {32, 64})
                for (int spread : {1, 2, 4}) {
                    // TS: A from TMEM must be K-major (a_major = 0); B MN-major
                    const int amaj = ts ? 0 : 1;
                    if (kind == 0) { if (ts) rate<0, 1><<<1, 128>>>(n, nm, spread, amaj, 1, d, mdim); else rate<0, 0><<<1, 128>>>(n, nm, spread, amaj, 1, d, mdim); }
                    else { if (ts) rate<1, 1><<<1, 128>>>(n, nm, spread, amaj, 1, d, mdim); else rate<1, 0><<<1, 128>>>(n, nm, spread, amaj, 1, d, mdim); }
                    cudaError_t e = cudaDeviceSynchronize();
                    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                    printf("%s M=%d %s N=%3d spread=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (floor %.0f)\n",
                           ts ? "TS" : "SS", mdim, kind ? "bf16" : "tf32", n, spread, (double)h[0] / nm, (double)h[1] / nm, 128.0 * n / 256.0);
                }
    return 0;
}
