// Micro-test of a single tcgen05.mma with MN-major SW128 operands: tf32 vs bf16.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

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

// KIND 0 tf32 (es 4, K 8), 1 bf16 (es 2, K 16). A: 128 x K MN-major, B: 32 x K MN-major. SW128.
template <int KIND>
__global__ void micro(const float *Ag /*[K][128]*/, const float *Bg /*[K][NB]*/, float *D /*[128][NB]*/, int amaj, int bmaj, int fmt_override) {
    constexpr int ES = KIND == 1 ? 2 : 4, KK = KIND == 1 ? 16 : 8;
    __shared__ __align__(1024) uint8_t sA[128 * 16 * 4];
    __shared__ __align__(1024) uint8_t sB[32 * 16 * 4];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // fill A: element (m,k): MN-major SW128: atom a = m / (128/ES) (1024 B per 8 k-rows) ; groups of 8 k rows at SBO
    const int AW = 128 / ES;  // elements per 128-B row
    const int A_ATOM_BYTES = KK * 128;  // one M atom spans all K rows (K/8 groups * 1024)
    for (int i = tid; i < 128 * KK; i += blockDim.x) {
        int m = i % 128, k = i / 128;
        int a = m / AW, col = (m % AW) * ES;
        int kg = k / 8, kr = k % 8;
        int chunk = col / 16, off = col % 16;
        int addr = a * A_ATOM_BYTES + kg * 1024 + kr * 128 + ((chunk ^ kr) * 16) + off;
        if (fmt_override == -2) addr = a * A_ATOM_BYTES + (k / 4) * 512 + (k % 4) * 128 + (((col / 32) ^ (k % 4)) * 32) + col % 32;
        float v = Ag[k * 128 + m];
        if (ES == 4) *reinterpret_cast<float *>(sA + addr) = v;
        else *reinterpret_cast<__nv_bfloat16 *>(sA + addr) = __float2bfloat16(v);
    }
    const int BWE = 128 / ES;  // B: N=32 -> ES=4: 128 B one atom; ES=2: 64 B (use SW128 with 64 elements? keep N = 32 -> 64 B)
    constexpr int NB = 128 / ES;
    for (int i = tid; i < NB * KK; i += blockDim.x) {
        int n = i % NB, k = i / NB;
        int col = n * ES;  // < 128
        int kg = k / 8, kr = k % 8;
        int chunk = col / 16, off = col % 16;
        int addr = kg * 1024 + kr * 128 + ((chunk ^ kr) * 16) + off;
        if (fmt_override == -2) addr = (k / 4) * 512 + (k % 4) * 128 + (((col / 32) ^ (k % 4)) * 32) + col % 32;
        float v = Bg[k * NB + n];
        if (ES == 4) *reinterpret_cast<float *>(sB + addr) = v;
        else *reinterpret_cast<__nv_bfloat16 *>(sB + addr) = __float2bfloat16(v);
    }
    (void)BWE;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (tid == 0) {
        uint32_t fmt = fmt_override >= 0 ? fmt_override : (KIND == 1 ? 1u : 2u);
        const uint32_t lt = fmt_override == -2 ? 1u : 2u, sbo = fmt_override == -2 ? 512u : 1024u;
        uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) | (((uint32_t)NB >> 3) << 17) | ((128u >> 4) << 24);
        uint64_t ad = smem_desc(smem_u32(sA), A_ATOM_BYTES, sbo, lt);
        uint64_t bd = smem_desc(smem_u32(sB), 4096, sbo, lt);
        if (KIND == 1)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(0));
        else
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    // wait
    {
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) D[(warp * 32 + lane) * NB + i] = __uint_as_float(v[i]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
    }
}

template <int KIND>
void run(int amaj, int bmaj, int fmt_override) {
    const int KK = KIND == 1 ? 16 : 8;
    const int NB = KIND == 1 ? 64 : 32;
    float hA[16 * 128], hB[16 * 64], hD[128 * 64];
    for (int k = 0; k < KK; ++k) for (int m = 0; m < 128; ++m) hA[k * 128 + m] = (float)((m * 7 + k * 3) % 5) - 2.f;
    for (int k = 0; k < KK; ++k) for (int n = 0; n < NB; ++n) hB[k * NB + n] = (float)((n * 5 + k) % 3) - 1.f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xff, sizeof hD);
    micro<KIND><<<1, 128>>>(dA, dB, dD, amaj, bmaj, fmt_override);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    double err = 0, ref2 = 0; int zeros = 0;
    for (int m = 0; m < 128; ++m) for (int n = 0; n < 32; ++n) {
        double s = 0; for (int k = 0; k < KK; ++k) s += (double)hA[k * 128 + m] * hB[k * NB + n];
        err += (hD[m * NB + n] - s) * (hD[m * NB + n] - s); ref2 += s * s; zeros += hD[m * NB + n] == 0.f;
    }
    printf("KIND=%d amaj=%d bmaj=%d fmt=%d: %s relerr=%.3e zeros=%d D[0][0..3]=%g %g %g %g\n", KIND, amaj, bmaj, fmt_override,
           cudaGetErrorString(e), sqrt(err / ref2), zeros, hD[0], hD[1], hD[2], hD[3]);
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

int main() {
    run<1>(1, 1, -1);
    run<0>(1, 1, -1);
    run<0>(1, 1, -2);
    return 0;
}
