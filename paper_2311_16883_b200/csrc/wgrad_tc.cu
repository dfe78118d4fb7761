// wgrad_tc.cu -- BSR weight gradient on the 5th-generation tensor cores
// (row a6 of SURVEY §8a; BJ "TMA-fed tcgen05/TMEM block-sparse GEMM").
//
//   dW[J*b + c][n] = sum over stored blocks (I, J), sum over r < b of
//                    values(I,J)[r][c] * dY[I*b + r][n]
//
// Orientation: the MMA computes D = dW^T tile-wise,
//   D[n][kcol] (TMEM: 128 lanes = 128 columns n of dY, one TMEM column per
//   kcol of X) += A[n][r] * B[r][kcol]
// with A = the b x 128 slab of dY of block row I (MN-major: n contiguous,
// exactly dY's row-major layout) and B = the stored X blocks of that block
// row (MN-major: kcol contiguous, exactly the BSR block layout).  Every kept
// block becomes b/UMMA_K MMAs of shape 128 x b x UMMA_K into its own TMEM
// column range, so pruned blocks cost nothing; runs of adjacent kept blocks
// (consecutive in BSR storage, hence consecutive in shared memory) merge into
// one MMA with N = run * b <= 256.  Block rows without a kept block in the
// CTA's column range are never read.
//
// CTA = (128-column tile of dY) x (range of <= 512 kcols: TMEM columns) x
// (range of block rows: split-K).  Warp roles: warp 0 = TMA producer (one
// lane), warp 1 = MMA issuer (one lane), warp 2 = TMEM allocator, warps 4-7 =
// epilogue (tcgen05.ld -> fp32 stores, or red.global.add across splits).
// Shared-memory stages hold one block row each (A slab + its kept blocks),
// swizzled by TMA exactly as the UMMA descriptors expect (SW128 for dY; SW32 /
// SW64 / SW128 for blocks whose row is 32 / 64 / >=128 bytes wide).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "launch.h"

namespace bsrp {
namespace tc {

constexpr int kThreads = 256;
constexpr int kMetaBytes = 64;     // per stage: [0] = block count (255 = end), [1..] = relative J
constexpr int kSmemBudget = 227 * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Bounded wait: a pipeline bug traps (launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins > (1u << 26)) __trap();
    }
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap *tm, uint64_t *bar, void *dst, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

template <int KIND>
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    if constexpr (KIND == 1) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
    } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
            "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
    }
}

// UMMA shared-memory matrix descriptor (sm_100): start, leading-byte offset
// (stride between MN atoms for swizzled MN-major), stride-byte offset (between
// 8-row K groups), version 1, swizzle layout type.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

// Instruction descriptor: fp32 accumulate, A/B format (1 = bf16, 2 = tf32),
// both operands MN-major, M = 128, N = n.
template <int KIND>
__device__ __forceinline__ uint32_t instr_desc(uint32_t n) {
    constexpr uint32_t fmt = KIND == 1 ? 1u : 2u;
    return (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 15) | (1u << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24);
}

#define TMEM_LD16(taddr, v)                                                                                     \
    asm volatile(                                                                                               \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),       \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])  \
        : "r"(taddr))

__device__ __forceinline__ void tmem_st16_zero(uint32_t taddr) {
    const uint32_t z = 0;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(z)
        : "memory");
}

struct Params {
    const int32_t *rowptr, *colidx;
    float *dW;
    int64_t nbr, N, K;
    int nkr, nsplit, kr_blocks;  // kcol range = kr_blocks blocks
    int stages, stage_bytes, mode;  // mode: 0 store, 1 load-add-store, 2 red.add
    uint32_t tmem_cols;
};

template <int KIND, int B>
struct Cfg {
    static constexpr int ES = KIND == 1 ? 2 : 4;
    static constexpr int UK = KIND == 1 ? 16 : 8;           // MMA K per instruction
    static constexpr int AW = 128 / ES;                     // dY columns per 128-byte swizzle atom
    static constexpr int A_ATOMS = 128 / AW;                // atoms along M = 128
    static constexpr int A_BYTES = B * 128 * ES;            // b rows x 128 columns
    static constexpr int A_LBO = B * 128;                   // bytes between M atoms
    static constexpr int BW = (B * ES < 128) ? B * ES : 128;  // block row bytes per swizzle atom
    static constexpr int B_ATOMS = B * ES / BW;
    static constexpr int BLOCK_BYTES = B * B * ES;
    static constexpr int B_LBO = B * BW;                    // bytes between N atoms
    // MN-major tf32 operands only exist in the 128-byte swizzle with 32-byte
    // atomicity (UMMA layout type 1, TMA SWIZZLE_128B_ATOM_32B): 128-byte rows,
    // 32-byte chunks permuted by (row % 4), K groups of 4 rows.  bf16 uses the
    // plain SW32/64/128 layouts with K groups of 8 rows.
    static constexpr bool TF32 = KIND == 0;
    static constexpr int KGROUP = TF32 ? 4 : 8;             // K rows per swizzle group
    static constexpr int A_SBO = KGROUP * 128;              // bytes between K groups of A
    static constexpr uint32_t A_LAYOUT = TF32 ? 1u : 2u;
    static constexpr int A_KSTEP = UK * 128;                // bytes per MMA K step in A
    static constexpr int B_SBO = KGROUP * BW;               // bytes between K groups of B
    static constexpr int B_KSTEP = UK * BW;                 // bytes per MMA K step in B
    static constexpr uint32_t B_LAYOUT = TF32 ? 1u : BW == 128 ? 2u : BW == 64 ? 4u : 6u;  // SW128_32B / SW128 / SW64 / SW32
    static_assert(!TF32 || BW == 128, "tf32 MN-major operands need 128-byte block rows (b >= 32)");
    static constexpr int MAX_RUN = 256 / B;                 // blocks per MMA (N <= 256)
};

template <int KIND, int B>
__global__ void __launch_bounds__(kThreads, 1)
    wgrad_tc_kernel(const __grid_constant__ CUtensorMap tm_dy, const __grid_constant__ CUtensorMap tm_val, Params p) {
    using C = Cfg<KIND, B>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *meta = smem + (size_t)p.stages * p.stage_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(meta + p.stages * kMetaBytes);
    uint64_t *empty = full + p.stages;
    uint64_t *accfull = empty + p.stages;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(accfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int t = blockIdx.x;
    const int split = t % p.nsplit;
    t /= p.nsplit;
    const int kr = t % p.nkr;
    const int nt = t / p.nkr;
    const int n0 = nt * 128;
    const int nbc = (int)(p.K / B);
    const int J0 = kr * p.kr_blocks;
    const int nbJ = min(p.kr_blocks, nbc - J0);
    const int64_t Ib = (int64_t)split * p.nbr / p.nsplit, Ie = (int64_t)(split + 1) * p.nbr / p.nsplit;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dy)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_val)) : "memory");
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        mbar_init(accfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(p.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;

    // zero the accumulator columns this CTA owns (MMAs then always accumulate)
    if (warp >= 4) {
        const uint32_t lane_base = (uint32_t)((warp - 4) * 32) << 16;
        for (int c = 0; c < nbJ * B; c += 16) tmem_st16_zero(tmem + lane_base + c);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == 0 && lane == 0) {
        // ------------------------------------------------ TMA producer
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t I = Ib; I < Ie; ++I) {
            const int p0 = __ldg(p.rowptr + I), p1 = __ldg(p.rowptr + I + 1);
            int q0 = p0;
            while (q0 < p1 && __ldg(p.colidx + q0) < J0) ++q0;
            int q1 = q0;
            while (q1 < p1 && __ldg(p.colidx + q1) < J0 + nbJ) ++q1;
            const int cnt = q1 - q0;
            if (cnt == 0) continue;
            mbar_wait(empty + stage, phase ^ 1);
            uint8_t *m = meta + stage * kMetaBytes;
            m[0] = (uint8_t)cnt;
            for (int q = 0; q < cnt; ++q) m[1 + q] = (uint8_t)(__ldg(p.colidx + q0 + q) - J0);
            mbar_arrive_expect_tx(full + stage, (uint32_t)(C::A_BYTES + cnt * C::BLOCK_BYTES));
            uint8_t *sA = smem + (size_t)stage * p.stage_bytes;
            uint8_t *sB = sA + C::A_BYTES;
#pragma unroll
            for (int a = 0; a < C::A_ATOMS; ++a)
                tma_load_2d(&tm_dy, full + stage, sA + a * C::A_LBO, n0 + a * C::AW, (int)(I * B));
            for (int q = 0; q < cnt; ++q)
#pragma unroll
                for (int h = 0; h < C::B_ATOMS; ++h)
                    tma_load_2d(&tm_val, full + stage, sB + q * C::BLOCK_BYTES + h * C::B_LBO, h * (C::BW / C::ES),
                                (q0 + q) * B);
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
        mbar_wait(empty + stage, phase ^ 1);  // end marker
        meta[stage * kMetaBytes] = 255;
        mbar_arrive(full + stage);
    } else if (warp == 1 && lane == 0) {
        // ------------------------------------------------ MMA issuer
        int stage = 0;
        uint32_t phase = 0;
        for (;;) {
            mbar_wait(full + stage, phase);
            tc_fence_after();
            const uint8_t *m = meta + stage * kMetaBytes;
            const int cnt = m[0];
            if (cnt == 255) break;
            const uint32_t sA = smem_u32(smem + (size_t)stage * p.stage_bytes);
            const uint32_t sB = sA + C::A_BYTES;
            int q = 0;
            while (q < cnt) {
                const int J = m[1 + q];
                int L = 1;
                while (q + L < cnt && L < C::MAX_RUN && m[1 + q + L] == J + L) ++L;
                const uint32_t idesc = instr_desc<KIND>((uint32_t)(L * B));
#pragma unroll
                for (int s = 0; s < B / C::UK; ++s) {
                    const uint64_t ad = smem_desc(sA + s * C::A_KSTEP, C::A_LBO, C::A_SBO, C::A_LAYOUT);
                    const uint64_t bd =
                        smem_desc(sB + q * C::BLOCK_BYTES + s * C::B_KSTEP, C::B_LBO, C::B_SBO, C::B_LAYOUT);
                    tc_mma<KIND>(tmem + (uint32_t)(J * B), ad, bd, idesc, 1u);
                }
                q += L;
            }
            tc_commit(empty + stage);  // frees the stage once these MMAs complete
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
        tc_commit(accfull);
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        mbar_wait(accfull, 0);
        tc_fence_after();
        const int ew = warp - 4;
        const int64_t n = n0 + ew * 32 + lane;
        const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
        for (int c = 0; c < nbJ * B; c += 16) {
            uint32_t v[16];
            TMEM_LD16(tmem + lane_base + c, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                float *dst = p.dW + ((int64_t)J0 * B + c + i) * p.N + n;
                const float x = __uint_as_float(v[i]);
                if (p.mode == 2) {
                    atomicAdd(dst, x);
                } else if (p.mode == 1) {
                    *dst += x;
                } else {
                    *dst = x;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
    }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

static CUtensorMapSwizzle swz(int bytes) {
    if (bytes == -128) return CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    return bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
}

static cudaError_t make_map(CUtensorMap *tm, const void *base, CUtensorMapDataType dt, int es, uint64_t cols,
                            uint64_t rows, uint32_t box_cols, uint32_t box_rows, int swizzle_bytes) {
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * (cuuint64_t)es};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(tm, dt, 2, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

struct Plan {
    int kr_blocks, nkr, stages, stage_bytes, nsplit, smem;
    uint32_t tmem_cols;
};

template <int KIND, int B>
static Plan plan_for(int64_t M, int64_t K, int64_t N) {
    using C = Cfg<KIND, B>;
    Plan pl{};
    const int nbc = (int)(K / B);
    const int fixed = 1024 + 256;  // alignment slack + barriers + TMEM slot
    // largest kcol range (<= 512 TMEM columns) that still leaves >= 3 stages
    int maxb = std::min(512 / B, nbc);
    while (maxb > 1 && 3 * (C::A_BYTES + maxb * C::BLOCK_BYTES + kMetaBytes) + fixed > kSmemBudget) --maxb;
    pl.nkr = (nbc + maxb - 1) / maxb;
    pl.kr_blocks = (nbc + pl.nkr - 1) / pl.nkr;
    pl.stage_bytes = (C::A_BYTES + pl.kr_blocks * C::BLOCK_BYTES + 1023) & ~1023;
    pl.stages = std::min(8, (kSmemBudget - fixed) / (pl.stage_bytes + kMetaBytes));
    pl.smem = pl.stages * (pl.stage_bytes + kMetaBytes) + fixed;
    uint32_t cols = 32;
    while (cols < (uint32_t)(pl.kr_blocks * B)) cols <<= 1;
    pl.tmem_cols = cols;
    const int64_t tiles = (N / 128) * pl.nkr;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nbr = M / B;
    pl.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(nbr, sms / std::max<int64_t>(1, tiles)));
    return pl;
}

template <int KIND, int B>
static cudaError_t launch_t(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnzb,
                            int64_t M, int64_t K, const void *dY, int64_t N, float *dW, int accumulate,
                            cudaStream_t stream) {
    using C = Cfg<KIND, B>;
    const Plan pl = plan_for<KIND, B>(M, K, N);
    const CUtensorMapDataType dt = KIND == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUtensorMap tm_dy, tm_val;
    cudaError_t e = make_map(&tm_dy, dY, dt, C::ES, (uint64_t)N, (uint64_t)M, C::AW, B, C::TF32 ? -128 : 128);
    if (e != cudaSuccess) return e;
    e = make_map(&tm_val, values, dt, C::ES, (uint64_t)B, (uint64_t)nnzb * B, C::BW / C::ES, B,
                 C::TF32 ? -128 : C::BW);
    if (e != cudaSuccess) return e;
    Params p{};
    p.rowptr = rowptr;
    p.colidx = colidx;
    p.dW = dW;
    p.nbr = M / B;
    p.N = N;
    p.K = K;
    p.nkr = pl.nkr;
    p.nsplit = pl.nsplit;
    p.kr_blocks = pl.kr_blocks;
    p.stages = pl.stages;
    p.stage_bytes = pl.stage_bytes;
    p.tmem_cols = pl.tmem_cols;
    if (pl.nsplit > 1) {
        p.mode = 2;
        if (!accumulate) {
            e = cudaMemsetAsync(dW, 0, (size_t)K * N * sizeof(float), stream);
            if (e != cudaSuccess) return e;
        }
    } else {
        p.mode = accumulate ? 1 : 0;
    }
    auto kern = wgrad_tc_kernel<KIND, B>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((N / 128) * pl.nkr * pl.nsplit);
    kern<<<grid, kThreads, pl.smem, stream>>>(tm_dy, tm_val, p);
    count_launch();
    return cudaGetLastError();
}

}  // namespace tc

size_t wgrad_tc_ws_bytes(int64_t, int64_t, int, int64_t) { return 0; }

cudaError_t launch_wgrad_tc(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnzb,
                            int kind, int64_t M, int64_t K, int b, const void *dY, int64_t N, float *dW,
                            int accumulate, void *, cudaStream_t stream) {
    if (!values || nnzb == 0) {  // no stored block: dW = 0 (or unchanged)
        return accumulate ? cudaSuccess : cudaMemsetAsync(dW, 0, (size_t)K * N * sizeof(float), stream);
    }
#define TC_CASE(KD, B_) \
    if (kind == KD && b == B_) return tc::launch_t<KD, B_>(rowptr, colidx, values, nnzb, M, K, dY, N, dW, accumulate, stream);
    TC_CASE(0, 32) TC_CASE(0, 64) TC_CASE(1, 16) TC_CASE(1, 32) TC_CASE(1, 64)
#undef TC_CASE
    return cudaErrorInvalidValue;
}

}  // namespace bsrp
