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
// (range of block rows: split-K).  Warp roles: warp 0 = TMA producer, warp 1 =
// MMA issuer, warp 2 = TMEM allocator, warp 3 = block-row metadata prefetcher
// (rowptr/colidx chunks into shared memory, double-buffered), warps 4-7 =
// epilogue (tcgen05.ld -> fp32 stores of this split's partial tile).
// Shared memory holds an A ring (one b x 128 dY slab per block row, loaded with
// ONE 3-D TMA) and a B ring of block slots (a row's kept blocks are consecutive
// in BSR storage and land in consecutive slots, loaded G blocks per 4-D TMA),
// swizzled by TMA exactly as the UMMA descriptors expect.  The producer turns
// each row into a list of MMA runs (consecutive block columns, N <= 256) so the
// per-row instruction count of both single-thread roles stays small -- the
// per-row issue cost, not HBM, bounds a naive version of this kernel.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "launch.h"

namespace bsrp {
namespace tc {

constexpr int kThreads = 256;
// per stage (uint4 units), written by the B producer: [0].x = number of MMA runs
// (kEndMarker = no more rows); [1..] = one MMA run each, ready to issue:
// x = TMEM address of its first column, y = low word of the B descriptor (k-step
// 0), z = UMMA instruction descriptor (encodes N = run length * b)
constexpr int kMetaQuads = 34;
constexpr uint32_t kEndMarker = 0xFFFFu;
constexpr int kStageExtra = kMetaQuads * 16 + 4 + 16;  // meta + slot-use word + full/empty mbarriers
constexpr int kSmemBudget = 227 * 1024;
constexpr int kColCap = 1024;      // kept blocks of one metadata chunk (colidx staged in smem; one run each at most)
constexpr int kRowCap = 255;       // block rows of one metadata chunk
// alignment slack + barriers/TMEM slot + rowptr/colidx scratch + two row-plan buffers
// (16-byte row records + 8-byte run records)
constexpr int kFixedSmem = 1024 + 1024 + 4 * (kRowCap + 1) + 2 * kColCap + 2 * (16 * kRowCap + 8 * kColCap);
constexpr int kSplitSMs = 148;     // bound on split-K CTAs used to size the workspace (B200: 148 SMs)

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

__device__ __forceinline__ void tma_load_3d(const CUtensorMap *tm, uint64_t *bar, uint32_t dst, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(const CUtensorMap *tm, uint64_t *bar, uint32_t dst, int x, int y, int z,
                                            int w) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
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

// All B/UK k-steps of one MMA run in a single asm block: descriptors advance by
// constant byte offsets (>> 4) inside PTX, so the issuing thread moves the base
// descriptors into uniform registers once per run instead of once per MMA.
#define BSRP_MMA2(KS)                                                                                    \
    asm volatile("{\n.reg .b64 a1, b1;\n"                                                                 \
                 "add.s64 a1, %1, %4;\nadd.s64 b1, %2, %5;\n"                                             \
                 "tcgen05.mma.cta_group::1.kind::" KS " [%0], %1, %2, %3, 1;\n"                          \
                 "tcgen05.mma.cta_group::1.kind::" KS " [%0], a1, b1, %3, 1;\n}\n" ::"r"(d_tmem),         \
                 "l"(a_desc), "l"(b_desc), "r"(idesc), "n"(AK), "n"(BK))
#define BSRP_MMA4(KS)                                                                                    \
    asm volatile("{\n.reg .b64 a1, b1, a2, b2, a3, b3;\n"                                                 \
                 "add.s64 a1, %1, %4;\nadd.s64 b1, %2, %5;\n"                                             \
                 "add.s64 a2, %1, %6;\nadd.s64 b2, %2, %7;\n"                                             \
                 "add.s64 a3, %1, %8;\nadd.s64 b3, %2, %9;\n"                                             \
                 "tcgen05.mma.cta_group::1.kind::" KS " [%0], %1, %2, %3, 1;\n"                          \
                 "tcgen05.mma.cta_group::1.kind::" KS " [%0], a1, b1, %3, 1;\n"                          \
                 "tcgen05.mma.cta_group::1.kind::" KS " [%0], a2, b2, %3, 1;\n"                          \
                 "tcgen05.mma.cta_group::1.kind::" KS " [%0], a3, b3, %3, 1;\n}\n" ::"r"(d_tmem),         \
                 "l"(a_desc), "l"(b_desc), "r"(idesc), "n"(AK), "n"(BK), "n"(2 * AK), "n"(2 * BK),         \
                 "n"(3 * AK), "n"(3 * BK))
template <int KIND, int NSTEP, int AK, int BK>
__device__ __forceinline__ void tc_mma_run(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc) {
    if constexpr (NSTEP == 1) {
        tc_mma<KIND>(d_tmem, a_desc, b_desc, idesc, 1u);
    } else if constexpr (NSTEP == 2) {
        if constexpr (KIND == 1) BSRP_MMA2("f16"); else BSRP_MMA2("tf32");
    } else if constexpr (NSTEP == 4) {
        if constexpr (KIND == 1) BSRP_MMA4("f16"); else BSRP_MMA4("tf32");
    } else {
        static_assert(NSTEP % 4 == 0, "k steps per block");
#pragma unroll
        for (int s = 0; s < NSTEP; s += 4)
            tc_mma_run<KIND, 4, AK, BK>(d_tmem, a_desc + (uint64_t)(s * AK), b_desc + (uint64_t)(s * BK), idesc);
    }
}
#undef BSRP_MMA2
#undef BSRP_MMA4

// tcgen05.mma issued by one elected lane of a converged warp; the 64-bit
// descriptors are assembled from 32-bit halves inside PTX.  Every operand is
// warp-uniform, so ptxas keeps them in uniform registers.
template <int KIND>
__device__ __forceinline__ void tc_mma_elect(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo,
                                             uint32_t b_hi, uint32_t idesc) {
    if constexpr (KIND == 1) {
        asm volatile(
            "{\n.reg .pred p;\n.reg .b64 a, b;\nmov.b64 a, {%1, %2};\nmov.b64 b, {%3, %4};\n"
            "elect.sync _|p, 0xffffffff;\n"
            "@p tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %5, 1;\n}\n" ::"r"(d_tmem),
            "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc));
    } else {
        asm volatile(
            "{\n.reg .pred p;\n.reg .b64 a, b;\nmov.b64 a, {%1, %2};\nmov.b64 b, {%3, %4};\n"
            "elect.sync _|p, 0xffffffff;\n"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], a, b, %5, 1;\n}\n" ::"r"(d_tmem),
            "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc));
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
    float *dW, *ws;
    int64_t nbr, N, K;
    int nkr, nsplit, kr_blocks;  // kcol range = kr_blocks blocks
    int stages, nbslots, mode;   // A-ring stages, B-ring block slots; mode: 0 store, 1 load-add-store, 3 partial -> ws[split]
    int chunk_rows;              // block rows of one metadata chunk (rowptr + colidx staged in smem)
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
    static constexpr int G = BLOCK_BYTES >= 8192 ? 1 : BLOCK_BYTES >= 2048 ? 4 : 8;  // blocks per B TMA
};

#ifdef WGRAD_TRACE
__device__ unsigned long long g_trace[160][256];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TRACE(slot) (g_trace[blockIdx.x][(slot)] = gtime())
#else
#define TRACE(slot) ((void)0)
#endif
#ifndef WGRAD_TRACE_MODE
#define WGRAD_TRACE_MODE 0  // dev experiments only: 1 = no loads, 2 = no MMAs
#endif

// Slow wait for warps that idle for the whole main loop (epilogue): back off so
// they do not steal issue slots from the producer and MMA warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) __nanosleep(256);
}

template <int KIND, int B>
__global__ void __launch_bounds__(kThreads, 1)
    wgrad_tc_kernel(const __grid_constant__ CUtensorMap tm_dy, const __grid_constant__ CUtensorMap tm_val,
                    const __grid_constant__ CUtensorMap tm_dw, const __grid_constant__ CUtensorMap tm_ws, Params p) {
    using C = Cfg<KIND, B>;
    // shared memory: [A ring: stages x A_BYTES][B ring: nbslots x BLOCK_BYTES][meta: stages x kMetaPairs]
    //   [slot use: stages][mbarriers][TMEM slot][rowptr scratch][colidx scratch][2 x row records][2 x run records]
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *ringA = smem;
    uint8_t *ringB = ringA + (size_t)p.stages * C::A_BYTES;
    uint4 *meta = reinterpret_cast<uint4 *>(ringB + (size_t)p.nbslots * C::BLOCK_BYTES);
    uint32_t *s_used = reinterpret_cast<uint32_t *>(meta + p.stages * kMetaQuads);
    uint64_t *full = reinterpret_cast<uint64_t *>(s_used + ((p.stages + 1) & ~1));
    uint64_t *empty = full + p.stages;
    uint64_t *accfull = empty + p.stages;
    uint64_t *plan_full = accfull + 1;     // [2]
    uint64_t *plan_empty = plan_full + 2;  // [2]
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(plan_empty + 2);
    int4 *s_rows = reinterpret_cast<int4 *>((reinterpret_cast<uintptr_t>(s_tmem + 4) + 15) & ~uintptr_t(15));
    // s_rows [2][kRowCap]: cnt | nruns << 16, B-ring need, run offset, first value index
    uint2 *s_runs = reinterpret_cast<uint2 *>(s_rows + 2 * kRowCap);      // [2][kColCap]
    int32_t *s_rp = reinterpret_cast<int32_t *>(s_runs + 2 * kColCap);   // [kRowCap + 1]
    uint16_t *s_col = reinterpret_cast<uint16_t *>(s_rp + kRowCap + 1);  // [kColCap]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Consecutive CTAs take consecutive 128-column tiles of the same block rows,
    // so CTAs that run together read adjacent 512-byte pieces of the same dY rows.
    const int ntn = (int)(p.N / 128);
    int t = blockIdx.x;
    const int nt = t % ntn;
    t /= ntn;
    const int kr = t % p.nkr;
    const int split = t / p.nkr;
    const int n0 = nt * 128;
    const int nbc = (int)(p.K / B);
    const int J0 = kr * p.kr_blocks;
    const int nbJ = min(p.kr_blocks, nbc - J0);
    const int64_t Ib = (int64_t)split * p.nbr / p.nsplit, Ie = (int64_t)(split + 1) * p.nbr / p.nsplit;
    // chunk 0 is short (32 rows) so the first plan is ready early; later chunks are chunk_rows long
    const int first_rows = min(32, p.chunk_rows);
    const int64_t nrows_cta = Ie - Ib;
    const int nchunks = nrows_cta <= first_rows ? (nrows_cta > 0 ? 1 : 0)
                                                : 1 + (int)((nrows_cta - first_rows + p.chunk_rows - 1) / p.chunk_rows);
    auto chunk_start = [&](int c) -> int64_t { return c == 0 ? Ib : Ib + first_rows + (int64_t)(c - 1) * p.chunk_rows; };
    auto chunk_len = [&](int c) -> int {
        return (int)min((int64_t)(c == 0 ? first_rows : p.chunk_rows), Ie - chunk_start(c));
    };
    if (threadIdx.x == 0) TRACE(0);

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dy)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_val)) : "memory");
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(full + s, 2);   // A producer + B producer
            mbar_init(empty + s, 1);  // the MMA warp's commit
        }
        mbar_init(accfull, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(plan_full + i, 1);
            mbar_init(plan_empty + i, 2);  // both producers release a plan chunk
        }
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

    if (warp == 3) {
        // ------------------------------------------------ row planner
        // For each chunk of block rows: rowptr + colidx into shared memory, then
        // one lane per row derives the row's kept-block count, B-ring need (G
        // rounded), first value index and its MMA runs (consecutive block columns,
        // <= MAX_RUN blocks, each a TMEM column + slot offset + instruction
        // descriptor), written to a double-buffered plan one chunk ahead of the
        // producer.  The single-thread producer and MMA roles then do almost no
        // per-row arithmetic.
        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            const int64_t Ic = chunk_start(c);
            const int nrow = chunk_len(c);
            for (int i = lane; i <= nrow; i += 32) s_rp[i] = __ldg(p.rowptr + Ic + i);
            __syncwarp();
            const int base = s_rp[0], total = s_rp[nrow] - base;
            for (int e = lane; e < total; e += 32) s_col[e] = (uint16_t)__ldg(p.colidx + base + e);
            if (lane == 0) mbar_wait(plan_empty + buf, ((c >> 1) & 1) ^ 1);
            __syncwarp();
            int4 *rows = s_rows + buf * kRowCap;
            uint2 *runs = s_runs + buf * kColCap;
            int run_base = 0;
            for (int r0 = 0; r0 < nrow; r0 += 32) {
                const int r = r0 + lane;
                int q0 = 0, cnt = 0, nruns = 0;
                if (r < nrow) {
                    q0 = s_rp[r] - base;
                    int q1 = s_rp[r + 1] - base;
                    if (p.nkr > 1) {
                        while (q0 < q1 && (int)s_col[q0] < J0) ++q0;
                        int q = q0;
                        while (q < q1 && (int)s_col[q] < J0 + nbJ) ++q;
                        q1 = q;
                    }
                    cnt = q1 - q0;
                    int jprev = -2, rlen = 0;
                    for (int q = 0; q < cnt; ++q) {
                        const int J = (int)s_col[q0 + q] - J0;
                        if (J == jprev + 1 && rlen < C::MAX_RUN && true) {
                            ++rlen;
                        } else {
                            ++nruns;
                            rlen = 1;
                        }
                        jprev = J;
                    }
                }
                // exclusive warp scan of nruns -> this row's run offset
                int incl = nruns;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int off = run_base + incl - nruns;
                run_base += __shfl_sync(0xffffffffu, incl, 31);
                if (r < nrow) {
                    int jprev = -2, rlen = 0, rstart = 0, k = off;
                    for (int q = 0; q < cnt; ++q) {
                        const int J = (int)s_col[q0 + q] - J0;
                        if (J == jprev + 1 && rlen < C::MAX_RUN && true) {
                            ++rlen;
                        } else {
                            if (rlen)
                                runs[k++] = make_uint2((uint32_t)((jprev - rlen + 1) * B) | ((uint32_t)rstart << 16),
                                                       instr_desc<KIND>((uint32_t)(rlen * B)));
                            rstart = q;
                            rlen = 1;
                        }
                        jprev = J;
                    }
                    if (rlen)
                        runs[k++] = make_uint2((uint32_t)((jprev - rlen + 1) * B) | ((uint32_t)rstart << 16),
                                               instr_desc<KIND>((uint32_t)(rlen * B)));
                    rows[r] = make_int4(cnt | (nruns << 16), (cnt + C::G - 1) / C::G * C::G, off, base + q0);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(plan_full + buf);
        }
    } else if (warp >= 4) {
        // zero the accumulator columns this CTA owns (MMAs then always accumulate)
        const uint32_t lane_base = (uint32_t)((warp - 4) * 32) << 16;
        for (int c = 0; c < nbJ * B; c += 16) tmem_st16_zero(tmem + lane_base + c);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (warp == 1 || warp == 2 || warp >= 4) {  // the MMA warps start only after the accumulator is zeroed
        tc_fence_before();
        asm volatile("bar.sync 1, 192;" ::: "memory");
        tc_fence_after();
    }

    if ((warp == 0 || warp == 4) && lane == 0) {
        // ------------------------------------------------ TMA producers (one thread each)
        // Both walk the same sequence of kept block rows (row j uses stage j % stages).
        // Warp 0 loads row j's b x 128 dY slab (one 3-D TMA) into the A ring; warp 4
        // (an epilogue warp, idle until the accumulator is final) places the row's
        // kept blocks in consecutive B-ring slots (never wrapping: a row that would
        // wrap starts at slot 0 and the tail slots are skipped), loads them G blocks
        // per 4-D TMA and writes the stage's ready-to-issue MMA runs.  `full` needs
        // both arrivals plus all bytes; stages and slots are reclaimed in order as
        // the MMA commits arrive on `empty`.
        const bool is_a = warp == 0;
        int j = 0;  // kept rows issued so far
        int tail = 0, bhead = 0, bfree = p.nbslots;
        const uint32_t sA0 = smem_u32(ringA), sB0 = smem_u32(ringB);
        const uint32_t b_lo0 = (uint32_t)smem_desc(sB0, C::B_LBO, C::B_SBO, C::B_LAYOUT);
        long long cyc_wait = 0, cyc_issue = 0, cyc_start = clock64();
        (void)cyc_wait; (void)cyc_issue; (void)cyc_start;
        // The first n_spec rows are in the sequence whether or not they keep a block:
        // their dY slabs are requested before the planner has read rowptr/colidx, so
        // the first HBM round trip overlaps the plan (an empty row costs one slab).
        const int n_spec = (int)min((int64_t)min(p.stages, first_rows), Ie - Ib);
        if (is_a)
            for (int r = 0; r < n_spec; ++r) {
                mbar_arrive_expect_tx(full + r, (uint32_t)C::A_BYTES);
                tma_load_3d(&tm_dy, full + r, sA0 + r * C::A_BYTES, 0, (int)(Ib + r) * B, n0 / C::AW);
            }
        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            const int64_t Ic = chunk_start(c);
            const int nrow = chunk_len(c);
            mbar_wait(plan_full + buf, (c >> 1) & 1);
            const int4 *rows = s_rows + buf * kRowCap;
            const uint2 *runs = s_runs + buf * kColCap;
            for (int r = 0; r < nrow; ++r) {
                const int4 rr = rows[r];
                const int cnt = rr.x & 0xFFFF;
                const bool spec = c == 0 && r < n_spec;
                if (cnt == 0 && !spec) continue;
                const int stage = j % p.stages;
                if (spec && is_a) {  // slab already requested above
                    ++j;
                    continue;
                }
#ifdef WGRAD_TRACE
                const long long tw0 = clock64();
#endif
                if (is_a) {
                    if (j >= p.stages) mbar_wait(empty + stage, (uint32_t)((j / p.stages) - 1) & 1u);
                } else {
                    const int need = rr.y;
                    const int waste = bhead + need > p.nbslots ? p.nbslots - bhead : 0;
                    while (j - tail >= p.stages || bfree < need + waste) {  // reclaim the oldest row
                        mbar_wait(empty + tail % p.stages, (uint32_t)(tail / p.stages) & 1u);
                        bfree += (int)s_used[tail % p.stages];
                        ++tail;
                    }
                    const int slot0 = waste ? 0 : bhead;
                    s_used[stage] = (uint32_t)(need + waste);
                    bhead = slot0 + need;
                    if (bhead == p.nbslots) bhead = 0;
                    bfree -= need + waste;
                    // ready-to-issue runs: TMEM address, B descriptor low word, instruction descriptor
                    const int nruns = rr.x >> 16;
                    uint4 *m = meta + stage * kMetaQuads;
                    for (int i = 0; i < nruns; ++i) {  // compact run word: column | B-ring slot << 10 | length << 22
                        const uint2 run = runs[rr.z + i];
                        const uint32_t len = ((run.y >> 17) & 0x3Fu) * 8u / (uint32_t)B;
                        m[1 + i].x = (run.x & 0x3FFu) | ((uint32_t)(slot0 + (int)(run.x >> 16)) << 10) | (len << 22);
                    }
                    m[0].x = (uint32_t)nruns;
#ifdef WGRAD_TRACE
                    const long long tw1 = clock64();
                    cyc_wait += tw1 - tw0;
#endif
                    mbar_arrive_expect_tx(full + stage, (uint32_t)(need * C::BLOCK_BYTES));
                    for (int g = 0; g < need; g += C::G)
                        tma_load_4d(&tm_val, full + stage, sB0 + (slot0 + g) * C::BLOCK_BYTES, 0, 0, 0, rr.w + g);
#ifdef WGRAD_TRACE
                    cyc_issue += clock64() - tw1;
#endif
                }
                if (is_a) {
#ifdef WGRAD_TRACE
                    const long long tw1 = clock64();
                    cyc_wait += tw1 - tw0;
#endif
                    mbar_arrive_expect_tx(full + stage, (uint32_t)C::A_BYTES);
                    tma_load_3d(&tm_dy, full + stage, sA0 + stage * C::A_BYTES, 0, (int)(Ic + r) * B, n0 / C::AW);
#ifdef WGRAD_TRACE
                    cyc_issue += clock64() - tw1;
#endif
                }
                ++j;
            }
            mbar_arrive(plan_empty + buf);
        }
#ifdef WGRAD_TRACE
        g_trace[blockIdx.x][210 + 4 * (warp == 4)] = (unsigned long long)cyc_wait;
        g_trace[blockIdx.x][211 + 4 * (warp == 4)] = (unsigned long long)cyc_issue;
        g_trace[blockIdx.x][212 + 4 * (warp == 4)] = (unsigned long long)(clock64() - cyc_start);
        g_trace[blockIdx.x][213 + 4 * (warp == 4)] = (unsigned long long)j;
#endif
        // end marker in stage j % stages: free it, then both producers arrive (no bytes)
        const int stage = j % p.stages;
        if (j >= p.stages) mbar_wait(empty + stage, (uint32_t)((j / p.stages) - 1) & 1u);
        if (!is_a) meta[stage * kMetaQuads] = make_uint4(kEndMarker, 0u, 0u, 0u);
        mbar_arrive(full + stage);
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (whole warp, one elected lane issues)
        // Lane i loads word i of the stage's metadata (header + runs) with ONE shared
        // load; each run word becomes warp-uniform with a single masked redux, and
        // the descriptors are built from it with uniform arithmetic, so every
        // tcgen05.mma is one predicated UTCHMMA.
        const uint64_t a_desc0 = smem_desc(smem_u32(ringA), C::A_LBO, C::A_SBO, C::A_LAYOUT);
        const uint32_t a_lo0 = (uint32_t)a_desc0, a_hi = (uint32_t)(a_desc0 >> 32);
        const uint64_t b_desc0 = smem_desc(smem_u32(ringB), C::B_LBO, C::B_SBO, C::B_LAYOUT);
        const uint32_t b_lo0 = (uint32_t)b_desc0, b_hi = (uint32_t)(b_desc0 >> 32);
        const uint32_t idesc0 = instr_desc<KIND>(0u);
        int stage = 0;
        uint32_t phase = 0;
        long long mw = 0, mi = 0, m_start = clock64(), nrow_m = 0;
        (void)mw; (void)mi; (void)m_start; (void)nrow_m;
        for (;;) {
#ifdef WGRAD_TRACE
            const long long t0m = clock64();
#endif
            mbar_wait(full + stage, phase);
            tc_fence_after();
#ifdef WGRAD_TRACE
            const long long t1m = clock64();
            mw += t1m - t0m;
            ++nrow_m;
#endif
            const uint32_t m_addr = smem_u32(meta + stage * kMetaQuads);
            uint32_t wl;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wl) : "r"(m_addr + lane * 16u));
            const uint32_t nruns = __reduce_or_sync(0xffffffffu, lane == 0 ? wl : 0u);
            if (nruns == kEndMarker) break;
            const uint32_t a_lo = a_lo0 + (uint32_t)((stage * C::A_BYTES) >> 4);
            for (uint32_t i = 0; i < nruns; ++i) {
                uint32_t w = wl;
                if (i + 1 >= 32) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(m_addr + (i + 1) * 16u));
                const uint32_t rw = __reduce_or_sync(0xffffffffu, (i + 1 >= 32 || lane == i + 1) ? w : 0u);
                const uint32_t d = tmem + (rw & 0x3FFu);
                const uint32_t b_lo = b_lo0 + ((rw >> 10) & 0xFFFu) * (uint32_t)(C::BLOCK_BYTES >> 4);
                const uint32_t idesc = idesc0 | ((((rw >> 22) & 0x3Fu) * (uint32_t)B >> 3) << 17);
#pragma unroll
                for (int s = 0; s < B / C::UK; ++s)
                    tc_mma_elect<KIND>(d, a_lo + ((s * C::A_KSTEP) >> 4), a_hi, b_lo + ((s * C::B_KSTEP) >> 4), b_hi,
                                       idesc);
            }
            __syncwarp();
            if (lane == 0) tc_commit(empty + stage);  // frees the stage (and its B slots) once these MMAs complete
            __syncwarp();
#ifdef WGRAD_TRACE
            mi += clock64() - t1m;
#endif
            if (++stage == p.stages) { stage = 0; phase ^= 1; }
        }
#ifdef WGRAD_TRACE
        if (lane == 0) {
            g_trace[blockIdx.x][218] = (unsigned long long)mw;
            g_trace[blockIdx.x][219] = (unsigned long long)mi;
            g_trace[blockIdx.x][220] = (unsigned long long)(clock64() - m_start);
        }
#endif
        if (lane == 0) tc_commit(accfull);
    }
    if (warp >= 4) {
        __syncwarp();  // warp 4's lane 0 rejoins after its B-producer loop
        // ------------------------------------------------ epilogue
        // TMEM -> registers -> a [32 kcol][128 n] fp32 staging tile in the (now
        // idle) A ring -> one TMA bulk tensor store (or reduce-add) per 16 kcols.
        // Full 512-byte row segments leave the SM through the TMA unit instead of
        // 128-byte scattered STGs.  mode 3 stores this split's partial tile into
        // its own workspace slice (summed afterwards in split order:
        // deterministic); mode 1 adds into dW (accumulate, one split).
        mbar_wait_sleep(accfull, 0);
        tc_fence_after();
        if (threadIdx.x == 128) TRACE(203);
        const int ew = warp - 4;
        const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
        float *stage_buf = reinterpret_cast<float *>(ringA);  // 2 x [32][128]
        const int ncols = nbJ * B;
        const int row0 = (p.mode == 3 ? split * (int)p.K : 0) + J0 * B;
        const CUtensorMap *tm_o = p.mode == 3 ? &tm_ws : &tm_dw;
        for (int c = 0, it = 0; c < ncols; c += 32, ++it) {
            float *sb = stage_buf + (it & 1) * (32 * 128);
            if (it >= 2) {  // the TMA store issued two chunks ago must have finished reading this buffer
                if (threadIdx.x == 128) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                asm volatile("bar.sync 2, 128;" ::: "memory");
            }
            uint32_t v[32];
            TMEM_LD16(tmem + lane_base + c, v);
            TMEM_LD16(tmem + lane_base + c + 16, (v + 16));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 32; ++i) sb[i * 128 + ew * 32 + lane] = __uint_as_float(v[i]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync 2, 128;" ::: "memory");
            if (threadIdx.x == 128) {
                const int nh = min(32, ncols - c) / 16;
                for (int h = 0; h < nh; ++h) {
                    const uint32_t src = smem_u32(sb + h * 16 * 128);
                    if (p.mode == 1)
                        asm volatile(
                            "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                reinterpret_cast<uint64_t>(tm_o)),
                            "r"(n0), "r"(row0 + c + h * 16), "r"(src)
                            : "memory");
                    else
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                                         reinterpret_cast<uint64_t>(tm_o)),
                                     "r"(n0), "r"(row0 + c + h * 16), "r"(src)
                                     : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
        if (threadIdx.x == 128) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    if (threadIdx.x == 128) TRACE(204);
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
    }
}

// dW (+)= sum over splits of the partial tiles, in split order (deterministic).
// Each thread owns float4 column blocks; up to 16 split loads are issued ahead
// of the (ordered) adds so the L2-resident partials stream at full rate.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float4 *__restrict__ ws, float4 *__restrict__ dW,
                                                            int64_t n4, int nsplit, int accumulate) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 a = accumulate ? dW[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s = 0; s < nsplit; s += 16) {  // up to 16 independent loads in flight, then ordered adds
            float4 v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (s + u < nsplit) v[u] = __ldcs(ws + (size_t)(s + u) * n4 + i);
#pragma unroll
            for (int u = 0; u < 16; ++u)
                if (s + u < nsplit) {
                    a.x += v[u].x; a.y += v[u].y; a.z += v[u].z; a.w += v[u].w;
                }
        }
        dW[i] = a;
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
    if (bytes == 0) return CU_TENSOR_MAP_SWIZZLE_NONE;
    if (bytes == -128) return CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    return bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
}

// Tensor map with explicit dims / byte strides / box (dims[0] contiguous).
static cudaError_t make_map(CUtensorMap *tm, const void *base, CUtensorMapDataType dt, int rank, const cuuint64_t *dims,
                            const cuuint64_t *strides, const cuuint32_t *box, int swizzle_bytes) {
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = fn(tm, dt, rank, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

struct Plan {
    int kr_blocks, nkr, stages, nbslots, nsplit, smem, chunk_rows;
    uint32_t tmem_cols;
};

// sms: SMs the split-K grid may fill (the device's count at launch, kSplitSMs
// for the pure workspace query).  avg_cnt: expected kept blocks per block row
// inside one TMEM column range (sizes the A ring against the B ring).
template <int KIND, int B>
static Plan plan_for(int64_t M, int64_t K, int64_t N, int sms, double avg_cnt = -1.0) {
    using C = Cfg<KIND, B>;
    Plan pl{};
    const int nbc = (int)(K / B);
    const int ring = kSmemBudget - kFixedSmem;
    // largest kcol range (<= 512 TMEM columns) whose full row (A slab + every
    // block) fits twice in the rings
    int maxb = std::min(512 / B, nbc);
    auto need_of = [](int blocks) { return (blocks + C::G - 1) / C::G * C::G; };
    while (maxb > 1 && 2 * (C::A_BYTES + kStageExtra) + 2 * need_of(maxb) * C::BLOCK_BYTES > ring) --maxb;
    pl.nkr = (nbc + maxb - 1) / maxb;
    pl.kr_blocks = (nbc + pl.nkr - 1) / pl.nkr;
    if (avg_cnt < 0) avg_cnt = pl.kr_blocks;
    avg_cnt = std::max(1.0, std::min<double>(avg_cnt, pl.kr_blocks));
    // rows in flight: stages x (A slab + avg_cnt blocks) fills the ring
    // rows in flight: stages x (A slab + the average row's block slots) fills the ring
    const double avg_need = std::ceil(avg_cnt / C::G) * C::G + 0.5 * (C::G - 1);
    int stages = (int)(ring / (C::A_BYTES + kStageExtra + avg_need * C::BLOCK_BYTES));
    stages = std::max(2, std::min(64, stages));
    int nb = (ring - stages * (C::A_BYTES + kStageExtra)) / C::BLOCK_BYTES;
    while (nb < 2 * need_of(pl.kr_blocks) && stages > 2) {  // a full row must fit even after a wrap
        --stages;
        nb = (ring - stages * (C::A_BYTES + kStageExtra)) / C::BLOCK_BYTES;
    }
    pl.stages = stages;
    pl.nbslots = nb;
    pl.smem = stages * (C::A_BYTES + kStageExtra) + pl.nbslots * C::BLOCK_BYTES + kFixedSmem;
    pl.chunk_rows = std::max(1, std::min(kRowCap, kColCap / nbc));  // a chunk's kept blocks fit the colidx/run buffers
    uint32_t cols = 32;
    while (cols < (uint32_t)(pl.kr_blocks * B)) cols <<= 1;
    pl.tmem_cols = cols;
    const int64_t tiles = (N / 128) * pl.nkr;
    const int64_t nbr = M / B;
    const int64_t cap = std::min<int64_t>(sms, kSplitSMs);
    pl.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(nbr, cap / std::max<int64_t>(1, tiles)));
    return pl;
}

template <int KIND, int B>
static cudaError_t launch_t(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnzb,
                            int64_t M, int64_t K, const void *dY, int64_t N, float *dW, int accumulate,
                            float *ws, cudaStream_t stream) {
    using C = Cfg<KIND, B>;
    int dev = 0, sms = kSplitSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // kept blocks per block row inside one TMEM column range, on average
    Plan pl = plan_for<KIND, B>(M, K, N, sms);
    const double avg_cnt = (double)nnzb / (double)(M / B) * pl.kr_blocks / (double)(K / B);
    pl = plan_for<KIND, B>(M, K, N, sms, avg_cnt);
    const CUtensorMapDataType dt = KIND == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUtensorMap tm_dy, tm_val;
    // dY as (column within a 128-byte atom, row, atom): one box = the b x 128 slab
    // of a block row, atom-major in shared memory (A_LBO apart)
    const cuuint64_t dy_dims[3] = {(cuuint64_t)C::AW, (cuuint64_t)M, (cuuint64_t)(N / C::AW)};
    const cuuint64_t dy_str[2] = {(cuuint64_t)N * C::ES, 128};
    const cuuint32_t dy_box[3] = {(cuuint32_t)C::AW, (cuuint32_t)B, (cuuint32_t)C::A_ATOMS};
    cudaError_t e = make_map(&tm_dy, dY, dt, 3, dy_dims, dy_str, dy_box, C::TF32 ? -128 : 128);
    if (e != cudaSuccess) return e;
    // values as (element within a swizzle atom row, block row, atom, block): one
    // box = G consecutive stored blocks, each atom-major (B_LBO apart)
    const cuuint64_t v_dims[4] = {(cuuint64_t)(C::BW / C::ES), (cuuint64_t)B, (cuuint64_t)C::B_ATOMS, (cuuint64_t)nnzb};
    const cuuint64_t v_str[3] = {(cuuint64_t)B * C::ES, (cuuint64_t)C::BW, (cuuint64_t)C::BLOCK_BYTES};
    const cuuint32_t v_box[4] = {(cuuint32_t)(C::BW / C::ES), (cuuint32_t)B, (cuuint32_t)C::B_ATOMS, (cuuint32_t)C::G};
    e = make_map(&tm_val, values, dt, 4, v_dims, v_str, v_box, C::TF32 ? -128 : C::BW);
    if (e != cudaSuccess) return e;
    // epilogue outputs: dW (K x N fp32) and the split-K workspace (nsplit*K x N), 128 x 16 boxes
    CUtensorMap tm_dw, tm_ws;
    const cuuint64_t o_dims[2] = {(cuuint64_t)N, (cuuint64_t)K};
    const cuuint64_t o_str[1] = {(cuuint64_t)N * 4};
    const cuuint32_t o_box[2] = {128, 16};
    e = make_map(&tm_dw, dW, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, o_dims, o_str, o_box, 0);
    if (e != cudaSuccess) return e;
    tm_ws = tm_dw;
    if (pl.nsplit > 1) {
        const cuuint64_t w_dims[2] = {(cuuint64_t)N, (cuuint64_t)K * pl.nsplit};
        e = make_map(&tm_ws, ws, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w_dims, o_str, o_box, 0);
        if (e != cudaSuccess) return e;
    }
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
    p.nbslots = pl.nbslots;
    p.tmem_cols = pl.tmem_cols;
    p.chunk_rows = pl.chunk_rows;
    p.ws = ws;
    p.mode = pl.nsplit > 1 ? 3 : accumulate ? 1 : 0;
#ifdef WGRAD_TMA_REDUCE
    if (pl.nsplit > 1) {  // experiment: TMA bulk reduce-add of every split into dW
        p.mode = 1;
        if (!accumulate) cudaMemsetAsync(dW, 0, (size_t)K * N * 4, stream);
    }
#endif
    auto kern = wgrad_tc_kernel<KIND, B>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((N / 128) * pl.nkr * pl.nsplit);
    kern<<<grid, kThreads, pl.smem, stream>>>(tm_dy, tm_val, tm_dw, tm_ws, p);
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess || pl.nsplit == 1 || p.mode == 1) return e;
    const int64_t n4 = K * N / 4;
    const unsigned rgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, (int64_t)sms * 8));
    splitk_reduce_kernel<<<rgrid, 256, 0, stream>>>(reinterpret_cast<const float4 *>(ws),
                                                    reinterpret_cast<float4 *>(dW), n4, pl.nsplit, accumulate);
    count_launch();
    return cudaGetLastError();
}

}  // namespace tc

size_t wgrad_tc_ws_bytes(int64_t M, int64_t K, int b, int64_t N) {
    tc::Plan pl{};
#define WS_CASE(B_) if (b == B_) pl = tc::plan_for<1, B_>(M, K, N, tc::kSplitSMs);
    WS_CASE(16) WS_CASE(32) WS_CASE(64)
#undef WS_CASE
    // the tf32 plan has fewer TMEM-column ranges than or as many as the bf16 one,
    // hence at least as many splits: take the larger of the two
    tc::Plan pt{};
    if (b == 32) pt = tc::plan_for<0, 32>(M, K, N, tc::kSplitSMs);
    if (b == 64) pt = tc::plan_for<0, 64>(M, K, N, tc::kSplitSMs);
    const int ns = std::max(pl.nsplit, pt.nsplit);
    return ns > 1 ? (size_t)ns * K * N * sizeof(float) : 0;
}

cudaError_t launch_wgrad_tc(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnzb,
                            int kind, int64_t M, int64_t K, int b, const void *dY, int64_t N, float *dW,
                            int accumulate, void *ws, cudaStream_t stream) {
    if (!values || nnzb == 0) {  // no stored block: dW = 0 (or unchanged)
        return accumulate ? cudaSuccess : cudaMemsetAsync(dW, 0, (size_t)K * N * sizeof(float), stream);
    }
#define TC_CASE(KD, B_) \
    if (kind == KD && b == B_) return tc::launch_t<KD, B_>(rowptr, colidx, values, nnzb, M, K, dY, N, dW, accumulate, \
                                                            static_cast<float *>(ws), stream);
    TC_CASE(0, 32) TC_CASE(0, 64) TC_CASE(1, 16) TC_CASE(1, 32) TC_CASE(1, 64)
#undef TC_CASE
    return cudaErrorInvalidValue;
}

}  // namespace bsrp
