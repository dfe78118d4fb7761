// wgrad_tc.cu -- BSR weight gradient on the 5th-generation tensor cores
// (row a6 of SURVEY §8a; BJ "TMA-fed tcgen05/TMEM block-sparse GEMM").
//
//   dW[J*b + c][n] = sum over stored blocks (I, J), sum over r < b of
//                    values(I,J)[r][c] * dY[I*b + r][n]
//
// Orientation: the MMA computes D = dW^T tile-wise,
//   D[n][kcol] (TMEM: 128 lanes = 128 columns n of dY, one TMEM column per
//   kcol of X) += A[n][r] * B[r][kcol]
// with A = the b x 128 slab of dY of block row I and B = the stored X blocks of
// that block row (MN-major: kcol contiguous, exactly the BSR block layout,
// staged in shared memory by TMA).  Every kept block becomes b/UMMA_K MMAs of
// shape 128 x b x UMMA_K into its own TMEM column range, so pruned blocks cost
// nothing; runs of adjacent kept blocks (consecutive in BSR storage, hence
// consecutive in shared memory) merge into one MMA with N = run * b <= 256.
// Block rows without a kept block in the CTA's column range are never read.
//
// A lives in TENSOR memory (the `.kind [d], [a_tmem], b_desc` form): the slab is
// shared by every run of its row, and an MMA that reads A from shared memory
// pays 4 KB of shared-memory bandwidth per instruction (measured floor 32 + N/4
// cycles per MMA, scratch/umma_mw.cu) -- more than the math itself for the
// short runs of a pruned row (N/2 cycles).  Each slab is loaded by ONE 2-D
// TMA into a shared-memory A ring (per-thread global loads top out near half
// the HBM bandwidth for this access pattern, scratch/ldg_stream.cu), then warps
// 4-7 move it shared -> registers -> tcgen05.st into one of NA TMEM A buffers;
// with A in TMEM the MMAs only read their B blocks from shared memory.
//
// CTA = (128-column tile of dY) x (range of kcols: TMEM columns) x (range of
// block rows: split-K).  Warp roles: warp 0 = B producer (TMA), warp 1 = MMA
// issuer for the lower half of the accumulator columns, warp 2 = TMEM allocator
// then MMA issuer for the upper half, warp 3 = block-row planner (rowptr/colidx
// chunks -> per-row MMA runs and B-ring slots, double-buffered), warps 4-7 = A
// movers for the even rows of the sequence during the main loop, then the
// epilogue (tcgen05.ld -> TMA bulk stores of this split's partial tile), warp 8 =
// A producer (dY slab TMAs), warps 9-12 = A movers for the odd rows.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "launch.h"

namespace bsrp {
namespace tc {

constexpr int kStages = 24;        // rows whose B blocks may be resident at once
constexpr int kMaxA = 4;           // TMEM A buffers (rows in flight between the A movers and the MMA warps)
constexpr int kMaxSA = 8;          // shared-memory A ring stages (dY slabs in flight from HBM)
constexpr int kMaxIssuers = 4;     // MMA-issuing warps, each owning a contiguous range of accumulator columns
// FP32 grade (3xTF32): tcgen05's fp32 accumulation truncates (measured: the
// rel-F error of bf16-exact products grows linearly with the chain length,
// 3.9e-5 at 200704 rows), so a split's chain of MMAs into one
// TMEM accumulator is capped; the split-K reduce then sums the partials with
// round-to-nearest.  4.1e-6 was measured for 2090-row tf32 chains at keep 1.
constexpr int kX3ChainRows = 1536;
constexpr int kSmemBudget = 227 * 1024;
constexpr int kColCap = 1536;      // stored blocks of one metadata chunk (colidx staged in smem; one run each at most)
constexpr int kStepCap = 64;       // steps of one metadata chunk
constexpr int kMaxR = 4;           // block rows per step (b = 16)
// alignment slack + barriers/TMEM slot + slot-use words + two plan buffers (16-byte
// step records, 8-byte block-row records, 4-byte run words) + rowptr/colidx scratch
constexpr int kFixedSmem = 1024 + 1024 + kStages * 4 + 2 * (16 * kStepCap + 8 * kStepCap * kMaxR + 4 * kColCap) +
                           4 * (kStepCap * kMaxR + 1) + 2 * kColCap;
constexpr int kSplitSMs = 148;     // bound on split-K CTAs used to size the workspace (B200: 148 SMs)
constexpr int kMaxSplits = 4096;   // bound on split-K slices (chain-capped FP32-grade plans)
constexpr int kEpiBytes = 2 * 32 * 128 * 4;  // epilogue staging (two 32 x 128 fp32 tiles, reuses the B ring)

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
// Slow wait for warps that idle for a long stretch: back off so they do not
// steal issue slots from the producer and MMA warps.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) __nanosleep(256);
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

// tcgen05.mma with A in TMEM, issued by one elected lane of a converged warp;
// the B descriptor is assembled from 32-bit halves inside PTX.  Every operand is
// warp-uniform, so ptxas keeps them in uniform registers.
template <int KIND>
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi,
                                          uint32_t idesc) {
    if constexpr (KIND == 1) {
        asm volatile(
            "{\n.reg .pred p;\n.reg .b64 b;\nmov.b64 b, {%2, %3};\n"
            "elect.sync _|p, 0xffffffff;\n"
            "@p tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], b, %4, 1;\n}\n" ::"r"(d_tmem),
            "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc));
    } else {
        asm volatile(
            "{\n.reg .pred p;\n.reg .b64 b;\nmov.b64 b, {%2, %3};\n"
            "elect.sync _|p, 0xffffffff;\n"
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], b, %4, 1;\n}\n" ::"r"(d_tmem),
            "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc));
    }
}

// All NSTEP k-steps of one MMA run (A in TMEM) in ONE asm block: one elect, the
// operands enter once, and the per-step A column / B address offsets are added
// inside PTX, so the issuing warp spends ~2 instructions per MMA.
#define BSRP_TS_HEAD "{\n.reg .pred p;\n.reg .b32 a<8>, bl<8>;\n.reg .b64 b<8>;\nelect.sync _|p, 0xffffffff;\n"
#define BSRP_TS_STEP(KS, S)                                                                             \
    "add.u32 a" #S ", %1, " #S "*%5;\nadd.u32 bl" #S ", %2, " #S "*%6;\nmov.b64 b" #S ", {bl" #S ", %3};\n" \
    "@p tcgen05.mma.cta_group::1.kind::" KS " [%0], [a" #S "], b" #S ", %4, 1;\n"
#define BSRP_TS_ARGS                                                                                      \
    ::"r"(d_tmem), "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "n"(AKC), "n"(BK16)
template <int KIND, int NSTEP, int AKC, int BK16>
__device__ __forceinline__ void tc_mma_ts_run(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi,
                                              uint32_t idesc) {
    if constexpr (NSTEP == 1) {
        if constexpr (KIND == 1) asm volatile(BSRP_TS_HEAD BSRP_TS_STEP("f16", 0) "}\n" BSRP_TS_ARGS);
        else asm volatile(BSRP_TS_HEAD BSRP_TS_STEP("tf32", 0) "}\n" BSRP_TS_ARGS);
    } else if constexpr (NSTEP == 2) {
        if constexpr (KIND == 1) asm volatile(BSRP_TS_HEAD BSRP_TS_STEP("f16", 0) BSRP_TS_STEP("f16", 1) "}\n" BSRP_TS_ARGS);
        else asm volatile(BSRP_TS_HEAD BSRP_TS_STEP("tf32", 0) BSRP_TS_STEP("tf32", 1) "}\n" BSRP_TS_ARGS);
    } else if constexpr (NSTEP == 4) {
        if constexpr (KIND == 1)
            asm volatile(BSRP_TS_HEAD BSRP_TS_STEP("f16", 0) BSRP_TS_STEP("f16", 1) BSRP_TS_STEP("f16", 2)
                             BSRP_TS_STEP("f16", 3) "}\n" BSRP_TS_ARGS);
        else
            asm volatile(BSRP_TS_HEAD BSRP_TS_STEP("tf32", 0) BSRP_TS_STEP("tf32", 1) BSRP_TS_STEP("tf32", 2)
                             BSRP_TS_STEP("tf32", 3) "}\n" BSRP_TS_ARGS);
    } else {
        static_assert(NSTEP == 8, "k steps per block");
        if constexpr (KIND == 1)
            asm volatile(BSRP_TS_HEAD BSRP_TS_STEP("f16", 0) BSRP_TS_STEP("f16", 1) BSRP_TS_STEP("f16", 2)
                             BSRP_TS_STEP("f16", 3) BSRP_TS_STEP("f16", 4) BSRP_TS_STEP("f16", 5)
                                 BSRP_TS_STEP("f16", 6) BSRP_TS_STEP("f16", 7) "}\n" BSRP_TS_ARGS);
        else
            asm volatile(BSRP_TS_HEAD BSRP_TS_STEP("tf32", 0) BSRP_TS_STEP("tf32", 1) BSRP_TS_STEP("tf32", 2)
                             BSRP_TS_STEP("tf32", 3) BSRP_TS_STEP("tf32", 4) BSRP_TS_STEP("tf32", 5)
                                 BSRP_TS_STEP("tf32", 6) BSRP_TS_STEP("tf32", 7) "}\n" BSRP_TS_ARGS);
    }
}
#undef BSRP_TS_HEAD
#undef BSRP_TS_STEP
#undef BSRP_TS_ARGS

// FP32 grade (KIND 2): per k step three MMAs with A in TMEM --
//   [d]  += A_hi . B_hi      [dc] += A_lo . B_hi      [dc] += A_hi . B_lo
// A_lo sits ACOLS TMEM columns after A_hi; the B_lo copy of the B ring sits
// `blo` descriptor units (16 bytes) after B.
#define BSRP_X3_HEAD \
    "{\n.reg .pred p;\n.reg .b32 ah<8>, al<8>, bl<8>, bm<8>;\n.reg .b64 b<8>, c<8>;\nelect.sync _|p, 0xffffffff;\n"
#define BSRP_X3_STEP(S)                                                                                          \
    "add.u32 ah" #S ", %2, " #S "*%7;\nadd.u32 al" #S ", ah" #S ", %9;\nadd.u32 bl" #S ", %3, " #S "*%8;\n"        \
    "add.u32 bm" #S ", bl" #S ", %6;\nmov.b64 b" #S ", {bl" #S ", %4};\nmov.b64 c" #S ", {bm" #S ", %4};\n"          \
    "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah" #S "], b" #S ", %5, 1;\n"                                    \
    "@p tcgen05.mma.cta_group::1.kind::tf32 [%1], [al" #S "], b" #S ", %5, 1;\n"                                    \
    "@p tcgen05.mma.cta_group::1.kind::tf32 [%1], [ah" #S "], c" #S ", %5, 1;\n"
#define BSRP_X3_ARGS                                                                                  \
    ::"r"(d_tmem), "r"(dc_tmem), "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(blo), "n"(AKC), \
        "n"(BK16), "n"(ACOLS)
template <int NSTEP, int AKC, int BK16, int ACOLS>
__device__ __forceinline__ void tc_mma_x3_run(uint32_t d_tmem, uint32_t dc_tmem, uint32_t a_tmem, uint32_t b_lo,
                                              uint32_t b_hi, uint32_t idesc, uint32_t blo) {
    if constexpr (NSTEP == 4) {
        asm volatile(BSRP_X3_HEAD BSRP_X3_STEP(0) BSRP_X3_STEP(1) BSRP_X3_STEP(2) BSRP_X3_STEP(3) "}\n" BSRP_X3_ARGS);
    } else {
        static_assert(NSTEP == 8, "k steps per block (b = 32 or 64)");
        asm volatile(BSRP_X3_HEAD BSRP_X3_STEP(0) BSRP_X3_STEP(1) BSRP_X3_STEP(2) BSRP_X3_STEP(3) BSRP_X3_STEP(4)
                         BSRP_X3_STEP(5) BSRP_X3_STEP(6) BSRP_X3_STEP(7) "}\n" BSRP_X3_ARGS);
    }
}
#undef BSRP_X3_HEAD
#undef BSRP_X3_STEP
#undef BSRP_X3_ARGS

// UMMA shared-memory matrix descriptor (sm_100): start, leading-byte offset
// (stride between MN atoms for swizzled MN-major), stride-byte offset (between
// K groups), version 1, swizzle layout type.
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
// A K-major (A in TMEM), B MN-major, M = 128, N = n.
template <int KIND>
__host__ __device__ __forceinline__ uint32_t instr_desc(uint32_t n) {
    constexpr uint32_t fmt = KIND == 1 ? 1u : 2u;  // bf16 or tf32 (KIND 0 and 2)
    return (1u << 4) | (fmt << 7) | (fmt << 10) | (0u << 15) | (1u << 16) | ((n >> 3) << 17) | ((128u >> 4) << 24);
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
// 8 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t *v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

struct Params {
    const int32_t *rowptr, *colidx;
    const uint8_t *values;
    float *dW, *ws;
    float *mc;                   // multimem (NVLS multicast) address of the summed dW, or null
    int mc_unicast;              // 1: mc is a plain device address, reduced with red.global (test hook)
    int64_t nbr, N, K;
    int nkr, nsplit, kr_blocks;  // kcol range = kr_blocks blocks
    int nbslots, na, mode;       // B-ring block slots, TMEM A buffers; mode: 0 store, 1 reduce-add, 3 partial -> ws[split],
                                 // 4 multimem reduce-add into p.mc (NVLS; one split)
    int chunk_steps;             // steps of one metadata chunk (rowptr + colidx staged in smem)
    int sa;                      // shared-memory A ring stages
    uint32_t a_col0;             // first TMEM column of the A buffers
    uint32_t corr_col;           // FP32 grade: TMEM column of the correction accumulator (main + corr_col)
    int pdl_trig;                // PDL successor trigger: 0 none, 1 at start, 2 at the epilogue
};

// KIND: 0 = tf32 (one MMA per k step, operands truncated to tf32 by the tensor
// core), 1 = bf16, 2 = FP32 grade (3xTF32): every operand x is split into
// hi = x with the low 13 mantissa bits cleared (exactly a tf32 value) and
// lo = x - hi (exact in fp32), and
//   D_main += A_hi . B_hi        D_corr += A_lo . B_hi + A_hi . B_lo
// (A_lo . B_lo, ~2^-22 relative, is dropped); D = D_main + D_corr with one fp32
// round-to-nearest add in the epilogue.  The corrections have their own TMEM
// accumulator so the main chain takes one truncating accumulation per k step,
// as in the tf32 path, instead of three.
template <int KIND, int B>
struct Cfg {
    static constexpr bool X3 = KIND == 2;
    static constexpr int ES = KIND == 1 ? 2 : 4;
    static constexpr int UK = KIND == 1 ? 16 : 8;           // MMA K per instruction
    static constexpr int A_COLS = B * ES / 4;               // TMEM columns of one block row's slab (32-bit, K packed)
    static constexpr int A_ROW = X3 ? 2 * A_COLS : A_COLS;  // per block row: hi slab [+ lo slab]
    static constexpr int A_KCOLS = UK * ES / 4;             // TMEM columns per MMA K step (8)
    static constexpr int BW = (B * ES < 128) ? B * ES : 128;  // block row bytes per swizzle atom
    static constexpr int B_ATOMS = B * ES / BW;
    static constexpr int BLOCK_BYTES = B * B * ES;
    static constexpr int B_LBO = B * BW;                    // bytes between N atoms
    // MN-major tf32 operands only exist in the 128-byte swizzle with 32-byte
    // atomicity (UMMA layout type 1, TMA SWIZZLE_128B_ATOM_32B): 128-byte rows,
    // 32-byte chunks permuted by (row % 4), K groups of 4 rows.  bf16 uses the
    // plain SW32/64/128 layouts with K groups of 8 rows.
    static constexpr bool TF32 = KIND != 1;
    static constexpr int KGROUP = TF32 ? 4 : 8;             // K rows per swizzle group
    static constexpr int B_SBO = KGROUP * BW;               // bytes between K groups of B
    static constexpr int B_KSTEP = UK * BW;                 // bytes per MMA K step in B
    static constexpr uint32_t B_LAYOUT = TF32 ? 1u : BW == 128 ? 2u : BW == 64 ? 4u : 6u;  // SW128_32B / SW128 / SW64 / SW32
    static_assert(!TF32 || BW == 128, "tf32 MN-major operands need 128-byte block rows (b >= 32)");
    static constexpr int MAX_RUN = 256 / B;                 // blocks per MMA (N <= 256)
    // blocks per B TMA (a row's kept blocks are loaded G at a time, the count rounded up to
    // G slots); the FP32 grade loads them one by one: its B ring is half as deep (B_lo copy)
    // and every rounded-up slot would also be split (measured faster)
    static constexpr int G = X3 ? 1 : BLOCK_BYTES >= 8192 ? 1 : BLOCK_BYTES >= 2048 ? 4 : 8;
    // One pipeline step = R consecutive block rows (64 dY rows): one dY slab TMA,
    // one TMEM A buffer, one trip through every barrier.  The per-step
    // synchronisation (each mbarrier wait costs ~100 cycles even when the phase
    // has completed) is paid once per 64 rows instead of once per block row.
    // FP32 grade: one block row per step (its A buffer holds hi and lo).  tf32 at
    // b = 32: one block row too -- a 32-column A buffer leaves room for four of them
    // next to a 384-column accumulator (two with 64-row steps); measured C2 76.7 ->
    // 65.8 us, B24 fc1 shard 245 -> 207 us.  bf16 keeps 64-row steps (R = 1 measured
    // slower there: 48 -> 57 us; its 64-row A buffer is 32 columns already).
    static constexpr int R = (X3 || B >= 64 || (KIND == 0 && B == 32)) ? 1 : 64 / B;
    static constexpr int SROWS = R * B;                     // dY rows per step
    static constexpr int A_STEP = R * A_ROW;                // TMEM columns of one step's A buffer
    static constexpr int SLAB = SROWS * 128 * ES;           // one dY slab (SROWS rows x 128 columns, row-major)
    static constexpr int ACC_MULT = X3 ? 2 : 1;             // accumulators (main [+ correction])
    // A single warp issues one tcgen05.mma per ~45-55 cycles (measured,
    // DESIGN.md §6); the FP32 grade issues 3x the MMAs, from four warps.
    static constexpr int ISSUERS = X3 ? 4 : 2;
    static constexpr int SPLITTERS = X3 ? 4 : 0;            // warps splitting landed B blocks into hi / lo
    // warps: 0 B producer, 1-2 MMA, 3 planner, 4-7 A movers (even steps) + epilogue,
    // 8 A producer, 9-12 A movers (odd steps); FP32 grade: 13-14 splitters, 15-16 MMA,
    // 17-18 splitters -- the four MMA warps sit on the four SM sub-partitions (warp % 4 =
    // 1, 2, 3, 0), as in the issue-rate micro-benchmark (at C2 the placement measured
    // the same as warps 1, 2, 13, 14: the per-step pipeline, not the issue slot, paces it)
    static constexpr int WARPS = 13 + (ISSUERS - 2) + SPLITTERS;
    static constexpr int THREADS = 32 * WARPS;
    static constexpr int BAR1_THREADS = 32 * (8 + ISSUERS);  // issuers + A movers (accumulator zeroed)
    __device__ static constexpr int issuer(int w) {          // MMA issuer index of warp w, or -1
        return w == 1 ? 0 : w == 2 ? 1 : (X3 && w == 15) ? 2 : (X3 && w == 16) ? 3 : -1;
    }
    __device__ static constexpr int splitter(int w) {        // splitter index of warp w, or -1
        return !X3 ? -1 : w == 13 ? 0 : w == 14 ? 1 : w == 17 ? 2 : w == 18 ? 3 : -1;
    }
};

// This thread's dY column of the step's slab in shared memory (row-major, 128
// columns per row): SROWS values; consecutive lanes read consecutive elements
// (conflict-free).
template <int KIND, int N_>
__device__ __forceinline__ void lds_slab(uint32_t (&v)[N_], uint32_t saddr) {
    static_assert(KIND == 0 || KIND == 1, "lds_slab: tf32 / fp32-grade use KIND 0");
#pragma unroll
    for (int k = 0; k < N_; ++k) {
        if constexpr (KIND == 1) {
            unsigned short h;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(saddr + k * 256));
            v[k] = h;
        } else {
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v[k]) : "r"(saddr + k * 512));
        }
    }
}

// The slab into TMEM columns [taddr, taddr + N_ * ES / 4) of this thread's lane
// (K-major A: column j holds K element j, or K elements 2j, 2j+1 for bf16).
// fp32 -> (hi, lo): hi keeps the sign, exponent and the 10 mantissa bits a tf32
// operand holds; lo = x - hi is exact in fp32 (and again truncated to tf32 by the
// tensor core: a 2^-22-relative term).
__device__ __forceinline__ uint32_t tf32_hi(uint32_t x) { return x & 0xffffe000u; }
__device__ __forceinline__ uint32_t tf32_lo(uint32_t x) {
    return __float_as_uint(__uint_as_float(x) - __uint_as_float(x & 0xffffe000u));
}

template <int KIND, int N_>
__device__ __forceinline__ void store_slab(uint32_t taddr, const uint32_t (&v)[N_]) {
    if constexpr (KIND == 1) {
#pragma unroll
        for (int c = 0; c < N_ / 2; c += 8) {
            uint32_t w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = v[2 * (c + i)] | (v[2 * (c + i) + 1] << 16);
            tmem_st8(taddr + c, w);
        }
    } else if constexpr (KIND == 2) {
        // hi slab at [taddr, taddr + N_), lo slab right after it
#pragma unroll
        for (int c = 0; c < N_; c += 8) {
            uint32_t h[8], l[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                h[i] = tf32_hi(v[c + i]);
                l[i] = tf32_lo(v[c + i]);
            }
            tmem_st8(taddr + c, h);
            tmem_st8(taddr + N_ + c, l);
        }
    } else {
#pragma unroll
        for (int c = 0; c < N_; c += 8) tmem_st8(taddr + c, v + c);
    }
}

template <int KIND, int B>
__global__ void __launch_bounds__(Cfg<KIND, B>::THREADS, 1)
    wgrad_tc_kernel(const __grid_constant__ CUtensorMap tm_dy, const __grid_constant__ CUtensorMap tm_val,
                    const __grid_constant__ CUtensorMap tm_dw, const __grid_constant__ CUtensorMap tm_ws, Params p) {
    using C = Cfg<KIND, B>;
    constexpr int R = C::R;
    // shared memory: [A ring: sa x SLAB][B ring: nbslots x BLOCK_BYTES][FP32 grade: B_lo ring, same
    //   size][slot use: kStages][mbarriers][TMEM slot][step records][sub-row records][run words]
    //   [rowptr scratch][colidx scratch]
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *ringA = smem;
    uint8_t *ringB = ringA + (size_t)p.sa * C::SLAB;
    const size_t ringB_bytes = (size_t)p.nbslots * C::BLOCK_BYTES;
    uint32_t *s_used = reinterpret_cast<uint32_t *>(ringB + ringB_bytes * C::ACC_MULT);
    uint64_t *full = reinterpret_cast<uint64_t *>(s_used + kStages);
    uint64_t *empty = full + kStages;
    uint64_t *afull = empty + kStages;     // [kMaxA]
    uint64_t *aempty = afull + kMaxA;      // [kMaxA]
    uint64_t *sfull = aempty + kMaxA;      // [kMaxSA] A ring: slab landed (TMA bytes)
    uint64_t *sempty = sfull + kMaxSA;     // [kMaxSA] A ring: slab read by the four A movers
    uint64_t *accfull = sempty + kMaxSA;
    uint64_t *plan_full = accfull + 1;     // [2]
    uint64_t *plan_empty = plan_full + 2;  // [2]
    uint64_t *lofull = plan_empty + 2;     // [kStages] FP32 grade: the step's B blocks split into hi / lo
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(lofull + kStages);
    // s_steps [2][kStepCap] (one per step of the chunk): x = MMA runs, y = B-ring
    //   slots used (needs + wasted tail slots) | in-sequence << 30, z = first run
    //   word, w = B bytes
    // s_sub [2][kStepCap * R] (one per block row): x = first value index, y = first
    //   B-ring slot | blocks to load (G rounded) << 16
    // s_runs [2][kColCap]: one ready-to-issue word per MMA run: TMEM column |
    //   B-ring slot << 10 | run length (blocks) << 22 | block row within the step << 28
    int4 *s_steps = reinterpret_cast<int4 *>((reinterpret_cast<uintptr_t>(s_tmem + 4) + 15) & ~uintptr_t(15));
    uint2 *s_sub = reinterpret_cast<uint2 *>(s_steps + 2 * kStepCap);
    uint32_t *s_runs = reinterpret_cast<uint32_t *>(s_sub + 2 * kStepCap * R);
    int32_t *s_rp = reinterpret_cast<int32_t *>(s_runs + 2 * kColCap);  // [kStepCap * R + 1]
    uint16_t *s_col = reinterpret_cast<uint16_t *>(s_rp + kStepCap * R + 1);  // [kColCap]

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
    const int64_t nst = (p.nbr + R - 1) / R;  // steps (the last one may hold fewer than R block rows)
    const int64_t Sb = (int64_t)split * nst / p.nsplit, Se = (int64_t)(split + 1) * nst / p.nsplit;
    // chunk 0 is short (8 steps) so the first plan is ready early; later chunks are chunk_steps long
    const int first_steps = min(8, p.chunk_steps);
    const int64_t nsteps_cta = Se - Sb;
    const int nchunks = nsteps_cta <= first_steps ? (nsteps_cta > 0 ? 1 : 0)
                                                  : 1 + (int)((nsteps_cta - first_steps + p.chunk_steps - 1) / p.chunk_steps);
    auto chunk_start = [&](int c) -> int64_t {
        return c == 0 ? Sb : Sb + first_steps + (int64_t)(c - 1) * p.chunk_steps;
    };
    auto chunk_len = [&](int c) -> int {
        return (int)min((int64_t)(c == 0 ? first_steps : p.chunk_steps), Se - chunk_start(c));
    };
    // The first n_spec steps are in the sequence whether or not they keep a block:
    // their dY slabs are requested before the planner has read rowptr/colidx, so
    // the first HBM round trip overlaps the plan (an empty step costs one slab).
    const int n_spec = (int)min((int64_t)min(p.sa, first_steps), nsteps_cta);
    // MMA issuer i owns accumulator blocks [jb(i), jb(i + 1)); runs never cross a boundary
    auto jb = [&](int i) -> int { return (i * nbJ + C::ISSUERS - 1) / C::ISSUERS; };
    auto is_boundary = [&](int J) -> bool {
        bool r = false;
#pragma unroll
        for (int i = 1; i < C::ISSUERS; ++i) r |= J == jb(i);
        return r;
    };

    if (warp == 0 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_val)) : "memory");
    if (warp == 8 && lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dy)) : "memory");
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + s, 1);              // the B producer (+ TMA bytes)
            mbar_init(empty + s, C::ISSUERS);    // the MMA warps' commits
            mbar_init(lofull + s, C::SPLITTERS ? C::SPLITTERS : 1);  // one arrival per splitter warp
        }
        for (int a = 0; a < kMaxA; ++a) {
            mbar_init(afull + a, 4);              // one arrival per A-mover warp
            mbar_init(aempty + a, C::ISSUERS);    // the MMA warps' commits
        }
        for (int s = 0; s < kMaxSA; ++s) {
            mbar_init(sfull + s, 1);   // the A producer's expect_tx (+ TMA bytes)
            mbar_init(sempty + s, 4);  // one arrival per A-mover warp
        }
        mbar_init(accfull, C::ISSUERS);
        for (int i = 0; i < 2; ++i) {
            mbar_init(plan_full + i, 1);
            mbar_init(plan_empty + i, C::ISSUERS);  // the MMA warps release a plan chunk
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                     "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    // PDL: the prologue above overlapped the predecessor's tail; no global
    // access before this point.  The split-K reduce may be scheduled now.
    pdl_wait();
    if (p.pdl_trig == 1) pdl_trigger();

    if (warp == 3) {
        // ------------------------------------------------ step planner
        // For each chunk of steps: rowptr + colidx into shared memory, then one
        // lane per step derives, for each of its block rows, the kept blocks in
        // this CTA's column range, their B-ring slots (G rounded) and first value
        // index, and the step's MMA runs (consecutive block columns of one block
        // row, <= MAX_RUN blocks, split at the issuers' column boundary).  B-ring
        // slots are handed out in sequence order (a block row that would wrap
        // starts at slot 0 and the tail slots are skipped), so every slot is fixed
        // here, not at run time: the run words are final and the B producer only
        // reclaims slots and issues TMAs.  Double-buffered, one chunk ahead.
        int bhead = 0;  // B-ring head, the same in every lane
        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            const int64_t Rc = chunk_start(c) * R;  // first block row of the chunk
            const int ns = chunk_len(c);
            const int nrow = (int)(min((chunk_start(c) + ns) * R, p.nbr) - Rc);
            for (int i = lane; i <= nrow; i += 32) s_rp[i] = __ldg(p.rowptr + Rc + i);
            __syncwarp();
            const int base = s_rp[0], total = s_rp[nrow] - base;
            for (int e = lane; e < total; e += 32) s_col[e] = (uint16_t)__ldg(p.colidx + base + e);
            if (lane == 0) mbar_wait(plan_empty + buf, ((c >> 1) & 1) ^ 1);
            __syncwarp();
            int4 *steps = s_steps + buf * kStepCap;
            uint2 *subs = s_sub + buf * kStepCap * R;
            uint32_t *runs = s_runs + buf * kColCap;
            int run_base = 0;
            for (int s0 = 0; s0 < ns; s0 += 32) {
                const int st = s0 + lane;
                int q0[R], cnt[R];
                int nruns = 0, nonempty = 0;
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int r = st * R + q;
                    q0[q] = 0;
                    cnt[q] = 0;
                    if (st < ns && r < nrow) {
                        int a = s_rp[r] - base, z = s_rp[r + 1] - base;
                        nonempty |= z > a;
                        if (p.nkr > 1) {
                            while (a < z && (int)s_col[a] < J0) ++a;
                            int y = a;
                            while (y < z && (int)s_col[y] < J0 + nbJ) ++y;
                            z = y;
                        }
                        q0[q] = a;
                        cnt[q] = z - a;
                        int jprev = -2, rlen = 0;
                        for (int k = 0; k < cnt[q]; ++k) {
                            const int J = (int)s_col[a + k] - J0;
                            if (J == jprev + 1 && rlen < C::MAX_RUN && !is_boundary(J)) {
                                ++rlen;
                            } else {
                                ++nruns;
                                rlen = 1;
                            }
                            jprev = J;
                        }
                    }
                }
                const int inseq = st < ns && (nonempty || (c == 0 && st < n_spec));
                // exclusive warp scan of nruns -> this step's run offset
                int incl = nruns;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int off = run_base + incl - nruns;
                run_base += __shfl_sync(0xffffffffu, incl, 31);
                // B-ring slots, in sequence order: one contiguous range per step (its block
                // rows back to back, each G rounded); a step that would wrap starts at
                // slot 0 and the tail slots are skipped (counted as used)
                int need = 0;
#pragma unroll
                for (int q = 0; q < R; ++q) need += (cnt[q] + C::G - 1) / C::G * C::G;
                int step0 = 0, used = 0;
                for (uint32_t m = __ballot_sync(0xffffffffu, inseq != 0); m; m &= m - 1) {
                    const int l = __ffs(m) - 1;
                    const int nd = __shfl_sync(0xffffffffu, need, l);
                    const int ws = bhead + nd > p.nbslots ? p.nbslots - bhead : 0;
                    const int s_0 = ws ? 0 : bhead;
                    if (lane == l) {
                        step0 = s_0;
                        used = nd + ws;
                    }
                    bhead = s_0 + nd;
                    if (bhead == p.nbslots) bhead = 0;
                }
                const int bytes = need * C::BLOCK_BYTES;
                int slot0[R];
                slot0[0] = step0;
#pragma unroll
                for (int q = 1; q < R; ++q) slot0[q] = slot0[q - 1] + (cnt[q - 1] + C::G - 1) / C::G * C::G;
                if (st < ns) {
                    int k = off;
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int nd = (cnt[q] + C::G - 1) / C::G * C::G;
                        subs[st * R + q] = make_uint2((uint32_t)(base + q0[q]), (uint32_t)slot0[q] | ((uint32_t)nd << 16));
                        int jprev = -2, rlen = 0, rstart = 0;
                        auto emit = [&]() {
                            runs[k++] = (uint32_t)((jprev - rlen + 1) * B) | ((uint32_t)(slot0[q] + rstart) << 10) |
                                        ((uint32_t)rlen << 22) | ((uint32_t)q << 28);
                        };
                        for (int i = 0; i < cnt[q]; ++i) {
                            const int J = (int)s_col[q0[q] + i] - J0;
                            if (J == jprev + 1 && rlen < C::MAX_RUN && !is_boundary(J)) {
                                ++rlen;
                            } else {
                                if (rlen) emit();
                                rstart = i;
                                rlen = 1;
                            }
                            jprev = J;
                        }
                        if (rlen) emit();
                    }
                    steps[st] = make_int4(nruns, used | (inseq << 30), off, bytes);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(plan_full + buf);
            // Warm L2 with the chunk's stored blocks (one bulk prefetch per 32 KB, issued by
            // the first n-tile's CTA): the B loads of the 128-column tiles sharing these
            // block rows then hit L2 instead of all waiting on the same HBM fill.
            if (nt == 0) {
                const int64_t b0 = (int64_t)base * C::BLOCK_BYTES, nb = (int64_t)total * C::BLOCK_BYTES;
                for (int64_t o = (int64_t)lane * 32768; o < nb; o += 32 * 32768) {
                    const uint32_t sz = (uint32_t)min((int64_t)32768, nb - o);
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.values + b0 + o), "r"(sz) : "memory");
                }
            }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ B producer (one thread)
            // Walks the step sequence (step j uses stage j % kStages): once the step's
            // planned slots are free (stages and slots are reclaimed in order as the
            // MMA commits arrive on `empty`), loads each block row's kept blocks G per
            // 4-D TMA.
            int j = 0;  // steps issued so far
            int tail = 0, bfree = p.nbslots;
            const uint32_t sB0 = smem_u32(ringB);
            for (int c = 0; c < nchunks; ++c) {
                const int buf = c & 1;
                const int ns = chunk_len(c);
                mbar_wait(plan_full + buf, (c >> 1) & 1);
                const int4 *steps = s_steps + buf * kStepCap;
                const uint2 *subs = s_sub + buf * kStepCap * R;
                for (int st = 0; st < ns; ++st) {
                    const int4 rs = steps[st];
                    if (!(rs.y >> 30)) continue;
                    const int stage = j % kStages;
                    const int used = rs.y & 0xFFFFF;
                    // reclaim the oldest steps until the planned slots are free: enough
                    // free slots past the head, or an empty ring (a step that wrapped may
                    // count more than nbslots; bfree then goes negative until it is reclaimed)
                    while (j - tail >= kStages || (bfree < used && bfree < p.nbslots)) {
                        mbar_wait(empty + tail % kStages, (uint32_t)(tail / kStages) & 1u);
                        bfree += (int)s_used[tail % kStages];
                        ++tail;
                    }
                    s_used[stage] = (uint32_t)used;
                    bfree -= used;
                    mbar_arrive_expect_tx(full + stage, (uint32_t)rs.w);
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const uint2 sb = subs[st * R + q];
                        const int nd = (int)(sb.y >> 16);
                        const uint32_t dst = sB0 + (sb.y & 0xFFFFu) * C::BLOCK_BYTES;
                        for (int g = 0; g < nd; g += C::G)
                            tma_load_4d(&tm_val, full + stage, dst + g * C::BLOCK_BYTES, 0, 0, 0, (int)sb.x + g);
                    }
                    ++j;
                }
            }
        }
    } else if (C::issuer(warp) >= 0) {
        // ------------------------------------------------ MMA issuers (whole warps, one elected lane issues)
        // Issuer i (warps 1, 2, then 13.. for the FP32 grade) issues the runs in
        // accumulator blocks [jb(i), jb(i + 1)): a warp issues one tcgen05.mma per
        // ~45-55 cycles whatever its shape (measured), so several warps on
        // different SM sub-partitions keep the tensor pipe fed.  Each walks the
        // plan: a ballot over 32 step records finds the steps in the sequence,
        // lane i loads run word i of the step with ONE shared load, a ballot
        // selects this warp's runs and each run word becomes warp-uniform with a
        // single masked redux.
        tc_fence_before();
        asm volatile("bar.sync 1, %0;" ::"r"(C::BAR1_THREADS) : "memory");  // accumulator zeroed by warps 4-7
        tc_fence_after();
        const int iw = C::issuer(warp);
        const uint32_t col_lo = (uint32_t)(jb(iw) * B), col_hi = (uint32_t)(jb(iw + 1) * B);
        // warp-uniform copies (REDUX results live in uniform registers)
        const uint32_t tmem_u = __reduce_or_sync(0xffffffffu, tmem);
        const uint64_t b_desc0 = smem_desc(smem_u32(ringB), C::B_LBO, C::B_SBO, C::B_LAYOUT);
        const uint32_t b_lo0 = __reduce_or_sync(0xffffffffu, (uint32_t)b_desc0);
        const uint32_t b_hi = __reduce_or_sync(0xffffffffu, (uint32_t)(b_desc0 >> 32));
        const uint32_t blo_off = __reduce_or_sync(0xffffffffu, (uint32_t)(ringB_bytes >> 4));  // B_lo ring (FP32 grade)
        const uint32_t corr = __reduce_or_sync(0xffffffffu, p.corr_col);
        const uint32_t idesc0 = instr_desc<KIND>(0u);
        const uint32_t a_tm0 = tmem_u + p.a_col0;
        uint64_t *ready = C::X3 ? lofull : full;  // FP32 grade: B split into hi / lo by the splitter warps
        int stage = 0, a = 0;
        uint32_t phase = 0, aphase = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            const int ns = chunk_len(c);
            mbar_wait(plan_full + buf, (c >> 1) & 1);
            const int4 *steps = s_steps + buf * kStepCap;
            const uint32_t *runs = s_runs + buf * kColCap;
            for (int s0 = 0; s0 < ns; s0 += 32) {
                const int4 rec = s0 + lane < ns ? steps[s0 + lane] : make_int4(0, 0, 0, 0);
                for (uint32_t seq = __ballot_sync(0xffffffffu, (rec.y >> 30) != 0); seq; seq &= seq - 1) {
                    const int l = __ffs(seq) - 1;
                    const uint32_t nruns = __reduce_or_sync(0xffffffffu, lane == l ? (uint32_t)rec.x : 0u);
                    const uint32_t off = __reduce_or_sync(0xffffffffu, lane == l ? (uint32_t)rec.z : 0u);
                    mbar_wait(ready + stage, phase);
                    mbar_wait(afull + a, aphase);
                    tc_fence_after();
                    const uint32_t a_tm = a_tm0 + (uint32_t)(a * C::A_STEP);
                    for (uint32_t w0 = 0; w0 < nruns; w0 += 32) {
                        const uint32_t wl = w0 + lane < nruns ? runs[off + w0 + lane] : 0u;
                        const uint32_t col = wl & 0x3FFu;
                        uint32_t mine = __ballot_sync(0xffffffffu, w0 + lane < nruns && col >= col_lo && col < col_hi);
                        while (mine) {
                            const int i = __ffs(mine) - 1;
                            mine &= mine - 1;
                            const uint32_t rw = __reduce_or_sync(0xffffffffu, lane == i ? wl : 0u);
                            const uint32_t d = tmem_u + (rw & 0x3FFu);
                            const uint32_t b_lo = b_lo0 + ((rw >> 10) & 0xFFFu) * (uint32_t)(C::BLOCK_BYTES >> 4);
                            const uint32_t idesc = idesc0 | ((((rw >> 22) & 0x3Fu) * (uint32_t)B >> 3) << 17);
                            const uint32_t a_q = a_tm + ((rw >> 28) & 0x3u) * (uint32_t)C::A_ROW;
                            if constexpr (C::X3)
                                tc_mma_x3_run<B / C::UK, C::A_KCOLS, (C::B_KSTEP >> 4), C::A_COLS>(d, d + corr, a_q, b_lo, b_hi,
                                                                                                 idesc, blo_off);
                            else
                                tc_mma_ts_run<KIND, B / C::UK, C::A_KCOLS, (C::B_KSTEP >> 4)>(d, a_q, b_lo, b_hi, idesc);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) {
                        tc_commit(empty + stage);  // frees the stage (and its B slots) once these MMAs complete
                        tc_commit(aempty + a);     // frees the A buffer
                    }
                    __syncwarp();
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                    if (++a == p.na) { a = 0; aphase ^= 1; }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(plan_empty + buf);  // this chunk's plan is no longer read
        }
        if (lane == 0) tc_commit(accfull);
    } else if (C::X3 && C::splitter(warp) >= 0) {
        // ------------------------------------------------ B splitters (FP32 grade)
        // Walk the B producer's step sequence; once a step's blocks have landed
        // (`full`), write lo(x) = x - hi(x) of every value x at the same offset of
        // the B_lo ring (element-wise, so the swizzled layout and the MMA
        // descriptors carry over), then make the generic-proxy writes visible to
        // the tensor core and arrive on `lofull`.  hi(x) itself is not written:
        // kind::tf32 reads an fp32 operand as its sign, exponent and top 10
        // mantissa bits, i.e. exactly hi(x) (truncation; writing hi(x) explicitly
        // gave bit-identical dW, R15/R17).
        const int sw = C::splitter(warp);
        int j = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            const int ns = chunk_len(c);
            mbar_wait(plan_full + buf, (c >> 1) & 1);
            const int4 *steps = s_steps + buf * kStepCap;
            const uint2 *subs = s_sub + buf * kStepCap * R;
            for (int st = 0; st < ns; ++st) {
                const int4 rs = steps[st];
                if (!(rs.y >> 30)) continue;
                const int stage = j % kStages;
                mbar_wait(full + stage, (uint32_t)(j / kStages) & 1u);
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const uint2 sb = subs[st * R + q];
                    const int nd = (int)(sb.y >> 16);
                    const uint32_t hi0 = smem_u32(ringB) + (sb.y & 0xFFFFu) * (uint32_t)C::BLOCK_BYTES;
                    const uint32_t lo_off = (uint32_t)ringB_bytes;
                    const int n16 = nd * (C::BLOCK_BYTES / 16);
                    for (int i = sw * 32 + lane; i < n16; i += 32 * C::SPLITTERS) {
                        const uint32_t a = hi0 + (uint32_t)i * 16u;
                        uint32_t x0, x1, x2, x3;
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3) : "r"(a));
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a + lo_off), "r"(tf32_lo(x0)),
                                     "r"(tf32_lo(x1)), "r"(tf32_lo(x2)), "r"(tf32_lo(x3)) : "memory");
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(lofull + stage);
                ++j;
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ A producer (warp 8) and A movers (warps 4-7, 9-12)
        // Step j of the sequence: warp 8 lane 0 requests its dY slab (one 2-D TMA,
        // SROWS x 128, row-major) into A-ring stage j % sa as soon as the stage is
        // free; the movers move it shared -> registers (warp w owns TMEM lanes
        // 32 (w % 4) .. + 31, thread lane m = dY column n0 + m) -> tcgen05.st into
        // A buffer j % na.  Warps 4-7 take the even steps, warps 9-12 the odd ones.
        // Step-sequence cursor, the B producer's sequence: the n_spec speculative
        // steps, then every step with at least one stored block (rowptr read 32
        // steps at a time, one ballot).  Producer and movers each run it; it never
        // waits on the planner.
        int64_t wS = Sb + n_spec, wbase = 0, sS = Sb;
        uint32_t wmask = 0;
        auto next_step = [&](int64_t &S) -> bool {
            if (sS < Sb + n_spec) {
                S = sS++;
                return true;
            }
            while (!wmask) {
                if (wS >= Se) return false;
                const int64_t s = wS + lane;
                const bool ne = s < Se && __ldg(p.rowptr + min((s + 1) * R, p.nbr)) > __ldg(p.rowptr + s * R);
                wmask = __ballot_sync(0xffffffffu, ne);
                wbase = wS;
                wS += 32;
            }
            S = wbase + (__ffs(wmask) - 1);
            wmask &= wmask - 1;
            return true;
        };
        const uint32_t sA0 = smem_u32(ringA);
        if (warp == 8) {
            int64_t S;
            for (int j = 0; next_step(S); ++j) {
                if (lane == 0) {
                    const int s = j % p.sa;
                    if (j >= p.sa) mbar_wait(sempty + s, (uint32_t)((j / p.sa) - 1) & 1u);
                    mbar_arrive_expect_tx(sfull + s, (uint32_t)C::SLAB);
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                            sA0 + (uint32_t)(s * C::SLAB)),
                        "l"(reinterpret_cast<uint64_t>(&tm_dy)), "r"(n0), "r"((int)(S * C::SROWS)),
                        "r"(smem_u32(sfull + s))
                        : "memory");
                }
                __syncwarp();
            }
        } else {
            const int ew = warp & 3;
            const int par = warp >= 9;
            const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
            // zero the accumulator columns this CTA owns (MMAs then always accumulate)
            if (!par) {
                for (int c = 0; c < nbJ * B; c += 16) tmem_st16_zero(tmem + lane_base + c);
                if constexpr (C::X3)
                    for (int c = 0; c < nbJ * B; c += 16) tmem_st16_zero(tmem + lane_base + p.corr_col + c);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            tc_fence_before();
            asm volatile("bar.sync 1, %0;" ::"r"(C::BAR1_THREADS) : "memory");
            tc_fence_after();
            const uint32_t a_tm0 = tmem + lane_base + p.a_col0;
            const uint32_t my_col = (uint32_t)((ew * 32 + lane) * C::ES);
            int j = 0;
            int64_t S;
            for (; next_step(S); ++j) {
                if ((j & 1) != par) continue;
                const int s = j % p.sa;
                mbar_wait(sfull + s, (uint32_t)(j / p.sa) & 1u);
                uint32_t v[C::SROWS];
                lds_slab<(KIND == 1 ? 1 : 0), C::SROWS>(v, sA0 + (uint32_t)(s * C::SLAB) + my_col);
                __syncwarp();
                if (lane == 0) mbar_arrive(sempty + s);
                const int ab = j % p.na;
                if (j >= p.na) mbar_wait(aempty + ab, (uint32_t)((j / p.na) - 1) & 1u);
                tc_fence_after();
                if constexpr (C::X3) {  // per block row q: hi slab, then its lo slab (A_ROW columns)
#pragma unroll
                    for (int q = 0; q < R; ++q)
                        store_slab<2, B>(a_tm0 + (uint32_t)(ab * C::A_STEP + q * C::A_ROW),
                                         *reinterpret_cast<const uint32_t(*)[B]>(v + q * B));
                }
                else store_slab<KIND, C::SROWS>(a_tm0 + (uint32_t)(ab * C::A_STEP), v);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(afull + ab);
            }
        }
    }
    if (warp >= 4 && warp < 8) {
        // ------------------------------------------------ epilogue
        // TMEM -> registers -> a [32 kcol][128 n] fp32 staging tile in the (now
        // idle) rings -> one TMA bulk tensor store (or reduce-add) per 16 kcols.
        // Full 512-byte row segments leave the SM through the TMA unit instead of
        // 128-byte scattered STGs.  mode 3 stores this split's partial tile into
        // its own workspace slice (summed afterwards in split order:
        // deterministic); mode 1 adds into dW (accumulate, one split).
        mbar_wait_sleep(accfull, 0);
        if (p.pdl_trig == 2) pdl_trigger();
        tc_fence_after();
        const int ew = warp - 4;
        const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
        float *stage_buf = reinterpret_cast<float *>(ringA);  // 2 x [32][128] over the idle A/B rings
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
            if (p.mode == 4) {  // fused all-reduce: add this tile into the multicast dW (NVSwitch reduction)
                uint32_t w[32];
                if constexpr (C::X3) {
                    TMEM_LD16(tmem + lane_base + p.corr_col + c, w);
                    TMEM_LD16(tmem + lane_base + p.corr_col + c + 16, (w + 16));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int nrow = min(32, ncols - c);
                float *dst = p.mc + (int64_t)(row0 + c) * p.N + n0 + ew * 32 + lane;
#pragma unroll
                for (int i = 0; i < 32; ++i) {  // unrolled: v, w stay in registers
                    if (i >= nrow) break;
                    float x = __uint_as_float(v[i]);
                    if constexpr (C::X3) x = __fadd_rn(x, __uint_as_float(w[i]));
                    if (p.mc_unicast)
                        asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(dst + (int64_t)i * p.N), "f"(x)
                                     : "memory");
                    else
                        asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(dst + (int64_t)i * p.N),
                                     "f"(x)
                                     : "memory");
                }
                continue;
            }
            if constexpr (C::X3) {  // D = D_main + D_corr, one round-to-nearest fp32 add
                uint32_t w[32];
                TMEM_LD16(tmem + lane_base + p.corr_col + c, w);
                TMEM_LD16(tmem + lane_base + p.corr_col + c + 16, (w + 16));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__fadd_rn(__uint_as_float(v[i]), __uint_as_float(w[i])));
            } else {
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
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
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
    }
}

// dW (+)= sum over splits of the partial tiles, in split order (deterministic).
// Each thread owns float4 column blocks; up to 8 split loads are issued ahead
// of the (ordered) adds so the L2-resident partials stream at full rate.  <= 64
// registers: 4 CTAs per SM, so the C2 grid (576 CTAs) runs in one wave.
__global__ void __launch_bounds__(256, 4) splitk_reduce_kernel(const float4 *__restrict__ ws, float4 *__restrict__ dW,
                                                               int64_t n4, int nsplit, int accumulate, int trig,
                                                               float4 *__restrict__ mc, int mc_unicast) {
    if (trig) pdl_trigger();
    pdl_wait();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 a = accumulate ? dW[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s = 0; s < nsplit; s += 8) {  // up to 8 independent loads in flight, then ordered adds
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (s + u < nsplit) v[u] = __ldcs(ws + (size_t)(s + u) * n4 + i);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (s + u < nsplit) {
                    a.x += v[u].x; a.y += v[u].y; a.z += v[u].z; a.w += v[u].w;
                }
        }
        if (mc && mc_unicast) {  // test hook: the same reduction into a plain device address
            float *m = reinterpret_cast<float *>(mc + i);
            atomicAdd(m, a.x);
            atomicAdd(m + 1, a.y);
            atomicAdd(m + 2, a.z);
            atomicAdd(m + 3, a.w);
        } else if (mc)  // fused all-reduce: the split sum is added into the multicast dW (NVSwitch reduction)
            asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "f"(a.x),
                         "f"(a.y), "f"(a.z), "f"(a.w)
                         : "memory");
        else
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
    // The encoder is a driver-API call: it needs the device's context current in
    // this thread, which the runtime only makes current lazily.  A thread whose
    // first CUDA work is this call (e.g. PyTorch's autograd worker reusing cached
    // allocations) would get CUDA_ERROR_INVALID_CONTEXT; cudaSetDevice makes the
    // primary context current.
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaSetDevice(dev) != cudaSuccess) return cudaErrorInvalidDevice;
    CUresult r = fn(tm, dt, rank, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz(swizzle_bytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

struct Plan {
    int kr_blocks, nkr, nbslots, na, sa, nsplit, smem, chunk_steps;
    uint32_t a_col0, corr_col;
};

// sms: SMs the split-K grid may fill (the device's count at launch, kSplitSMs
// for the pure workspace query).
template <int KIND, int B>
static Plan plan_for(int64_t M, int64_t K, int64_t N, int sms) {
    using C = Cfg<KIND, B>;
    Plan pl{};
    const int nbc = (int)(K / B);
    // A ring: 64 KB of dY slabs per SM, 2..kMaxSA stages; the rest of shared memory
    // goes to the B ring (measured: with fp32 blocks the B ring's depth, not the A
    // ring's, bounds the main loop)
    // (FP32 grade: 2 stages, the B ring and its B_lo copy take the rest -- measured faster)
    // The stage count must be EVEN: the two A-mover groups take alternate steps, and
    // with an even count each group meets a stage on consecutive mbarrier phases
    // (an odd count lets a group's parity wait pass on a phase two behind).
    pl.sa = C::X3 ? 2 : std::max(2, std::min(kMaxSA, 65536 / C::SLAB)) & ~1;
    // B ring (FP32 grade: plus its B_lo copy of the same size)
    const int ring = (kSmemBudget - kFixedSmem - pl.sa * C::SLAB) / C::ACC_MULT;
    // largest kcol range whose accumulator(s) leave room for two A buffers in the
    // 512 TMEM columns and whose densest step (R block rows, every block, G rounded)
    // fits the B ring; <= 56 blocks keeps a run word's column in 10 bits
    int maxb = std::min(std::min((512 - 2 * C::A_STEP) / (B * C::ACC_MULT), 56), nbc);
    auto need_of = [](int blocks) { return (blocks + C::G - 1) / C::G * C::G; };
    while (maxb > 1 && C::R * need_of(maxb) * C::BLOCK_BYTES > ring) --maxb;
    pl.nkr = (nbc + maxb - 1) / maxb;
    pl.kr_blocks = (nbc + pl.nkr - 1) / pl.nkr;
    pl.corr_col = (uint32_t)(pl.kr_blocks * B);
    pl.na = std::min(kMaxA, (512 - C::ACC_MULT * pl.kr_blocks * B) / C::A_STEP);
    pl.a_col0 = (uint32_t)(512 - pl.na * C::A_STEP);
    pl.nbslots = std::min(4095, ring / C::BLOCK_BYTES);
    pl.smem = pl.sa * C::SLAB + C::ACC_MULT * pl.nbslots * C::BLOCK_BYTES + kFixedSmem;
    // a chunk's stored blocks (all columns) fit the colidx / run-word buffers
    pl.chunk_steps = std::min(kStepCap, kColCap / (C::R * nbc));
    const int64_t tiles = (N / 128) * pl.nkr;
    const int64_t nst = (M / B + C::R - 1) / C::R;
    const int64_t cap = std::min<int64_t>(sms, kSplitSMs);
    int64_t ns = std::max<int64_t>(1, cap / std::max<int64_t>(1, tiles));
    if (C::X3) {  // chain cap: at most kX3ChainRows rows of MMAs per TMEM accumulator
        const int64_t steps_cap = std::max<int64_t>(1, kX3ChainRows / C::SROWS);
        ns = std::max<int64_t>(ns, (nst + steps_cap - 1) / steps_cap);
    }
    pl.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>({nst, ns, (int64_t)kMaxSplits}));
    return pl;
}

template <int KIND, int B>
static cudaError_t launch_t(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnzb,
                            int64_t M, int64_t K, const void *dY, int64_t N, float *dW, int accumulate,
                            float *ws, cudaStream_t stream, float *mc, int nk, int mc_unicast) {
    using C = Cfg<KIND, B>;
    int dev = 0, sms = kSplitSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const Plan pl = plan_for<KIND, B>(M, K, N, sms);
    if (pl.chunk_steps < 1) return cudaErrorNotSupported;  // K / b too large for the chunk buffers
    if (nk && (pl.nsplit < 2 || mc)) return cudaErrorNotSupported;  // dW^T only through the split-K reduce
    const CUtensorMapDataType dt = KIND == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    // dY (N x M, row-major): one box = the SROWS x 128 slab of a step, row-major
    // in shared memory (no swizzle: the A movers read it column-wise)
    CUtensorMap tm_dy, tm_val;
    const cuuint64_t dy_dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    const cuuint64_t dy_str[1] = {(cuuint64_t)N * C::ES};
    const cuuint32_t dy_box[2] = {128, (cuuint32_t)C::SROWS};
    cudaError_t e = make_map(&tm_dy, dY, dt, 2, dy_dims, dy_str, dy_box, 0);
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
    p.values = static_cast<const uint8_t *>(values);
    p.dW = dW;
    p.nbr = M / B;
    p.N = N;
    p.K = K;
    p.nkr = pl.nkr;
    p.nsplit = pl.nsplit;
    p.kr_blocks = pl.kr_blocks;
    p.nbslots = pl.nbslots;
    p.na = pl.na;
    p.sa = pl.sa;
    p.a_col0 = pl.a_col0;
    p.corr_col = pl.corr_col;
    p.chunk_steps = pl.chunk_steps;
    p.ws = ws;
    p.mc = mc;
    p.mc_unicast = mc_unicast;
    p.mode = pl.nsplit > 1 ? 3 : mc ? 4 : accumulate ? 1 : 0;
    p.pdl_trig = (pdl_flags() & 2) ? 1 : (pdl_flags() & 4) ? 2 : 0;
    auto kern = wgrad_tc_kernel<KIND, B>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((N / 128) * pl.nkr * pl.nsplit);
    e = launch_pdl(pdl_flags() & 16, kern, dim3(grid), dim3(C::THREADS), (size_t)pl.smem, stream, tm_dy, tm_val, tm_dw, tm_ws, p);
    if (e != cudaSuccess) return e;
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess || pl.nsplit == 1) return e;
    if (nk) return launch_transpose_reduce(ws, dW, K, N, pl.nsplit, accumulate, stream);
    const int64_t n4 = K * N / 4;
    const unsigned rgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, (int64_t)sms * 4));
    e = launch_pdl(pdl_flags() & 32, splitk_reduce_kernel, dim3(rgrid), dim3(256), 0, stream, reinterpret_cast<const float4 *>(ws),
                   reinterpret_cast<float4 *>(dW), n4, (int)pl.nsplit, mc ? 0 : accumulate, (pdl_flags() & 8) ? 1 : 0,
                   reinterpret_cast<float4 *>(mc), mc_unicast);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

// dW^T (N x K, row-major: PyTorch's Linear.weight.grad layout; BSR_DW_NK) (+)=
// the sum over splits of K x N partial tiles, in split order -- the same adds as
// splitk_reduce_kernel, stored transposed through a 32 x 32 shared-memory tile
// (reads coalesced along N, writes along K).
__global__ void __launch_bounds__(256) transpose_reduce_kernel(const float *__restrict__ ws, float *__restrict__ dWt,
                                                               int64_t K, int64_t N, int nsplit, int accumulate) {
    __shared__ float tile[32][33];
    pdl_wait();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    const int64_t ntn = (N + 31) / 32, ntiles = ntn * ((K + 31) / 32);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t k0 = (t / ntn) * 32, n0 = (t % ntn) * 32;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t k = k0 + ty + 8 * r, n = n0 + tx;
            float a = 0.f;
            if (k < K && n < N) {
                if (accumulate) a = dWt[n * K + k];
                for (int s = 0; s < nsplit; ++s) a += __ldcs(ws + ((int64_t)s * K + k) * N + n);
            }
            tile[ty + 8 * r][tx] = a;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int64_t n = n0 + ty + 8 * r, k = k0 + tx;
            if (k < K && n < N) dWt[n * K + k] = tile[tx][ty + 8 * r];
        }
        __syncthreads();
    }
}

}  // namespace tc

cudaError_t launch_splitk_reduce(const float *ws, float *dW, int64_t n, int nsplit, int accumulate, cudaStream_t stream) {
    int dev = 0, sms = tc::kSplitSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n4 = n / 4;
    const unsigned rgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, (int64_t)sms * 4));
    cudaError_t e = launch_pdl(pdl_flags() & 32, tc::splitk_reduce_kernel, dim3(rgrid), dim3(256), 0, stream,
                               reinterpret_cast<const float4 *>(ws), reinterpret_cast<float4 *>(dW), n4, nsplit,
                               accumulate, (pdl_flags() & 8) ? 1 : 0, static_cast<float4 *>(nullptr), 0);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_transpose_reduce(const float *ws, float *dWt, int64_t K, int64_t N, int nsplit, int accumulate,
                                    cudaStream_t stream) {
    int dev = 0, sms = tc::kSplitSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = ((N + 31) / 32) * ((K + 31) / 32);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * 8));
    cudaError_t e = launch_pdl(pdl_flags() & 32, tc::transpose_reduce_kernel, dim3(grid), dim3(256), 0, stream, ws, dWt, K,
                               N, nsplit, accumulate);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

// FP32 grade per-run plan with more than one split: its split-K reduce can store
// dW^T directly (bsr_wgrad_nk's native path).
bool wgrad_x3_native_nk(int64_t M, int64_t K, int b, int64_t N) {
    tc::Plan pl{};
    if (b == 32) pl = tc::plan_for<2, 32>(M, K, N, tc::kSplitSMs);
    else if (b == 64) pl = tc::plan_for<2, 64>(M, K, N, tc::kSplitSMs);
    else return false;
    return pl.nsplit > 1 && pl.chunk_steps >= 1;
}

static size_t wgrad_runs_ws_bytes(int64_t M, int64_t K, int b, int64_t N) {
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

size_t wgrad_tc_ws_bytes(int64_t M, int64_t K, int b, int64_t N) {
    return std::max(wgrad_runs_ws_bytes(M, K, b, N), wgrad_span_ws_bytes(M, K, b, N));
}

// FP32 grade: the chain cap (kX3ChainRows) sets a floor on the splits.  The
// plan's split count does not depend on the device's SM count beyond 148.
size_t wgrad_x3_ws_bytes(int64_t M, int64_t K, int b, int64_t N) {
    tc::Plan pl{};
    if (b == 32) pl = tc::plan_for<2, 32>(M, K, N, tc::kSplitSMs);
    else if (b == 64) pl = tc::plan_for<2, 64>(M, K, N, tc::kSplitSMs);
    else return 0;
    return pl.nsplit > 1 ? (size_t)pl.nsplit * K * N * sizeof(float) : 0;
}

// Kernel choice (measured): the per-run kernel, except with many
// block columns (K / b >= 64: S12 fc2 at b = 16, B24 fc2 at b = 32), where it
// splits the kcols into several TMEM ranges that each re-read dY and issues one
// MMA per short run, while the span kernel's CTA pairs and dense-padded
// N <= 256 MMAs win (S12 fc2 bf16 b=16: 124 vs 200 us; B24 fc2 b=32: 2.38 vs
// 3.92 ms f32/tf32, 1.45 vs 2.91 ms bf16).  The FP32 grade exists in the per-run
// kernel only.
static bool use_runs_kernel(int kind, int algo, int b, int64_t K) {
    if (kind == 2) return true;
    if (algo == 1) return true;
    if (algo == 2) return false;
    if (kind == 0 && b == 16) return false;  // tf32 b = 16: only the span kernel pairs blocks into 128-byte rows
    return K / b < 64;
}

bool wgrad_tc_supported(int kind, int algo, int b, int64_t K, int64_t N) {
    if (N % 128 != 0 || b < 16 || b > 64) return false;
    if (kind == 2) {
        if (algo != 0 && algo != 1) return false;
        if (b == 32) return tc::plan_for<2, 32>(128, K, N, tc::kSplitSMs).chunk_steps >= 1;
        if (b == 64) return tc::plan_for<2, 64>(128, K, N, tc::kSplitSMs).chunk_steps >= 1;
        return false;
    }
    if (use_runs_kernel(kind, algo, b, K)) return !(kind == 0 && b == 16);
    return true;
}

cudaError_t launch_wgrad_tc(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnzb,
                            int kind, int algo, int64_t M, int64_t K, int b, const void *dY, int64_t N, float *dW,
                            int accumulate, void *ws, cudaStream_t stream, float *mc, int nk, int mc_unicast) {
    if ((mc || nk) && !use_runs_kernel(kind, algo, b, K)) return cudaErrorNotSupported;  // per-run kernel only
    if (!use_runs_kernel(kind, algo, b, K))
        return launch_wgrad_span(rowptr, colidx, values, nnzb, kind, M, K, b, dY, N, dW, accumulate, ws, stream);
    if (!values || nnzb == 0) {  // no stored block: dW = 0 (or unchanged; nothing to add into the multicast dW)
        if (nk) return cudaErrorNotSupported;
        return accumulate || mc ? cudaSuccess : cudaMemsetAsync(dW, 0, (size_t)K * N * sizeof(float), stream);
    }
#define TC_CASE(KD, B_) \
    if (kind == KD && b == B_) return tc::launch_t<KD, B_>(rowptr, colidx, values, nnzb, M, K, dY, N, dW, accumulate, \
                                                            static_cast<float *>(ws), stream, mc, nk, mc_unicast);
    TC_CASE(0, 32) TC_CASE(0, 64) TC_CASE(1, 16) TC_CASE(1, 32) TC_CASE(1, 64) TC_CASE(2, 32) TC_CASE(2, 64)
#undef TC_CASE
    return cudaErrorInvalidValue;
}

}  // namespace bsrp
