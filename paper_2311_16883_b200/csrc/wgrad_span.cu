// wgrad_span.cu -- BSR weight gradient on tcgen05 tensor cores with dense-padded
// row spans (row a6 of SURVEY §8a; BJ "TMA-fed tcgen05/TMEM
// block-sparse GEMM that walks BSR rows and skips pruned blocks").
//
//   dW[J*b + c][n] = sum over stored blocks (I, J), sum over r < b of
//                    values(I,J)[r][c] * dY[I*b + r][n]
//
// Orientation: D = dW^T tile-wise, D[n][kcol] += A[n][r] * B[r][kcol], with
//   A = the 128-column (per CTA) x b-row slab of dY of block row I and
//   B = the stored X blocks of that block row,
// both MN-major exactly as they sit in HBM (dY row-major, blocks row-major),
// both staged in shared memory by TMA.  TMEM holds D: 128 lanes = 128 columns
// n of dY, one TMEM column per kcol of the CTA's kcol range (<= 512).
//
// Why spans: one tcgen05.mma with M = 128 costs max(~71, N/2) SM cycles
// (DESIGN.md §10), so one MMA per run of adjacent kept blocks (N = 32..96 at
// keep 0.5) spends most of the tensor pipe on the fixed cost.  Here each block
// row's kcol range is cut into at most two chunks of <= 256 columns; within a
// chunk the MMA spans from the first to the last kept block, and the pruned
// blocks inside that span are ZERO-FILLED in shared memory by an out-of-bounds
// TMA box (no HBM or L2 traffic).  Chunks and block rows without a kept block
// in the CTA's range are skipped entirely (no dY read, no MMA): at keep 0.5
// the span MMAs cost ~1.05x the dense tensor time, at keep 0.1 most rows issue
// one narrow MMA or none.
//
// CG = 2 runs the MMA on a CTA pair (tcgen05 cta_group::2, M = 256: the pair
// covers 256 columns n).  Each CTA loads its own 128-column dY slab and HALF
// of each span's X blocks (spans are padded to an even block count), so the
// X blocks -- re-read once per n tile -- cost half the L2->SM traffic.
//
// Roles (256 threads): warp 0 = producer (plans 32 block rows per pass from
// rowptr/colidx, one lane issues the TMAs), warp 1 = MMA issuer (leader CTA
// only), warp 2 = TMEM allocator, warps 4-7 = TMEM zeroing, then the epilogue
// (tcgen05.ld -> coalesced fp32 stores of dW, dW +=, or a split-K partial).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "launch.h"

namespace bsrp {
namespace span {

constexpr int kThreads = 256;
constexpr int kMaxStages = 8;
constexpr int kSmemBudget = 227 * 1024;
constexpr int kBarBytes = 512;   // barriers, TMEM slot, stage meta, plan counts
constexpr int kColCap = 2048;    // colidx entries of one plan group staged in shared memory
constexpr int kFixedSmem = 1024 /*align*/ + kBarBytes + 2 * 32 * 16 /*plan*/ + 36 * 4 + 2 * kColCap;
constexpr int kSplitSMs = 148;
constexpr uint32_t kSentinel = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void dbg_timeout(uint32_t, uint32_t, uint32_t) {}
// Bounded wait: a pipeline bug traps (launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity, uint32_t what = 0, uint32_t info = 0) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins > (1u << 26)) {
            dbg_timeout(what, parity, info);
            __trap();
        }
    }
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        __nanosleep(128);
        if (++spins > (1u << 24)) {
            dbg_timeout(9, parity, 0);
            __trap();
        }
    }
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// TMA loads.  CG = 2: the .cta_group::2 form signals the LEADER CTA's mbarrier
// (the peer bit of the barrier address cleared), which expects both CTAs' bytes.

// The same loads issued by one elected lane of a converged warp whose operands are
// warp-uniform (no per-lane address waterfall in front of the UTMALDG).
template <int CG>
__device__ __forceinline__ void tma_3d_e(const CUtensorMap *tm, uint32_t bar, uint32_t dst, int x, int y, int z) {
    if constexpr (CG == 2)
        asm volatile(
            "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
            "@p cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n}\n" ::"r"(
                dst),
            "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(bar & 0xFEFFFFFFu)
            : "memory");
    else
        asm volatile(
            "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
            "@p cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n}\n" ::"r"(
                dst),
            "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(bar)
            : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_e(uint64_t *bar, uint32_t bytes) {
    asm volatile(
        "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
        "r"(bytes)
        : "memory");
}
__device__ __forceinline__ uint32_t uni(uint32_t x) { return __reduce_or_sync(0xffffffffu, x); }

// tcgen05.mma, both operands from shared memory, accumulate into TMEM; one
// elected lane of the (converged) issuing warp.
template <int KIND, int CG>
__device__ __forceinline__ void mma_ss(uint32_t d, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                                       uint32_t idesc) {
#define BSRP_SS(CGS, KS)                                                                                        \
    asm volatile("{\n.reg .pred p;\n.reg .b64 a, b;\nmov.b64 a, {%1, %2};\nmov.b64 b, {%3, %4};\n"          \
                 "elect.sync _|p, 0xffffffff;\n"                                                              \
                 "@p tcgen05.mma.cta_group::" CGS ".kind::" KS " [%0], a, b, %5, 1;\n}\n" ::"r"(d),          \
                 "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc))
    if constexpr (CG == 2) {
        if constexpr (KIND == 1) BSRP_SS("2", "f16"); else BSRP_SS("2", "tf32");
    } else {
        if constexpr (KIND == 1) BSRP_SS("1", "f16"); else BSRP_SS("1", "tf32");
    }
#undef BSRP_SS
}
// MMA completion -> mbarrier arrive (CG = 2: on both CTAs of the pair).
template <int CG>
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    if constexpr (CG == 2)
        asm volatile(
            "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
            "@p tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
                smem_u32(bar)),
            "h"((uint16_t)3)
            : "memory");
    else
        asm volatile(
            "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
            "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
            : "memory");
}

// UMMA shared-memory descriptor: start, LBO (stride between MN atoms), SBO
// (stride between K groups), version 1, layout type.
__host__ __device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

// Instruction descriptor: fp32 accumulate, A/B format (1 = bf16, 2 = tf32), A and
// B MN-major, M = 128 * CG, N = n.
template <int KIND, int CG>
__host__ __device__ __forceinline__ uint32_t instr_desc(uint32_t n) {
    constexpr uint32_t fmt = KIND == 1 ? 1u : 2u;
    return (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 15) | (1u << 16) | ((n >> 3) << 17) |
           ((128u * CG >> 4) << 24);
}

template <int KIND, int B>
struct Cfg {
    static constexpr int ES = KIND == 1 ? 2 : 4;
    static constexpr bool TF32 = KIND == 0;
    static constexpr int UK = KIND == 1 ? 16 : 8;  // MMA K per instruction
    static constexpr int KGROUP = TF32 ? 4 : 8;     // K rows per swizzle group
    // A = dY slab, 128 columns n x B rows, MN-major in 128-byte swizzle atoms
    // (32 tf32 / 64 bf16 columns per atom; tf32 uses the 32-byte-atomicity form).
    static constexpr int ATOM_E = 128 / ES;
    static constexpr int A_ATOMS = 128 / ATOM_E;
    static constexpr int SLAB = 128 * B * ES;
    static constexpr int A_LBO = B * 128;
    static constexpr int A_SBO = KGROUP * 128;
    static constexpr int A_KSTEP = UK * 128;
    static constexpr uint32_t A_LAYOUT = TF32 ? 1u : 2u;  // SW128_32B / SW128
    // B = X blocks, each [atom][B rows][BW bytes]; blocks BLOCK_BYTES apart.
    // PAIR (tf32, b = 16: 64-byte block rows): MN-major tf32 operands exist only in
    // 128-byte swizzle rows, so two adjacent blocks of a span share one atom
    // [B rows][128 B] (left / right half); the loaders place them there.
    static constexpr bool PAIR = TF32 && B * ES == 64;
    static constexpr int BW = PAIR ? 128 : (B * ES < 128) ? B * ES : 128;
    static constexpr int B_ATOMS = PAIR ? 1 : B * ES / BW;
    static constexpr int BLOCK_BYTES = B * B * ES;
    static constexpr int GRAN = PAIR ? 2 : 1;  // blocks per span granule (times CG)
    static constexpr int B_LBO = B * BW;
    static constexpr int B_SBO = KGROUP * BW;
    static constexpr int B_KSTEP = UK * BW;
    static constexpr uint32_t B_LAYOUT = TF32 ? 1u : BW == 128 ? 2u : BW == 64 ? 4u : 6u;
    static_assert(!TF32 || B * ES >= 64, "tf32 MN-major operands need 128-byte rows (b >= 16, blocks paired)");
    static constexpr int MAXCB = 256 / B;  // blocks per MMA (N <= 256)
    static constexpr int MAXJ = 512 / B;   // blocks per kcol range (TMEM columns)
};

struct Params {
    const int32_t *rowptr, *colidx;
    const uint8_t *values;
    float *out;          // dW (mode 0 / 1) or the split-K workspace (mode 3)
    int64_t nbr, N, K, nnzb;
    int nkr, kr_blocks, nsplit, nchunk, cb, stages, mode;
    uint32_t stage_bytes;
};

// MMA spans of one block row (warp-uniform): per chunk of cb blocks, the range
// from the first to the last kept block, padded to an even block count when a
// CTA pair splits it (each CTA holds len/2 blocks).
struct Spans {
    uint32_t w[2];  // MMA word per chunk: 1 << 31 | len << 16 | first TMEM column (0: no MMA)
    int f[2], len[2];
};
template <int B, int CG, int GRAN = 1>
__device__ __forceinline__ Spans row_spans(uint32_t mk, int nchunk, int cb) {
    Spans sp;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        sp.w[c] = 0u;
        sp.f[c] = 0;
        sp.len[c] = 0;
        if (c >= nchunk) continue;
        const uint32_t cm = (mk >> (c * cb)) & ((cb >= 32) ? 0xffffffffu : ((1u << cb) - 1u));
        if (!cm) continue;
        int f = __ffs(cm) - 1;
        int len = 32 - __clz(cm) - f;
        while (len % (GRAN * CG)) {  // whole granules: each CTA holds len/CG blocks, paired for tf32 b = 16
            if (f + len < cb) {
                ++len;
            } else {
                --f;
                ++len;
            }
        }
        sp.f[c] = f;
        sp.len[c] = len;
        sp.w[c] = (1u << 31) | ((uint32_t)len << 16) | (uint32_t)((c * cb + f) * B);
    }
    return sp;
}

// Byte offset of element byte `o` (row-major b x b block) in the TMA/UMMA
// shared-memory image of the block: [atom][row][BW bytes], then the layout's
// XOR swizzle (applied to the offset; blocks are aligned to the swizzle period).
template <int KIND, int B>
__device__ __forceinline__ uint32_t block_smem_off(uint32_t o) {
    constexpr int ES = KIND == 1 ? 2 : 4;
    constexpr uint32_t ROW = B * ES, BW = ROW < 128 ? ROW : 128;
    const uint32_t r = o / ROW, cbyte = o % ROW;
    const uint32_t L = (cbyte / BW) * (B * BW) + r * BW + cbyte % BW;
    if constexpr (KIND == 0) return L ^ (((L >> 7) & 3u) << 5);       // 128B swizzle, 32-byte atomicity
    else if constexpr (BW == 128) return L ^ (((L >> 7) & 7u) << 4);  // 128B swizzle
    else if constexpr (BW == 64) return L ^ (((L >> 7) & 3u) << 4);   // 64B swizzle
    else return L ^ (((L >> 7) & 1u) << 4);                           // 32B swizzle
}

template <int KIND, int B, int CG>
__global__ void __launch_bounds__(kThreads, 1)
    wgrad_span_kernel(const __grid_constant__ CUtensorMap tm_dy, Params p) {
    using C = Cfg<KIND, B>;
    // full-barrier arrivals per phase: the producer (+ dY bytes), the 128 loader threads'
    // cp.async completions, and for a pair the peer's relay
    constexpr uint32_t kFullArrivals = 1 + 128 + (CG == 2 ? 1 : 0);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = p.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
    uint64_t *empty = full + kMaxStages;
    uint64_t *accfull = empty + kMaxStages;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(accfull + 1);
    uint2 *s_meta = reinterpret_cast<uint2 *>(s_tmem + 2);  // [kMaxStages] per-chunk MMA words
    uint64_t *plan_full = reinterpret_cast<uint64_t *>(s_meta + kMaxStages);  // [2]
    uint64_t *plan_empty = plan_full + 2;                                      // [2]
    uint32_t *s_cnt = reinterpret_cast<uint32_t *>(plan_empty + 2);            // [2] records per plan group
    uint64_t *xfull = reinterpret_cast<uint64_t *>(s_cnt + 2);                  // [kMaxStages] peer: loaders done
    uint4 *s_plan = reinterpret_cast<uint4 *>(smem + (size_t)S * p.stage_bytes + kBarBytes);  // [2][32]
    int32_t *s_rp = reinterpret_cast<int32_t *>(s_plan + 2 * 32);                // [33]
    uint16_t *s_col = reinterpret_cast<uint16_t *>(s_rp + 36);                  // [kColCap]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
    int t = blockIdx.x / CG;
    const int ntp = (int)(p.N / (128 * CG));
    const int nt = t % ntp;
    t /= ntp;
    const int kr = t % p.nkr;
    const int split = t / p.nkr;
    const int n0 = (nt * CG + (int)rank) * 128;
    const int nbc = (int)(p.K / B);
    const int J0 = kr * p.kr_blocks;
    const int nbJ = min(p.kr_blocks, nbc - J0);
    const int64_t Ib = (int64_t)split * p.nbr / p.nsplit, Ie = (int64_t)(split + 1) * p.nbr / p.nsplit;

    if (warp == 1 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_dy)) : "memory");
        for (int i = 0; i < 2; ++i) {
            mbar_init(plan_full + i, 1);
            mbar_init(plan_empty + i, CG == 2 && rank != 0 ? 6 : 5);  // producer, 4 loader warps (+ peer relay)
        }
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, kFullArrivals);  // producer (+ dY TMA bytes), loader threads, peer relay
            mbar_init(xfull + s, 128);           // peer CTA: its loader threads' cp.async completions
            mbar_init(empty + s, 1);  // one MMA commit
        }
        mbar_init(accfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        if constexpr (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                         "r"(512u)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                         "r"(512u)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_tmem;
    if (warp >= 4) {  // zero the accumulator (the span MMAs always accumulate)
        const uint32_t lb = (uint32_t)((warp - 4) * 32) << 16;
        const uint32_t z = 0;
        for (int c = 0; c < 512; c += 16) {
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                    tmem + lb + (uint32_t)c),
                "r"(z)
                : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();

    const uint32_t smem0 = smem_u32(smem);
    if (warp == 3) {
        // ------------------------------------------------ planner
        // Groups of up to 32 block rows: rowptr and the group's colidx range are
        // staged in shared memory with coalesced loads, then lane i derives block
        // row i's kept-block mask over [J0, J0 + nbJ) and the value index of its
        // first kept block there; rows with a kept block are compacted into a plan
        // record (double-buffered, one group ahead of the producer).
        const int gr = min(32, kColCap / nbc);
        int g = 0;
        for (int64_t I0 = Ib;; I0 += gr, ++g) {
            const int buf = g & 1;
            const int nr = (int)min((int64_t)gr, Ie - I0);
            uint32_t mask = 0, base = 0;
            if (nr > 0) {
                for (int i = lane; i <= nr; i += 32) s_rp[i] = __ldg(p.rowptr + I0 + i);
                __syncwarp();
                const int b0 = s_rp[0], total = s_rp[nr] - b0;
                for (int e = lane; e < total; e += 32) s_col[e] = (uint16_t)__ldg(p.colidx + b0 + e);
                __syncwarp();
                if (lane < nr) {
                    int lo = s_rp[lane] - b0, hi = s_rp[lane + 1] - b0;
                    const int z = hi;
                    while (lo < hi) {  // first stored block with J >= J0
                        const int mid = (lo + hi) >> 1;
                        if ((int)s_col[mid] < J0) lo = mid + 1; else hi = mid;
                    }
                    base = (uint32_t)(b0 + lo);
                    for (int e = lo; e < z; ++e) {
                        const int J = (int)s_col[e] - J0;
                        if (J >= nbJ) break;
                        mask |= 1u << J;
                    }
                }
            }
            const uint32_t rows = __ballot_sync(0xffffffffu, mask != 0);
            // Warm L2 one plan group ahead of the producer: this CTA's dY slabs of the
            // group's rows (tensor-map prefetch) and the group's stored blocks (shared
            // by every n tile of these rows: one CTA pair pulls them from HBM).
            {
                if (mask)
                    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                                     reinterpret_cast<uint64_t>(&tm_dy)),
                                 "r"(0), "r"((int)((I0 + lane) * B)), "r"(n0 / C::ATOM_E)
                                 : "memory");
                if (nr > 0 && nt == 0) {
                    const int64_t v0 = (int64_t)s_rp[0] * C::BLOCK_BYTES, vb = (int64_t)(s_rp[nr] - s_rp[0]) * C::BLOCK_BYTES;
                    for (int64_t o = (int64_t)lane * 16384; o < vb; o += 32 * 16384)
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.values + v0 + o),
                                     "r"((uint32_t)min((int64_t)16384, vb - o))
                                     : "memory");
                }
            }
            if (lane == 0) mbar_wait_sleep(plan_empty + buf, ((g >> 1) & 1) ^ 1);
            __syncwarp();
            if (mask) s_plan[buf * 32 + __popc(rows & ((1u << lane) - 1u))] =
                make_uint4((uint32_t)(I0 + lane), mask, base, 0u);
            if (lane == 0) s_cnt[buf] = nr > 0 ? (uint32_t)__popc(rows) : kSentinel;
            __syncwarp();
            if (lane == 0) mbar_arrive(plan_full + buf);
            if (nr <= 0) break;
            __syncwarp();
        }
    } else if (warp == 0) {
        // ------------------------------------------------ producer
        // Whole warp, warp-uniform operands (REDUX copies), one elected lane issues.
        // Per block row: the dY slab (one 3-D box) and, per chunk, this CTA's half
        // of the span as maximal segments of consecutive stored blocks (consecutive
        // in BSR storage) or of pruned blocks (out-of-bounds: zeros), each cut into
        // boxes of 8/4/2/1 blocks.
        int stage = 0;
        uint32_t phase = 0;
        const int cb = p.cb;
        for (int g = 0;; ++g) {
            const int buf = g & 1;
            mbar_wait(plan_full + buf, (g >> 1) & 1);
            const uint32_t cnt = uni(s_cnt[buf]);
            if (cnt == kSentinel) break;
            for (uint32_t r = 0; r < cnt; ++r) {
                const uint4 rec = s_plan[buf * 32 + r];
                const uint32_t mk = uni(rec.y);
                const int bs = (int)uni(rec.z);
                const int row = (int)uni(rec.x);
                const Spans sp = row_spans<B, CG, C::GRAN>(mk, p.nchunk, cb);
                uint32_t bytes = (uint32_t)(CG * C::SLAB);
                (void)bs;
                mbar_wait(empty + stage, phase ^ 1u, 1, (uint32_t)stage | ((uint32_t)row << 8));
                const uint32_t sb = smem0 + (uint32_t)stage * p.stage_bytes;
                const uint32_t fb = smem_u32(full + stage);
                s_meta[stage] = make_uint2(sp.w[0], sp.w[1]);  // every lane stores the same words
                __syncwarp();
                if (rank == 0) mbar_arrive_expect_tx_e(full + stage, bytes);
                tma_3d_e<CG>(&tm_dy, fb, sb, 0, row * B, n0 / C::ATOM_E);
                __syncwarp();
                if (++stage == S) { stage = 0; phase ^= 1u; }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(plan_empty + buf);
        }
        if (lane == 0) {
        }
        if (rank == 0) {  // end of the sequence
            mbar_wait(empty + stage, phase ^ 1u, 2, (uint32_t)stage);
            s_meta[stage] = make_uint2(kSentinel, kSentinel);
            __syncwarp();
            if (lane == 0)  // stands in for every arrival of the phase (the loaders are done)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + stage)),
                             "r"(kFullArrivals)
                             : "memory");
        }
    } else if (warp == 1) {
        if (rank == 0) {
            // ------------------------------------------------ MMA issuer
            const uint64_t ad = smem_desc(smem0, C::A_LBO, C::A_SBO, C::A_LAYOUT);
            const uint64_t bd = smem_desc(smem0 + C::SLAB, C::B_LBO, C::B_SBO, C::B_LAYOUT);
            const uint32_t a_hi = (uint32_t)(ad >> 32), b_hi = (uint32_t)(bd >> 32);
            const uint32_t a_lo0 = (uint32_t)ad, b_lo0 = (uint32_t)bd;
            const uint32_t idesc0 = instr_desc<KIND, CG>(0u);
            const uint32_t cbb16 = (uint32_t)(p.cb / CG * C::BLOCK_BYTES) >> 4;
            int stage = 0;
            uint32_t phase = 0, nmma_dbg = 0;
            long long t_full = 0, t_iss = 0;
            (void)t_full; (void)t_iss;
            for (;;) {
                mbar_wait(full + stage, phase, 3, (uint32_t)stage | (nmma_dbg << 8));
                const uint2 m = s_meta[stage];
                if (m.x == kSentinel) break;
                tc_fence_after();
                const uint32_t so = ((uint32_t)stage * p.stage_bytes) >> 4;
#pragma unroll
                for (int k = 0; k < B / C::UK; ++k) {
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const uint32_t wc = c == 0 ? m.x : m.y;
                        if (!wc) continue;
                        const uint32_t ncol = ((wc >> 16) & 0x7FFFu) * (uint32_t)B;
                        mma_ss<KIND, CG>(tmem + (wc & 0xFFFFu), a_lo0 + so + (uint32_t)k * (C::A_KSTEP >> 4), a_hi,
                                         b_lo0 + so + (uint32_t)c * cbb16 + (uint32_t)k * (C::B_KSTEP >> 4), b_hi,
                                         idesc0 | ((ncol >> 3) << 17));
                    }
                }
                ++nmma_dbg;
                __syncwarp();
                mma_commit<CG>(empty + stage);  // frees the stage in both CTAs once these MMAs complete
                __syncwarp();
                if (++stage == S) { stage = 0; phase ^= 1u; }
            }
            __syncwarp();
            if (lane == 0) {
            }
            mma_commit<CG>(accfull);
        }
    } else if (CG == 2 && warp == 2 && rank != 0) {
        // ------------------------------------------------ peer relay
        // cp.async completions can only arrive on a CTA-local barrier: once the
        // peer's loaders' copies of a row have landed (xfull), one arrival on the
        // leader's full barrier of that stage, over the cluster.
        uint32_t full_leader = smem_u32(full);
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(full_leader) : "r"(full_leader));
        int stage = 0;
        uint32_t phase = 0;
        for (int g = 0;; ++g) {
            const int buf = g & 1;
            mbar_wait_sleep(plan_full + buf, (g >> 1) & 1);
            const uint32_t cnt = s_cnt[buf];
            if (cnt == kSentinel) break;
            for (uint32_t r = 0; r < cnt; ++r) {
                mbar_wait(xfull + stage, phase, 5, (uint32_t)stage);
                if (lane == 0)
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                     full_leader + (uint32_t)stage * 8u)
                                 : "memory");
                __syncwarp();
                if (++stage == S) { stage = 0; phase ^= 1u; }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(plan_empty + buf);
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ X-block loaders (then the epilogue)
        // The same plan sequence as the producer.  Each block row's share of its
        // spans is copied global -> shared with 16-byte cp.async (pruned blocks:
        // src-size 0, i.e. zero fill) straight into the swizzled UMMA image, on
        // the LSU path, while the TMA engine streams dY.  Every loader thread then
        // arms cp.async.mbarrier.arrive on the stage's full barrier (the peer CTA:
        // on its local xfull barrier, relayed to the leader by warp 2), so the
        // barrier completes when the copies land -- no waiting here.
        {
            constexpr int PPB = C::BLOCK_BYTES / 16;  // 16-byte pieces per block
            const int tid = threadIdx.x - 128;
            const int cb = p.cb, cbh = p.cb / CG;
            int stage = 0;
            uint32_t phase = 0;
            uint64_t *arrive_bar = (CG == 2 && rank != 0) ? xfull : full;
            for (int g = 0;; ++g) {
                const int buf = g & 1;
                mbar_wait_sleep(plan_full + buf, (g >> 1) & 1);
                const uint32_t cnt = s_cnt[buf];
                if (cnt == kSentinel) break;
                for (uint32_t r = 0; r < cnt; ++r) {
                    const uint4 rec = s_plan[buf * 32 + r];
                    const uint32_t mk = rec.y;
                    const int bs = (int)rec.z;
                    const Spans sp = row_spans<B, CG, C::GRAN>(mk, p.nchunk, cb);
                    mbar_wait(empty + stage, phase ^ 1u, 4, (uint32_t)stage);
                    const uint32_t xb = smem0 + (uint32_t)stage * p.stage_bytes + C::SLAB;
                    const int h0 = sp.len[0] / CG, h1 = sp.len[1] / CG;
                    const int total = (h0 + h1) * PPB;
                    for (int q = tid; q < total; q += 128) {
                        const int blk = q / PPB, off = q % PPB;
                        const int c = blk >= h0;
                        const int j = blk - (c ? h0 : 0);
                        const int J = c * cb + sp.f[c] + (int)rank * (c ? h1 : h0) + j;
                        const bool kept = J < nbJ && ((mk >> J) & 1u);
                        const int idx = kept ? bs + __popc(mk & ((1u << J) - 1u)) : 0;
                        const uint8_t *src = p.values + (int64_t)idx * C::BLOCK_BYTES + off * 16;
                        uint32_t dst;
                        if constexpr (C::PAIR) {  // block j: half (j & 1) of atom j / 2, 64-byte block rows
                            const uint32_t o = (uint32_t)off * 16u, L = (uint32_t)(j >> 1) * (B * 128u) +
                                                                         (o / 64u) * 128u + (uint32_t)(j & 1) * 64u + o % 64u;
                            dst = xb + (uint32_t)(c * cbh * C::BLOCK_BYTES) + (L ^ (((L >> 7) & 3u) << 5));
                        } else {
                            dst = xb + (uint32_t)((c * cbh + j) * C::BLOCK_BYTES) +
                                  block_smem_off<KIND, B>((uint32_t)off * 16u);
                        }
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                                     "r"(kept ? 16 : 0)
                                     : "memory");
                    }
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(arrive_bar + stage))
                                 : "memory");
                    if (++stage == S) { stage = 0; phase ^= 1u; }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(plan_empty + buf);
            }
        }
        // ------------------------------------------------ epilogue
        mbar_wait_sleep(accfull, 0);
        tc_fence_after();
        const int ew = warp - 4;
        const uint32_t lb = (uint32_t)(ew * 32) << 16;
        const int64_t n = n0 + ew * 32 + lane;
        float *out = p.out + (p.mode == 3 ? (int64_t)split * p.K * p.N : 0) + (int64_t)J0 * B * p.N + n;
        const int ncols = nbJ * B;
        for (int c = 0; c < ncols; c += 32) {
            uint32_t v[32];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(tmem + lb + (uint32_t)c));
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
                  "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
                  "=r"(v[30]), "=r"(v[31])
                : "r"(tmem + lb + (uint32_t)c + 16u));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int nc = min(32, ncols - c);
            float *o = out + (int64_t)c * p.N;
            if (p.mode == 1) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i < nc) o[(int64_t)i * p.N] += __uint_as_float(v[i]);
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i < nc) __stcg(o + (int64_t)i * p.N, __uint_as_float(v[i]));
            }
        }
    }
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if constexpr (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
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

static cudaError_t make_map(CUtensorMap *tm, const void *base, CUtensorMapDataType dt, int rank, const cuuint64_t *dims,
                            const cuuint64_t *strides, const cuuint32_t *box, CUtensorMapSwizzle sw) {
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
    CUresult r = fn(tm, dt, rank, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

struct Plan {
    int cg, nkr, kr_blocks, nchunk, cb, stages, nsplit, smem;
    uint32_t stage_bytes;
    bool ok;
};

template <int KIND, int B>
static Plan plan_for(int64_t M, int64_t K, int64_t N, int sms, int want_cg) {
    using C = Cfg<KIND, B>;
    Plan pl{};
    const int nbc = (int)(K / B);
    pl.cg = (want_cg == 2 && N % 256 == 0) ? 2 : 1;
    // kcol range: as wide as TMEM allows (one dY read per n tile), narrowed while
    // fewer than 3 pipeline stages fit in shared memory
    int maxJ = std::min(C::MAXJ, nbc);
    for (;;) {
        pl.nkr = (nbc + maxJ - 1) / maxJ;
        pl.kr_blocks = (nbc + pl.nkr - 1) / pl.nkr;
        pl.nchunk = (pl.kr_blocks + C::MAXCB - 1) / C::MAXCB;
        pl.cb = (pl.kr_blocks + pl.nchunk - 1) / pl.nchunk;
        while (pl.cb % (C::GRAN * pl.cg)) ++pl.cb;
        pl.stage_bytes = (uint32_t)((C::SLAB + pl.nchunk * (pl.cb / pl.cg) * C::BLOCK_BYTES + 1023) & ~1023);
        pl.stages = std::min(kMaxStages, (int)((kSmemBudget - kFixedSmem) / pl.stage_bytes));
        if (pl.stages >= 3 || maxJ <= 2) break;
        --maxJ;
    }
    pl.ok = pl.stages >= 2 && pl.cb <= C::MAXCB && pl.nchunk <= 2 && pl.cb <= 32 && nbc <= kColCap;
    pl.smem = (int)(pl.stages * pl.stage_bytes) + kFixedSmem;
    const int64_t ctas_per_split = (N / 128) * pl.nkr;  // CTAs (pairs count twice)
    const int64_t cap = std::min<int64_t>(sms, kSplitSMs);
    pl.nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(M / B, cap / std::max<int64_t>(1, ctas_per_split)));
    return pl;
}

// CTA pairs (cta_group::2) whenever N allows them (plan_for falls back to CG = 1).
constexpr int kWantCG = 2;


template <int KIND, int B, int CG>
static cudaError_t launch_cg(const Plan &pl, const CUtensorMap &tm_dy, const Params &p, cudaStream_t stream) {
    auto kern = wgrad_span_kernel<KIND, B, CG>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((p.N / 128) * pl.nkr * pl.nsplit);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = (size_t)pl.smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, tm_dy, p);
    count_launch();
    return e;
}

template <int KIND, int B>
static cudaError_t launch_t(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnzb, int64_t M,
                            int64_t K, const void *dY, int64_t N, float *dW, int accumulate, float *ws,
                            cudaStream_t stream) {
    using C = Cfg<KIND, B>;
    int dev = 0, sms = kSplitSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const Plan pl = plan_for<KIND, B>(M, K, N, sms, kWantCG);
    if (!pl.ok) return cudaErrorNotSupported;
    const CUtensorMapDataType dt = KIND == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const CUtensorMapSwizzle sw128 = C::TF32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
    // dY as (column within a 128-byte atom, row, atom): one box = the 128-column x
    // B-row slab of one block row, atom-major in shared memory
    CUtensorMap tm_dy;
    const cuuint64_t dy_dims[3] = {(cuuint64_t)C::ATOM_E, (cuuint64_t)M, (cuuint64_t)(N / C::ATOM_E)};
    const cuuint64_t dy_str[2] = {(cuuint64_t)N * C::ES, 128};
    const cuuint32_t dy_box[3] = {(cuuint32_t)C::ATOM_E, (cuuint32_t)B, (cuuint32_t)C::A_ATOMS};
    cudaError_t e = make_map(&tm_dy, dY, dt, 3, dy_dims, dy_str, dy_box, sw128);
    if (e != cudaSuccess) return e;
    Params p{};
    p.rowptr = rowptr;
    p.colidx = colidx;
    p.values = static_cast<const uint8_t *>(values);
    p.nbr = M / B;
    p.N = N;
    p.K = K;
    p.nnzb = nnzb;
    p.nkr = pl.nkr;
    p.kr_blocks = pl.kr_blocks;
    p.nsplit = pl.nsplit;
    p.nchunk = pl.nchunk;
    p.cb = pl.cb;
    p.stages = pl.stages;
    p.stage_bytes = pl.stage_bytes;
    p.mode = pl.nsplit > 1 ? 3 : accumulate ? 1 : 0;
    p.out = pl.nsplit > 1 ? ws : dW;
    e = pl.cg == 2 ? launch_cg<KIND, B, 2>(pl, tm_dy, p, stream) : launch_cg<KIND, B, 1>(pl, tm_dy, p, stream);
    if (e != cudaSuccess) return e;
    e = cudaGetLastError();
    if (e != cudaSuccess || pl.nsplit == 1) return e;
    return launch_splitk_reduce(ws, dW, K * N, pl.nsplit, accumulate, stream);
}

}  // namespace span


size_t wgrad_span_ws_bytes(int64_t M, int64_t K, int b, int64_t N) {
    int ns = 1;
#define WS_CASE(KD, B_)                                                          \
    if (b == B_) {                                                               \
        for (int cg = 1; cg <= 2; ++cg)                                          \
            ns = std::max(ns, span::plan_for<KD, B_>(M, K, N, span::kSplitSMs, cg).nsplit); \
    }
    WS_CASE(1, 16) WS_CASE(1, 32) WS_CASE(1, 64) WS_CASE(0, 16) WS_CASE(0, 32) WS_CASE(0, 64)
#undef WS_CASE
    return ns > 1 ? (size_t)ns * K * N * sizeof(float) : 0;
}

cudaError_t launch_wgrad_span(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnzb, int kind,
                              int64_t M, int64_t K, int b, const void *dY, int64_t N, float *dW, int accumulate,
                              void *ws, cudaStream_t stream) {
    if (!values || nnzb == 0) {
        return accumulate ? cudaSuccess : cudaMemsetAsync(dW, 0, (size_t)K * N * sizeof(float), stream);
    }
#define SP_CASE(KD, B_)                                                                                           \
    if (kind == KD && b == B_)                                                                                    \
        return span::launch_t<KD, B_>(rowptr, colidx, values, nnzb, M, K, dY, N, dW, accumulate, static_cast<float *>(ws), \
                                      stream);
    SP_CASE(0, 16) SP_CASE(0, 32) SP_CASE(0, 64) SP_CASE(1, 16) SP_CASE(1, 32) SP_CASE(1, 64)
#undef SP_CASE
    return cudaErrorInvalidValue;
}

}  // namespace bsrp
