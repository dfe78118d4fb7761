// prune.cu -- block l2 prune/pack on sm_100a (rows a1-a4 of SURVEY §8a).
//
// One persistent, cooperatively launched kernel does the whole forward-side
// step of the paper's operator:
//
//   phase 1  norms   : every warp streams one "unit" -- a 512-byte-wide strip
//                      of b rows covering G = 512/(b*elem) consecutive blocks of
//                      one block row -- with 128-bit loads, squares and sums
//                      each element column sequentially over the b rows (one
//                      fp32 accumulator per vector element), reduces the
//                      lanes of a block with a fixed xor-shuffle tree, and
//                      writes sumsq[f].  The first radix digit of the key is
//                      counted in a shared-memory histogram.
//   phase 2  select  : exact radix select of the k-th largest key over the
//                      fp32 bit patterns (12 + 10 + 9 bits); every CTA derives
//                      the same (prefix, shift, r) from the global histograms,
//                      refining only while the boundary bin is split.  Keys
//                      strictly above the prefix are kept, and the first r keys
//                      equal to it in flat order (BJ tie rule).
//   phase 3  scan    : per-CTA (above, tie) counts -> grid barrier -> CTA
//                      prefix -> block-wide scans in flat order give every
//                      kept block its output slot
//                        pos(f) = above_before(f) + min(r, tie_before(f))
//                      and rowptr / colidx.
//   phase 4  pack    : the same warp units re-read only kept blocks (L2-hot
//                      when X fits the 126 MB L2) and copy them as raw
//                      integer vectors into values[pos][b][b].
//
// Units are statically partitioned into contiguous ranges per CTA, so phases
// 1, 3 and 4 of a CTA touch the same flat range and need no cross-CTA data
// except the histograms and the per-CTA counts.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace bsrp {

constexpr int kThreads = 512;
constexpr int kH1 = 4096, kH2 = 1024, kH3 = 512;  // digit sizes: key bits 30..19, 18..9, 8..0
constexpr int kCandMax = kH1;  // boundary-bin candidates exchanged through the workspace

struct PruneParams {
    const void *X;
    int64_t K, nbr, nbc, N, k, units, upr;
    int32_t *rowptr, *colidx;
    void *values;
    float *sumsq;
    int32_t *slot;
    uint32_t *bar, *hist1, *hist2, *hist3, *cta_cnt;
    uint2 *cand;  // [kCandMax] (key, flat index) of the boundary bin's blocks
    int pdl_trig;   // 1: trigger the PDL successor before the pack phase
    int presummed;  // 1: block sums already in `sumsq` (act_sumsq_kernel); phase 1 skips X
    const unsigned long long *gstate;  // device-side global selection (select_global.cu): T, shift, r, k from here
};

// Selection key of a block: fp32 bits of sumsq (>= 0, so the integer order is
// the float order).  NaN is folded to 0x7fffffff and ranks above +inf (R12).
__device__ __forceinline__ uint32_t key_of(float s) { return __float_as_uint(s) & 0x7fffffffu; }

template <int ES, typename V>
__device__ __forceinline__ float elem(const V &v, int e) {
    if constexpr (ES == 4) {
        return __uint_as_float(word(v, e));
    } else {
        uint32_t w = word(v, e >> 1);
        return __uint_as_float((e & 1) ? (w & 0xffff0000u) : (w << 16));
    }
}

template <int ES, int B>
struct Geo {
    static constexpr int VB = (B * ES >= 16) ? 16 : B * ES;  // bytes per lane vector
    static constexpr int EPV = VB / ES;                      // elements per vector
    static constexpr int LPB = B / EPV;                      // lanes per block row
    static constexpr int G = kWarp / LPB;                    // blocks per warp unit
    static constexpr int R = (B < 16) ? (B < 8 ? B : 8) : 16;  // rows in flight per lane
    using V = typename Vec<VB>::T;
};

// Sum of squares of block (I, J) for this lane's vector column; returns the
// block total on every lane of the block's lane segment.
template <int ES, int B>
__device__ __forceinline__ float block_sumsq_warp(const void *X, int64_t K, int64_t I, int64_t J, int sub,
                                                  bool valid) {
    // ld.global.cg (L2 only, normal L2 priority) so that the phase-4 re-read of
    // the kept blocks hits L2 when X fits in it.
    using G_ = Geo<ES, B>;
    using V = typename G_::V;
    float acc[G_::EPV];
#pragma unroll
    for (int e = 0; e < G_::EPV; ++e) acc[e] = 0.f;
    if (valid) {
        const int64_t rs = K / G_::EPV;  // row stride in vectors
        const V *src = reinterpret_cast<const V *>(X) + (I * B) * rs + (J * B) / G_::EPV + sub;
#pragma unroll
        for (int r0 = 0; r0 < B; r0 += G_::R) {
            V v[G_::R];
#pragma unroll
            for (int rr = 0; rr < G_::R; ++rr) v[rr] = __ldcg(src + (r0 + rr) * rs);
#pragma unroll
            for (int rr = 0; rr < G_::R; ++rr)
#pragma unroll
                for (int e = 0; e < G_::EPV; ++e) {
                    float x = elem<ES>(v[rr], e);
                    acc[e] = fmaf(x, x, acc[e]);
                }
        }
    }
    // pairwise tree over the vector's element columns
#pragma unroll
    for (int w = 1; w < G_::EPV; w <<= 1)
#pragma unroll
        for (int e = 0; e < G_::EPV; e += 2 * w) acc[e] = acc[e] + acc[e + w];
    float s = acc[0];
    // xor tree over the LPB lanes of the block (identical result on each lane)
#pragma unroll
    for (int off = 1; off < G_::LPB; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    return s;
}

// Exclusive block scan of 64-bit values (blockDim.x == kThreads).
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t *s_warp, uint64_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint64_t t = lane < nw ? s_warp[lane] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, t, off);
            if (lane >= off) t += y;
        }
        s_warp[lane] = t;
    }
    __syncthreads();
    const uint64_t base = wid > 0 ? s_warp[wid - 1] : 0;
    total = s_warp[nw - 1];
    __syncthreads();
    return base + x - v;
}

// Find the bin that holds the `target`-th largest key (1-based) of a global
// histogram with `nbins` bins; returns (bin, count strictly above the bin).
// Thread 0 owns the top bins, so an exclusive prefix over threads = keys above.
template <bool GLOBAL = true>  // hist in global memory (read through L2) or in shared memory
__device__ __forceinline__ void select_bin(const uint32_t *hist, int nbins, uint32_t target, uint64_t *s_warp,
                                           uint32_t *s_out) {
    const int per = nbins / kThreads;  // 8, 2 or 1
    const int hi = nbins - threadIdx.x * per;
    uint32_t h[8];
    uint32_t local = 0;
    for (int i = 0; i < per; ++i) {
        h[i] = GLOBAL ? __ldcg(hist + hi - 1 - i) : hist[hi - 1 - i];  // descending bins
        local += h[i];
    }
    uint64_t total;
    uint32_t run = (uint32_t)block_excl_scan(local, s_warp, total);
    for (int i = 0; i < per; ++i) {
        if (run < target && run + h[i] >= target) {
            s_out[0] = hi - 1 - i;
            s_out[1] = run;
            s_out[2] = h[i];
        }
        run += h[i];
    }
    __syncthreads();
}

// Phase 3 of a CTA: flat-order scan of its block range [f0, f1) given the
// (above, tie) counts of every block before it (`pre`): output slots,
// colidx and rowptr, slot[f] = -1 for pruned blocks.
__device__ __forceinline__ void scan_and_index(const PruneParams &p, int64_t f0, int64_t f1, uint64_t pre,
                                               uint32_t prefix, int shift, uint32_t r, uint64_t *s_warp,
                                               const uint32_t *s_keys = nullptr) {
    uint32_t base_a = (uint32_t)(pre >> 32), base_t = (uint32_t)pre;
    if (blockIdx.x == 0 && threadIdx.x == 0) p.rowptr[0] = 0;
    for (int64_t fb = f0; fb < f1; fb += kThreads) {
        const int64_t f = fb + threadIdx.x;
        const bool in = f < f1;
        uint32_t a = 0, t = 0;
        if (in) {
            uint32_t kk = (s_keys ? s_keys[f] : key_of(p.sumsq[f])) >> shift;
            a = kk > prefix;
            t = kk == prefix;
        }
        uint64_t tot;
        uint64_t ex = block_excl_scan(((uint64_t)a << 32) | t, s_warp, tot);
        const uint32_t ab = base_a + (uint32_t)(ex >> 32), tb = base_t + (uint32_t)ex;
        if (in) {
            const uint32_t pos = ab + min(r, tb);
            const bool kept = (a || (t && tb < r)) && pos < (uint64_t)p.k;  // pos < k: guards a caller's wrong k
            const int64_t I = f / p.nbc, J = f - I * p.nbc;
            p.slot[f] = kept ? (int32_t)pos : -1;
            if (kept) p.colidx[pos] = (int32_t)J;
            if (J == p.nbc - 1) p.rowptr[I + 1] = (int32_t)(ab + a + min(r, tb + t));
        }
        base_a += (uint32_t)(tot >> 32);
        base_t += (uint32_t)tot;
    }
    __syncthreads();

}

// Phase 4 of a CTA: the same warp units re-read only the kept blocks and store
// them as raw integer vectors into values[slot] (bit-exact).
template <int ES, int B>
__device__ __forceinline__ void pack_kept(const PruneParams &p, int64_t u0, int64_t u1) {
    using G_ = Geo<ES, B>;
    using V = typename G_::V;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x / 32;
    const int j = lane / G_::LPB, sub = lane % G_::LPB;
    for (int64_t u = u0 + wid; u < u1; u += nw) {
        const int64_t I = u / p.upr, J = (u % p.upr) * G_::G + j;
        const int32_t s = (J < p.nbc) ? p.slot[I * p.nbc + J] : -1;
        if (s >= 0) {
            const int64_t rs = p.K / G_::EPV;
            const V *src = reinterpret_cast<const V *>(p.X) + (I * B) * rs + (J * B) / G_::EPV + sub;
            V *dst = reinterpret_cast<V *>(p.values) + (int64_t)s * (B * B / G_::EPV) + sub;
#pragma unroll
            for (int r0 = 0; r0 < B; r0 += G_::R) {
                V v[G_::R];
#pragma unroll
                for (int rr = 0; rr < G_::R; ++rr) v[rr] = __ldcg(src + (r0 + rr) * rs);
#pragma unroll
                for (int rr = 0; rr < G_::R; ++rr) __stcs(dst + (r0 + rr) * G_::LPB, v[rr]);
            }
        }
    }
}


template <int ES, int B>
__global__ void __launch_bounds__(kThreads, (B >= 16) ? 1 : 2) prune_kernel(PruneParams p) {
    using G_ = Geo<ES, B>;
    __shared__ uint32_t s_hist[kH1];  // level-1 histogram, then the candidate keys
    __shared__ uint32_t s_f[kCandMax];  // candidate flat indices
    __shared__ uint32_t s_h2[1024];     // candidate refinement histogram
    __shared__ uint64_t s_warp[32];
    __shared__ uint32_t s_sel[4];

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kThreads / 32;
    const int64_t u0 = (int64_t)blockIdx.x * p.units / gridDim.x;
    const int64_t u1 = (int64_t)(blockIdx.x + 1) * p.units / gridDim.x;
    auto flat_start = [&](int64_t u) -> int64_t {
        return u >= p.units ? p.N : (u / p.upr) * p.nbc + (u % p.upr) * G_::G;
    };
    const int64_t f0 = flat_start(u0), f1 = flat_start(u1);
    const int j = lane / G_::LPB, sub = lane % G_::LPB;
    uint32_t nbar = 0;
    // ---------------- phase 1: block sums of squares + level-1 histogram
    for (int i = threadIdx.x; i < kH1; i += kThreads) s_hist[i] = 0;
    __syncthreads();
    if (p.presummed) {  // sums written by the producer (act_sumsq_kernel): X is not read here
        for (int64_t f = f0 + threadIdx.x; f < f1; f += kThreads) atomicAdd(&s_hist[key_of(p.sumsq[f]) >> 19], 1u);
    } else {
        for (int64_t u = u0 + wid; u < u1; u += nw) {
            const int64_t I = u / p.upr, J = (u % p.upr) * G_::G + j;
            const bool valid = J < p.nbc;
            float s = block_sumsq_warp<ES, B>(p.X, p.K, I, J, sub, valid);
            if (valid && sub == 0) {
                p.sumsq[I * p.nbc + J] = s;
                atomicAdd(&s_hist[key_of(s) >> 19], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kH1; i += kThreads)
        if (s_hist[i]) atomicAdd(p.hist1 + i, s_hist[i]);
    grid_barrier(p.bar, nbar++);

    // ---------------- phase 2: radix select of the k-th largest key
    const uint32_t k = (uint32_t)p.k;
    select_bin(p.hist1, kH1, k, s_warp, s_sel);
    uint32_t prefix = s_sel[0], above = s_sel[1], bincnt = s_sel[2];
    int shift = 19;
    uint32_t r = k - above;
    uint64_t pre = 0;
    bool have_pre = false;
    if (r < bincnt) {
        // Candidate exchange (one barrier instead of two refinement rounds and the
        // scan barrier): every CTA publishes its count of keys above the boundary
        // bin and appends its keys inside the bin, with their flat index, to a
        // global list.  After the barrier each CTA resolves the exact threshold
        // from the list and its own prefix counts (CTAs before it + listed keys
        // before its range) -- when the bin fits the list.
        if (bincnt <= (uint32_t)kCandMax) {
            const uint32_t prefix1 = prefix;
            // pass A: this CTA's counts (keys above the bin, keys in it) -> one atomic
            // reservation of list slots per CTA (a single hot counter would serialise)
            uint32_t na = 0, ni = 0;
            for (int64_t f = f0 + threadIdx.x; f < f1; f += kThreads) {
                const uint32_t hb = key_of(p.sumsq[f]) >> 19;
                na += hb > prefix1;
                ni += hb == prefix1;
            }
            uint32_t slot0, ni_cta;
            {
                uint64_t tot;
                block_excl_scan(((uint64_t)na << 32) | ni, s_warp, tot);
                ni_cta = (uint32_t)tot;
                if (threadIdx.x == 0) {
                    p.cta_cnt[2 * blockIdx.x] = (uint32_t)(tot >> 32);
                    s_sel[3] = (uint32_t)tot ? atomicAdd(p.bar + 16, (uint32_t)tot) : 0u;
                }
                __syncthreads();
                slot0 = s_sel[3];
            }
            // pass B: append the bin's keys with their flat index, in flat order
            for (int64_t fb = f0; fb < f1 && ni_cta; fb += kThreads) {
                const int64_t f = fb + threadIdx.x;
                uint32_t key = 0;
                bool in = false;
                if (f < f1) {
                    key = key_of(p.sumsq[f]);
                    in = (key >> 19) == prefix1;
                }
                uint64_t tot;
                const uint32_t ex = (uint32_t)block_excl_scan(in ? 1u : 0u, s_warp, tot);
                const uint32_t slot = slot0 + ex;
                if (in && slot < (uint32_t)kCandMax) p.cand[slot] = make_uint2(key, (uint32_t)f);
                slot0 += (uint32_t)tot;
            }
            grid_barrier(p.bar, nbar++);
            const uint32_t nc = __ldcg(p.bar + 16);  // == bincnt
            {
                for (uint32_t i0 = threadIdx.x; i0 < nc; i0 += 8 * kThreads) {  // 8 independent loads in flight
                    uint2 c[8];
    #pragma unroll
                    for (int u = 0; u < 8; ++u) c[u] = i0 + u * kThreads < nc ? __ldcg(p.cand + i0 + u * kThreads) : uint2{};
    #pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (i0 + u * kThreads < nc) {
                            s_hist[i0 + u * kThreads] = c[u].x;
                            s_f[i0 + u * kThreads] = c[u].y;
                        }
                }
                __syncthreads();
                for (int pass = 0; pass < 2 && r < bincnt; ++pass) {  // key bits 18..9, then 8..0
                    const int w = pass == 0 ? 10 : 9;
                    const int nshift = shift - w;
                    for (int i = threadIdx.x; i < (1 << w); i += kThreads) s_h2[i] = 0;
                    __syncthreads();
                    for (uint32_t ib = 0; ib < nc; ib += kThreads) {
                        const uint32_t i = ib + threadIdx.x;
                        const uint32_t key = i < nc ? s_hist[i] : 0u;
                        const bool in = i < nc && (key >> shift) == prefix;
                        const uint32_t bin = (key >> nshift) & ((1u << w) - 1u);
                        const uint32_t im = __ballot_sync(0xffffffffu, in);
                        if (!im) continue;
                        const int l0 = __ffs(im) - 1;
                        const uint32_t b0 = __shfl_sync(0xffffffffu, bin, l0);
                        if (__all_sync(0xffffffffu, !in || bin == b0)) {  // a warp of ties adds once
                            if (lane == l0) atomicAdd(&s_h2[b0], (uint32_t)__popc(im));
                        } else if (in) {
                            atomicAdd(&s_h2[bin], 1u);
                        }
                    }
                    __syncthreads();
                    select_bin<false>(s_h2, 1 << w, r, s_warp, s_sel);
                    prefix = (prefix << w) | s_sel[0];
                    above += s_sel[1];
                    bincnt = s_sel[2];
                    shift = nshift;
                    r = k - above;
                }
                // (above, tie) counts of every block before this CTA's range
                uint64_t cnt = 0;
                for (int c = threadIdx.x; c < (int)blockIdx.x; c += kThreads) cnt += (uint64_t)__ldcg(p.cta_cnt + 2 * c) << 32;
                for (uint32_t i = threadIdx.x; i < nc; i += kThreads) {
                    if ((int64_t)s_f[i] >= f0) continue;
                    const uint32_t kk = s_hist[i] >> shift;
                    cnt += kk > prefix ? (uint64_t)1 << 32 : (kk == prefix ? 1u : 0u);
                }
                uint64_t tot;
                block_excl_scan(cnt, s_warp, tot);
                pre = tot;
                have_pre = true;
    }
        } else {
            // the boundary bin does not fit the list (large N or heavy ties): global
            // refinement rounds (decided from the global histogram, before any pass)
            for (int i = threadIdx.x; i < kH2; i += kThreads) s_hist[i] = 0;
            __syncthreads();
            for (int64_t f = f0 + threadIdx.x; f < f1; f += kThreads) {
                uint32_t key = key_of(p.sumsq[f]);
                if ((key >> 19) == prefix) atomicAdd(&s_hist[(key >> 9) & (kH2 - 1)], 1u);
            }
            __syncthreads();
            for (int i = threadIdx.x; i < kH2; i += kThreads)
                if (s_hist[i]) atomicAdd(p.hist2 + i, s_hist[i]);
            grid_barrier(p.bar, nbar++);
            select_bin(p.hist2, kH2, r, s_warp, s_sel);
            prefix = (prefix << 10) | s_sel[0];
            above += s_sel[1];
            bincnt = s_sel[2];
            shift = 9;
            r = k - above;
            if (r < bincnt) {  // refine on key bits 8..0
                for (int i = threadIdx.x; i < kH3; i += kThreads) s_hist[i] = 0;
                __syncthreads();
                for (int64_t f = f0 + threadIdx.x; f < f1; f += kThreads) {
                    uint32_t key = key_of(p.sumsq[f]);
                    if ((key >> 9) == prefix) atomicAdd(&s_hist[key & (kH3 - 1)], 1u);
                }
                __syncthreads();
                for (int i = threadIdx.x; i < kH3; i += kThreads)
                    if (s_hist[i]) atomicAdd(p.hist3 + i, s_hist[i]);
                grid_barrier(p.bar, nbar++);
                select_bin(p.hist3, kH3, r, s_warp, s_sel);
                prefix = (prefix << 9) | s_sel[0];
                above += s_sel[1];
                shift = 0;
                r = k - above;
            }
        }
    }
    // ---------------- phase 3: flat-order scan -> slots, colidx, rowptr
    if (!have_pre) {
        uint32_t na = 0, nt = 0;
        for (int64_t f = f0 + threadIdx.x; f < f1; f += kThreads) {
            uint32_t kk = key_of(p.sumsq[f]) >> shift;
            na += kk > prefix;
            nt += kk == prefix;
        }
        {
            uint64_t tot;
            block_excl_scan(((uint64_t)na << 32) | nt, s_warp, tot);
            if (threadIdx.x == 0) {
                p.cta_cnt[2 * blockIdx.x] = (uint32_t)(tot >> 32);
                p.cta_cnt[2 * blockIdx.x + 1] = (uint32_t)tot;
            }
        }
        grid_barrier(p.bar, nbar++);
        for (int c = threadIdx.x; c < (int)blockIdx.x; c += kThreads)
            pre += ((uint64_t)__ldcg(p.cta_cnt + 2 * c) << 32) | __ldcg(p.cta_cnt + 2 * c + 1);
        {
            uint64_t tot;
            block_excl_scan(pre, s_warp, tot);
            pre = tot;
        }
    }
    // Self-cleaning workspace: every CTA is past its last read of the barrier counter
    // and the histograms; the last one to get here zeroes them for the next launch
    // (so no per-launch memset is needed once the workspace was zero-filled).
    if (threadIdx.x == 0) {
        __threadfence();
        s_sel[3] = atomicAdd(p.bar + 32, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_sel[3]) {
        __threadfence();
        for (int i = threadIdx.x; i < kH1; i += kThreads) p.hist1[i] = 0;
        for (int i = threadIdx.x; i < kH2; i += kThreads) p.hist2[i] = 0;
        for (int i = threadIdx.x; i < kH3; i += kThreads) p.hist3[i] = 0;
        if (threadIdx.x == 0) {
            p.bar[0] = 0;
            p.bar[16] = 0;
            p.bar[32] = 0;
        }
    }
    scan_and_index(p, f0, f1, pre, prefix, shift, r, s_warp);
    // ---------------- phase 4: copy kept blocks (raw integer vectors)
    if (p.pdl_trig) pdl_trigger();  // the next kernel (launched with PDL) may start its prologue
    pack_kept<ES, B>(p, u0, u1);
    __syncthreads();
}

// ------------------------------------------------------------------ small-N path
// Two plain (non-cooperative) launches chained with programmatic dependent
// launch instead of one cooperative kernel with grid barriers, for N <= kSmallN
// keys (S12 fc1/fc2 at b >= 16-32, B24 per-rank fc1): the kernel boundary is the
// only grid-wide synchronisation.
//   prune_sums_kernel : phase 1 of prune_kernel (same units, same reduction tree,
//                       so bit-identical block sums).  It triggers its dependent
//                       at its start, so the finishing CTAs are already resident
//                       (waiting in griddepcontrol.wait) when the sums complete.
//   prune_finish_kernel: every CTA loads ALL N keys into shared memory and counts
//                       their first digit there (no global histogram, nothing to
//                       clean up), resolves the exact threshold (the boundary bin
//                       refined by two more digits over a candidate list in shared
//                       memory), counts the (above, tie) keys before its own flat
//                       range, then scans and packs its range as prune_kernel does.
//                       No grid barrier, no global atomics.
//   STOCH (bsr_prune_stochastic, R19): every CTA also resolves ranks k - w and
//                       k + w, walks all keys in flat order to mark ranks < k - w
//                       and collect the 2w boundary blocks, sorts them by rank in
//                       shared memory and applies the swaps -- each CTA reaches the
//                       same kept set and packs its own range.
constexpr int64_t kSmallN = 24576;  // keys held in shared memory by every finishing CTA (96 KB); measured:
                                    // at 37632 keys (S12 fc1 b = 16) the per-CTA passes cost more than the
                                    // cooperative kernel's barriers
constexpr int kSmallCand = 4096;    // boundary-bin candidates (key, flat index) in shared memory (32 KB)

template <int ES, int B>
__global__ void __launch_bounds__(kThreads, (B >= 16) ? 1 : 2) prune_sums_kernel(PruneParams p) {
    using G_ = Geo<ES, B>;
    __shared__ uint32_t s_hist[kH1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kThreads / 32;
    const int j = lane / G_::LPB, sub = lane % G_::LPB;
    const bool hist = p.hist1 != nullptr;  // global first-digit histogram (the multi-kernel stochastic path)
    if (hist) {
        for (int i = threadIdx.x; i < kH1; i += kThreads) s_hist[i] = 0;
        __syncthreads();
    }
    pdl_wait();  // launched with PDL: the predecessor (e.g. the previous step) has completed
    pdl_trigger();  // the finishing kernel may become resident now; it waits for this grid's completion
    if (p.presummed) {
        if (hist)
            for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < p.N; f += (int64_t)gridDim.x * kThreads)
                atomicAdd(&s_hist[key_of(p.sumsq[f]) >> 19], 1u);
    } else {
        for (int64_t u = (int64_t)blockIdx.x * nw + wid; u < p.units; u += (int64_t)gridDim.x * nw) {
            const int64_t I = u / p.upr, J = (u % p.upr) * G_::G + j;
            const bool valid = J < p.nbc;
            const float sq = block_sumsq_warp<ES, B>(p.X, p.K, I, J, sub, valid);
            if (valid && sub == 0) {
                p.sumsq[I * p.nbc + J] = sq;
                if (hist) atomicAdd(&s_hist[key_of(sq) >> 19], 1u);
            }
        }
    }
    if (hist) {
        __syncthreads();
        for (int i = threadIdx.x; i < kH1; i += kThreads)
            if (s_hist[i]) atomicAdd(p.hist1 + i, s_hist[i]);
    }
}

// Shared-memory histogram add with the warp's ties folded into one atomic
// (all lanes of the warp must call it).
__device__ __forceinline__ void hist_add_warp(uint32_t *h, uint32_t bin, bool valid) {
    const int lane = threadIdx.x & 31;
    const uint32_t m = __ballot_sync(0xffffffffu, valid);
    if (!m) return;
    const int l0 = __ffs(m) - 1;
    const uint32_t b0 = __shfl_sync(0xffffffffu, bin, l0);
    if (__all_sync(0xffffffffu, !valid || bin == b0)) {
        if (lane == l0) atomicAdd(&h[b0], (uint32_t)__popc(m));
    } else if (valid) {
        atomicAdd(&h[bin], 1u);
    }
}

// Refine a boundary bin (prefix at `shift`) by the next digits until the target's
// tie quota r is resolved or the key is exact.  arr/len: keys to histogram.
__device__ __forceinline__ void refine_bin(const uint32_t *arr, int len, uint32_t target, uint32_t &prefix, int &shift,
                                           uint32_t &above, uint32_t &bincnt, uint32_t &r, uint32_t *s_h2,
                                           uint64_t *s_warp, uint32_t *s_sel) {
    for (int pass = 0; pass < 2 && r < bincnt; ++pass) {
        const int w = pass == 0 ? 10 : 9;
        const int nshift = shift - w;
        for (int i = threadIdx.x; i < (1 << w); i += kThreads) s_h2[i] = 0;
        __syncthreads();
        for (int fb = 0; fb < len; fb += kThreads) {
            const int f = fb + threadIdx.x;
            const uint32_t key = f < len ? arr[f] : 0u;
            const bool in = f < len && (key >> shift) == prefix;
            hist_add_warp(s_h2, (key >> nshift) & ((1u << w) - 1u), in);
        }
        __syncthreads();
        select_bin<false>(s_h2, 1 << w, r, s_warp, s_sel);
        prefix = (prefix << w) | s_sel[0];
        above += s_sel[1];
        bincnt = s_sel[2];
        shift = nshift;
        r = target - above;
    }
}

struct StochArgs {
    int64_t w;  // boundary pairs (0: deterministic top-k)
    double prob;
    unsigned long long seed;
};

__device__ __forceinline__ double swap_uniform(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

// In-place descending bitonic sort of P (a power of two) 64-bit words in shared memory.
// (A variant visiting the P/2 pairs directly with 8 loads in flight per thread
// was no faster in the stochastic sweep -- profiles/r02e vs r02d -- and was dropped.)
__device__ __forceinline__ void bitonic_desc(unsigned long long *a, int P) {
    for (int kk = 2; kk <= P; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long x = a[i], y = a[ixj];
                    if ((i & kk) == 0 ? x < y : x > y) {
                        a[i] = y;
                        a[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
}

// Full passes over the N keys in shared memory use thread-contiguous chunks:
// thread t owns keys [t c, (t+1) c) with c odd (at each step the 32 lanes of a
// warp read 32 distinct banks), so thread order is flat order and a block scan of
// per-thread counts gives every thread its flat-order start.
__device__ __forceinline__ void my_chunk(int N, int &t0, int &t1) {
    const int c = ((N + kThreads - 1) / kThreads) | 1;
    t0 = min(N, (int)threadIdx.x * c);
    t1 = min(N, t0 + c);
}

constexpr uint32_t kDirectRank = 64;  // bins up to this size: direct ranks (O(bc^2) compares; measured: at
                                      // ~500 keys they cost 5 us, the two refinement digits ~1.5 us)

// Exact threshold of the tgt-th largest key (tgt >= 1) from the first-digit
// histogram in shared memory: keep keys (>> shift) > T and the first r keys
// (>> shift) == T in flat order.  The boundary bin's keys are listed (key, flat
// index; one pass, order free) and, when there are at most kDirectRank, each
// computes its own rank among them directly -- rank = #(larger keys) + #(equal keys at
// lower flat index) -- so the rank tgt-1 candidate gives the full key (shift 0)
// and its tie quota.  Larger bins are refined digit by digit (refine_bin) over
// the list, or over all keys when they exceed it.
// PRE: also return this CTA's scan start `pre` = (above << 32 | tie) over the keys
// at flat index < fpre, counted in the same passes (keys outside the boundary bin
// during the list pass, the bin's own keys from the list).
template <bool PRE>
__device__ __forceinline__ void resolve_target(const uint32_t *s_key, int N, int t0, int t1, uint32_t tgt,
                                               const uint32_t *s_h1, uint32_t *s_ck, uint32_t *s_cf,
                                               uint32_t *s_h2, uint64_t *s_warp, uint32_t *s_sel,
                                               uint32_t &T, int &shift, uint32_t &r, int fpre = 0,
                                               uint64_t *pre = nullptr) {
    select_bin<false>(s_h1, kH1, tgt, s_warp, s_sel);
    uint32_t pf = s_sel[0], ab = s_sel[1], bc = s_sel[2];
    shift = 19;
    r = tgt - ab;
    __syncthreads();
    uint32_t na = 0, nt = 0;
    if (r >= bc || bc > (uint32_t)kSmallCand) {
        if (r < bc)  // heavy ties: digit refinement over all keys
            refine_bin(s_key, N, tgt, pf, shift, ab, bc, r, s_h2, s_warp, s_sel);
        T = pf;      // else the whole bin is kept
        if (PRE) {
            for (int f = t0; f < min(t1, fpre); ++f) {
                const uint32_t kk = s_key[f] >> shift;
                na += kk > T;
                nt += kk == T;
            }
            uint64_t tot;
            block_excl_scan(((uint64_t)na << 32) | nt, s_warp, tot);
            *pre = tot;
        }
        return;
    }
    if (threadIdx.x == 0) s_sel[3] = 0;
    __syncthreads();
    for (int f = t0; f < t1; ++f) {
        const uint32_t key = s_key[f];
        const uint32_t d = key >> 19;
        if (PRE) na += d > pf && f < fpre;
        if (d == pf) {
            const uint32_t pos = atomicAdd(&s_sel[3], 1u);
            s_ck[pos] = key;
            s_cf[pos] = (uint32_t)f;
        }
    }
    __syncthreads();
    const uint32_t nc = bc;  // list length (refine_bin narrows bc)
    if (bc > kDirectRank) {
        refine_bin(s_ck, (int)bc, tgt, pf, shift, ab, bc, r, s_h2, s_warp, s_sel);
        T = pf;
    } else {
        if (threadIdx.x < bc) {
            const uint32_t ki = s_ck[threadIdx.x], fi = s_cf[threadIdx.x];
            uint32_t gt = 0, eq = 0;
            for (uint32_t j = 0; j < bc; ++j) {
                const uint32_t kj = s_ck[j];
                gt += kj > ki;
                eq += kj == ki && s_cf[j] < fi;
            }
            if (gt + eq == r - 1) {  // exactly one candidate holds rank r-1 within the bin
                s_sel[0] = ki;
                s_sel[1] = r - gt;  // ties of ki kept: those at lower flat index and itself
            }
        }
        __syncthreads();
        T = s_sel[0];
        r = s_sel[1];
        shift = 0;
    }
    if (PRE) {
        for (uint32_t i = threadIdx.x; i < nc; i += kThreads)
            if ((int)s_cf[i] < fpre) {
                const uint32_t kk = s_ck[i] >> shift;
                na += kk > T;
                nt += kk == T;
            }
        uint64_t tot;
        block_excl_scan(((uint64_t)na << 32) | nt, s_warp, tot);
        *pre = tot;
    }
    __syncthreads();
}

template <int ES, int B, bool STOCH>
__global__ void __launch_bounds__(kThreads, 1) prune_finish_kernel(PruneParams p, StochArgs sa) {
    extern __shared__ __align__(16) uint32_t s_dyn[];
    __shared__ uint32_t s_h2[1024];
    __shared__ uint64_t s_warp[32];
    __shared__ uint32_t s_sel[4];
    using G_ = Geo<ES, B>;
    const int N = (int)p.N;
    const int npad = (N + 3) & ~3;
    uint32_t *s_key = s_dyn;                 // [npad] key bits, flat order (STOCH: then the final marks)
    uint32_t *s_h1 = s_key + npad;           // [kH1] first-digit histogram
    uint32_t *s_ck = s_h1 + kH1;             // [kSmallCand] candidate keys    | STOCH: [P] 64-bit boundary
    uint32_t *s_cf = s_ck + kSmallCand;      // [kSmallCand] flat indices      |        list (sorted by rank)
    for (int i = threadIdx.x; i < kH1; i += kThreads) s_h1[i] = 0;
    pdl_wait();  // the sums kernel has completed: sumsq is final
    // every key into shared memory (16-byte loads, 4 in flight per thread)
    {
        const float4 *src = reinterpret_cast<const float4 *>(p.sumsq);
        const int n4 = N / 4;
        for (int i0 = 0; i0 < n4; i0 += 4 * kThreads) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kThreads + threadIdx.x;
                v[u] = i < n4 ? __ldcg(src + i) : float4{};
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kThreads + threadIdx.x;
                if (i < n4)
                    reinterpret_cast<uint4 *>(s_key)[i] =
                        make_uint4(key_of(v[u].x), key_of(v[u].y), key_of(v[u].z), key_of(v[u].w));
            }
        }
        for (int f = n4 * 4 + threadIdx.x; f < N; f += kThreads) s_key[f] = key_of(__ldcg(p.sumsq + f));
    }
    __syncthreads();
    int t0, t1;
    my_chunk(N, t0, t1);
    for (int f = t0; f < t1; ++f) atomicAdd(&s_h1[s_key[f] >> 19], 1u);  // first digit (bits 30..19)
    __syncthreads();
    uint32_t pf, r;
    int shift;
    const int64_t u0 = (int64_t)blockIdx.x * p.units / gridDim.x;
    const int64_t u1 = (int64_t)(blockIdx.x + 1) * p.units / gridDim.x;
    auto flat_start = [&](int64_t u) -> int64_t {
        return u >= p.units ? p.N : (u / p.upr) * p.nbc + (u % p.upr) * G_::G;
    };
    const int f0 = (int)flat_start(u0), f1 = (int)flat_start(u1);
    uint64_t pre = 0;
    if constexpr (!STOCH) {
        resolve_target<true>(s_key, N, t0, t1, (uint32_t)p.k, s_h1, s_ck, s_cf, s_h2, s_warp, s_sel, pf, shift, r,
                             f0, &pre);
    } else {
        // ranks [0, k - w) kept, [k - w, k + w) the boundary (R19)
        const int w = (int)sa.w;
        uint32_t T[2], rr[2];
        int sh[2];
        for (int t = 0; t < 2; ++t) {
            const uint32_t tgt = (uint32_t)(t == 0 ? p.k - w : p.k + w);
            if (tgt == 0) {  // empty selection: a prefix no key reaches
                T[t] = 0xffffffffu;
                sh[t] = 0;
                rr[t] = 0;
                continue;
            }
            resolve_target<false>(s_key, N, t0, t1, tgt, s_h1, s_ck, s_cf, s_h2, s_warp, s_sel, T[t], sh[t], rr[t]);
        }
        // marks in place of the keys: kept 0xffffffff, pruned 0x80000000, the 2w
        // boundary blocks keep their key (< 2^31) until listed
        constexpr uint32_t KEPT = 0xffffffffu, PRUNED = 0x80000000u;
        uint32_t nA = 0, nB = 0;
        for (int f = t0; f < t1; ++f) {
            const uint32_t key = s_key[f];
            nA += (key >> sh[0]) == T[0];
            nB += (key >> sh[1]) == T[1];
        }
        uint64_t tot;
        const uint64_t ex = block_excl_scan(((uint64_t)nA << 32) | nB, s_warp, tot);
        uint32_t bA = (uint32_t)(ex >> 32), bB = (uint32_t)ex, nbnd = 0;
        for (int f = t0; f < t1; ++f) {
            const uint32_t key = s_key[f];
            const uint32_t kA = key >> sh[0], kB = key >> sh[1];
            const bool inA = kA > T[0] || (kA == T[0] && bA < rr[0]);
            const bool inB = kB > T[1] || (kB == T[1] && bB < rr[1]);
            bA += kA == T[0];
            bB += kB == T[1];
            if (inA) s_key[f] = KEPT;
            else if (inB) ++nbnd;
            else s_key[f] = PRUNED;
        }
        uint32_t pb = (uint32_t)block_excl_scan(nbnd, s_warp, tot);
        if ((uint32_t)tot != 2u * (uint32_t)w) __trap();  // |ranks [k - w, k + w)| = 2w by construction
        unsigned long long *s_b = reinterpret_cast<unsigned long long *>(s_ck);
        for (int f = t0; f < t1; ++f) {
            const uint32_t v = s_key[f];
            if (v < PRUNED) {
                s_b[pb++] = ((unsigned long long)v << 32) | (0xffffffffu - (uint32_t)f);
                s_key[f] = PRUNED;
            }
        }
        int P = 1;
        while (P < 2 * w) P <<= 1;
        for (int i = 2 * w + threadIdx.x; i < P; i += kThreads) s_b[i] = 0ull;
        __syncthreads();
        bitonic_desc(s_b, P);
        // sorted position j holds rank k - w + j: j < w stays kept unless pair w-1-j
        // swaps, j >= w becomes kept iff pair j-w swaps
        for (int j = threadIdx.x; j < 2 * w; j += kThreads) {
            const int i = j < w ? w - 1 - j : j - w;
            const bool swapped = swap_uniform(sa.seed, (uint64_t)i) < sa.prob;
            if (j < w ? !swapped : swapped) s_key[0xffffffffu - (uint32_t)(s_b[j] & 0xffffffffull)] = KEPT;
        }
        __syncthreads();
        pf = PRUNED;  // kept = mark > PRUNED, no ties taken
        shift = 0;
        r = 0;
    }
    if constexpr (STOCH) {  // kept blocks before this CTA's flat range (marks)
        uint32_t na = 0;
        for (int f = threadIdx.x; f < f0; f += kThreads) na += s_key[f] > pf;
        uint64_t tot;
        block_excl_scan((uint64_t)na << 32, s_warp, tot);
        pre = tot;
    }
    scan_and_index(p, f0, f1, pre, pf, shift, r, s_warp, s_key);
    if (p.pdl_trig) pdl_trigger();
    pack_kept<ES, B>(p, u0, u1);
}

// Pack with a threshold chosen elsewhere (cross-rank global top-k, select_global.cu):
// keep keys (>> shift) > T and the first `r` keys == T in flat order.  The block
// sums of squares are already in the workspace (bsr_select_hist level 0).
template <int ES, int B>
__global__ void __launch_bounds__(kThreads, (B >= 16) ? 1 : 2) prune_apply_kernel(PruneParams p, uint32_t T, int shift, uint32_t r) {
    using G_ = Geo<ES, B>;
    __shared__ uint64_t s_warp[32];
    __shared__ uint32_t s_sel[4];
    if (p.gstate) {  // threshold, digit shift, tie quota and kept count decided on the device (GS_* words)
        T = (uint32_t)p.gstate[1];
        shift = (int)p.gstate[2];
        r = (uint32_t)p.gstate[6];
        p.k = (int64_t)p.gstate[7];
    }
    const int64_t u0 = (int64_t)blockIdx.x * p.units / gridDim.x;
    const int64_t u1 = (int64_t)(blockIdx.x + 1) * p.units / gridDim.x;
    auto flat_start = [&](int64_t u) -> int64_t {
        return u >= p.units ? p.N : (u / p.upr) * p.nbc + (u % p.upr) * G_::G;
    };
    const int64_t f0 = flat_start(u0), f1 = flat_start(u1);
    uint32_t na = 0, nt = 0;
    for (int64_t f = f0 + threadIdx.x; f < f1; f += kThreads) {
        const uint32_t kk = key_of(p.sumsq[f]) >> shift;
        na += kk > T;
        nt += kk == T;
    }
    {
        uint64_t tot;
        block_excl_scan(((uint64_t)na << 32) | nt, s_warp, tot);
        if (threadIdx.x == 0) {
            p.cta_cnt[2 * blockIdx.x] = (uint32_t)(tot >> 32);
            p.cta_cnt[2 * blockIdx.x + 1] = (uint32_t)tot;
        }
    }
    grid_barrier(p.bar, 0);
    uint64_t pre = 0;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += kThreads)
        pre += ((uint64_t)__ldcg(p.cta_cnt + 2 * c) << 32) | __ldcg(p.cta_cnt + 2 * c + 1);
    {
        uint64_t tot;
        block_excl_scan(pre, s_warp, tot);
        pre = tot;
    }
    if (threadIdx.x == 0) {  // self-cleaning barrier counter (see prune_kernel)
        __threadfence();
        s_sel[3] = atomicAdd(p.bar + 32, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_sel[3] && threadIdx.x == 0) {
        __threadfence();
        p.bar[0] = 0;
        p.bar[32] = 0;
    }
    scan_and_index(p, f0, f1, pre, T, shift, r, s_warp);
    pack_kept<ES, B>(p, u0, u1);
}

// k == N: every block kept, no norms needed -- a single copy pass.
template <int ES, int B>
__global__ void __launch_bounds__(256) keep_all_kernel(PruneParams p) {
    using G_ = Geo<ES, B>;
    using V = typename G_::V;
    const int lane = threadIdx.x & 31;
    const int j = lane / G_::LPB, sub = lane % G_::LPB;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = wg; u < p.units; u += nwg) {
        const int64_t I = u / p.upr, J = (u % p.upr) * G_::G + j;
        if (J >= p.nbc) continue;
        const int64_t f = I * p.nbc + J;
        if (sub == 0) {
            p.colidx[f] = (int32_t)J;
            if (J == 0) p.rowptr[I] = (int32_t)f;
            if (I == p.nbr - 1 && J == p.nbc - 1) p.rowptr[p.nbr] = (int32_t)p.N;
        }
        const int64_t rs = p.K / G_::EPV;
        const V *src = reinterpret_cast<const V *>(p.X) + (I * B) * rs + (J * B) / G_::EPV + sub;
        V *dst = reinterpret_cast<V *>(p.values) + f * (B * B / G_::EPV) + sub;
#pragma unroll
        for (int r0 = 0; r0 < B; r0 += G_::R) {
            V v[G_::R];
#pragma unroll
            for (int rr = 0; rr < G_::R; ++rr) v[rr] = ld_stream(src + (r0 + rr) * rs);
#pragma unroll
            for (int rr = 0; rr < G_::R; ++rr) __stcs(dst + (r0 + rr) * G_::LPB, v[rr]);
        }
    }
}

// Producer fusion: X = act(Z) written once, and the block sums
// of squares of the written X accumulated in the same pass -- same per-element
// order and reduction tree as block_sumsq_warp, so the sums are bit-identical to
// the ones prune_kernel's phase 1 would compute from X.  A later prune with
// `presummed` skips phase 1's read of X.  act: 0 = identity, 1 = GELU (tanh form).
__device__ __forceinline__ float act_fn(float z, int act) {
    if (act == 1) {
        const float u = 0.7978845608028654f * fmaf(0.044715f * z, z * z, z);
        return 0.5f * z * (1.0f + tanhf(u));
    }
    return z;
}

template <int ES, int B>
__global__ void __launch_bounds__(256) act_sumsq_kernel(const void *Z, void *X, int64_t K, int64_t nbc, int64_t units,
                                                        int64_t upr, int act, float *sumsq) {
    using G_ = Geo<ES, B>;
    using V = typename G_::V;
    const int lane = threadIdx.x & 31;
    const int j = lane / G_::LPB, sub = lane % G_::LPB;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = wg; u < units; u += nwg) {
        const int64_t I = u / upr, J = (u % upr) * G_::G + j;
        const bool valid = J < nbc;
        float acc[G_::EPV];
#pragma unroll
        for (int e = 0; e < G_::EPV; ++e) acc[e] = 0.f;
        if (valid) {
            const int64_t rs = K / G_::EPV;
            const V *src = reinterpret_cast<const V *>(Z) + (I * B) * rs + (J * B) / G_::EPV + sub;
            V *dst = reinterpret_cast<V *>(X) + (I * B) * rs + (J * B) / G_::EPV + sub;
#pragma unroll
            for (int r0 = 0; r0 < B; r0 += G_::R) {
                V v[G_::R];
#pragma unroll
                for (int rr = 0; rr < G_::R; ++rr) v[rr] = ld_stream(src + (r0 + rr) * rs);
#pragma unroll
                for (int rr = 0; rr < G_::R; ++rr) {
                    uint32_t w[G_::VB / 4];
#pragma unroll
                    for (int q = 0; q < G_::VB / 4; ++q) w[q] = word(v[rr], q);
#pragma unroll
                    for (int e = 0; e < G_::EPV; ++e) {
                        float x = act_fn(elem<ES>(v[rr], e), act);
                        if constexpr (ES == 4) {
                            w[e] = __float_as_uint(x);
                        } else {
                            const uint32_t h = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x));
                            x = __uint_as_float(h << 16);
                            w[e >> 1] = (e & 1) ? ((w[e >> 1] & 0xffffu) | (h << 16)) : ((w[e >> 1] & 0xffff0000u) | h);
                        }
                        acc[e] = fmaf(x, x, acc[e]);
                    }
                    V o;
                    if constexpr (G_::VB == 16) o = make_uint4(w[0], w[1], w[2], w[3]);
                    else if constexpr (G_::VB == 8) o = make_uint2(w[0], w[1]);
                    else o = w[0];
                    dst[(r0 + rr) * rs] = o;
                }
            }
        }
#pragma unroll
        for (int w = 1; w < G_::EPV; w <<= 1)
#pragma unroll
            for (int e = 0; e < G_::EPV; e += 2 * w) acc[e] = acc[e] + acc[e + w];
        float s = acc[0];
#pragma unroll
        for (int off = 1; off < G_::LPB; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (valid && sub == 0) sumsq[I * nbc + J] = s;
    }
}

// Test hook: phase 1 only, written to a caller buffer.
template <int ES, int B>
__global__ void __launch_bounds__(256) sumsq_kernel(const void *X, int64_t K, int64_t nbc, int64_t units,
                                                    int64_t upr, float *sumsq) {
    using G_ = Geo<ES, B>;
    const int lane = threadIdx.x & 31;
    const int j = lane / G_::LPB, sub = lane % G_::LPB;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t u = wg; u < units; u += nwg) {
        const int64_t I = u / upr, J = (u % upr) * G_::G + j;
        const bool valid = J < nbc;
        float s = block_sumsq_warp<ES, B>(X, K, I, J, sub, valid);
        if (valid && sub == 0) sumsq[I * nbc + J] = s;
    }
}

// Warps per decompress unit (each copying B / parts rows): more warps in flight for
// the wide blocks, whose units are 16 KB (fp32) of output each.
template <int B>
constexpr int kDecompRowParts = B >= 32 ? 2 : 1;

// BSR -> dense: every output row segment written once (zeros or the block).
// The warp's unit covers G consecutive block columns of one block row; the
// row's stored columns are scanned 32 at a time with one coalesced colidx load
// per chunk (instead of a dependent binary search per lane), each hit parks its
// stored index in a per-warp shared-memory slot.  Rows are copied RD at a time
// (16 in flight per lane for the wide blocks).
template <int ES, int B>
__global__ void __launch_bounds__(256) decompress_kernel(const int32_t *__restrict__ rowptr,
                                                         const int32_t *__restrict__ colidx,
                                                         const void *__restrict__ values, int64_t K, int64_t nbc,
                                                         int64_t units, int64_t upr, void *__restrict__ Xout) {
    pdl_wait();  // launched with PDL: no global access before the predecessor completes
    using G_ = Geo<ES, B>;
    using V = typename G_::V;
    constexpr int RD = (B < 16) ? B : 16;
    constexpr int RS = kDecompRowParts<B>;  // warps per unit, each copying B / RS rows
    constexpr int BR = B / RS;
    __shared__ int s_pos[256 / 32][G_::G];  // B >= 16 lookup slots
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int j = lane / G_::LPB, sub = lane % G_::LPB;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwg = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t task = wg; task < units * RS; task += nwg) {
        const int64_t u = task / RS;
        const int part = (int)(task - u * RS);
        const int64_t I = u / upr;
        const int Jb = (int)((u % upr) * G_::G);
        const int64_t J = Jb + j;
        int lo;
        if constexpr (B >= 16) {
            if (lane < G_::G) s_pos[wid][lane] = -1;
            __syncwarp();
            const int rb = __ldg(rowptr + I), re = __ldg(rowptr + I + 1);
            // entries with col >= Jb start no earlier than re - (nbc - Jb) (columns are unique and ascending)
            for (int c = max(rb, re - (int)(nbc - Jb)); c < re; c += 32) {
                const int idx = c + lane;
                const int col = idx < re ? __ldg(colidx + idx) : 0x7fffffff;
                if (col >= Jb && col < Jb + G_::G) s_pos[wid][col - Jb] = idx;
                if (__shfl_sync(0xffffffffu, col, 31) >= Jb + G_::G) break;  // colidx ascending: past the unit
            }
            __syncwarp();
            lo = s_pos[wid][j];
            __syncwarp();  // slots are re-initialised by the next unit
        } else {
            // small blocks: G = 16..32 columns per unit, one per lane group -- a
            // per-lane binary search keeps the lookups independent (measured
            // faster than the chunk scan for b = 4 at 1-4 GiB, profiles/r01_sweep_v7)
            int l = __ldg(rowptr + I), h = __ldg(rowptr + I + 1);
            const int he = h;
            while (l < h) {
                const int mid = (l + h) >> 1;
                if (__ldg(colidx + mid) < J) l = mid + 1; else h = mid;
            }
            lo = (J < nbc && l < he && __ldg(colidx + l) == J) ? l : -1;
        }
        if (J >= nbc) continue;
        const int64_t rs = K / G_::EPV;
        V *dst = reinterpret_cast<V *>(Xout) + (I * B + part * BR) * rs + (J * B) / G_::EPV + sub;
        if (lo >= 0) {
            const V *src = reinterpret_cast<const V *>(values) + (int64_t)lo * (B * B / G_::EPV) + part * BR * G_::LPB + sub;
            constexpr int RDP = RD < BR ? RD : BR;
#pragma unroll
            for (int r0 = 0; r0 < BR; r0 += RDP) {
                V v[RDP];
#pragma unroll
                for (int rr = 0; rr < RDP; ++rr) v[rr] = ld_stream(src + (r0 + rr) * G_::LPB);
#pragma unroll
                for (int rr = 0; rr < RDP; ++rr) __stcs(dst + (r0 + rr) * rs, v[rr]);
            }
        } else {
            V z{};
#pragma unroll 8
            for (int r = 0; r < BR; ++r) __stcs(dst + r * rs, z);
        }
    }
}

// ------------------------------------------------------------------ host side
static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

PruneWs prune_ws_layout(int64_t N) {
    PruneWs w;
    size_t o = 0;
    w.hdr = o;      o += align256(64 * 4);
    w.hist1 = o;    o += align256(kH1 * 4);
    w.hist2 = o;    o += align256(kH2 * 4);
    w.hist3 = o;    o += align256(kH3 * 4);
    w.sstate = o;   o += align256(2 * 8 * 4 + 4);  // bsr_prune_stochastic: [2][ST_WORDS] + boundary counter
    w.shist = o;    o += align256(2 * kH2 * 4);    // bsr_prune_stochastic: refinement histograms
    w.zero_bytes = o;
    w.cta_cnt = o;  o += align256(2 * kMaxGrid * 4);
    w.sumsq = o;    o += align256((size_t)N * 4);
    w.slot = o;     o += align256((size_t)N * 4);
    w.cand = o;     o += align256((size_t)kCandMax * 8);
    w.total = o;
    return w;
}

template <int ES, int B>
static int units_per_row(int64_t nbc) {
    return (int)((nbc + Geo<ES, B>::G - 1) / Geo<ES, B>::G);
}

static int num_sms() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// Dynamic shared memory of the small-N finishing kernel: keys, first-digit histogram, then the candidate list or (STOCH) the boundary list.
static size_t small_smem_bytes(int64_t N, int64_t units, int64_t w) {
    size_t tail = (size_t)kSmallCand * 8;
    if (w > 0) {
        int64_t P = 1;
        while (P < 2 * w) P <<= 1;
        tail = std::max(tail, (size_t)P * 8);
    }
    (void)units;
    return (size_t)((N + 3) & ~int64_t(3)) * 4 + (size_t)kH1 * 4 + tail;
}
constexpr size_t kSmallSmemMax = 216 * 1024;  // + the kernel's static shared memory stays under 227 KB

// The small-N pair: sums (no global histogram) -> finishing kernel, chained with PDL.
template <int ES, int B, bool STOCH>
static cudaError_t launch_small_t(PruneParams p, StochArgs sa, cudaStream_t stream) {
    p.hist1 = nullptr;  // the finishing CTAs count the first digit themselves
    const size_t smem = small_smem_bytes(p.N, p.units, STOCH ? sa.w : 0);
    cudaError_t e = cudaFuncSetAttribute(prune_finish_kernel<ES, B, STOCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t per = kThreads / 32;  // one unit per warp
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((p.units + per - 1) / per, (int64_t)num_sms()));
    e = launch_pdl(pdl_flags() & 128, prune_sums_kernel<ES, B>, dim3((unsigned)grid), dim3(kThreads), 0, stream, p);
    if (e != cudaSuccess) return e;
    count_launch();
    e = launch_pdl(true, prune_finish_kernel<ES, B, STOCH>, dim3((unsigned)grid), dim3(kThreads), smem, stream, p, sa);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <int ES, int B>
static cudaError_t launch_prune_t(PruneParams p, cudaStream_t stream, void *ws, const PruneWs &w) {
    if (p.k == 0) {
        return cudaMemsetAsync(p.rowptr, 0, (size_t)(p.nbr + 1) * 4, stream);
    }
    if (p.k == p.N) {
        int64_t blocks = std::min<int64_t>((p.units + 7) / 8, 148 * 16);
        keep_all_kernel<ES, B><<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, stream>>>(p);
        count_launch();
        return cudaGetLastError();
    }
    // (no per-launch memset: the kernels leave their workspace header zeroed, see above)
    cudaError_t e = cudaSuccess;
    if (p.N <= kSmallN && small_smem_bytes(p.N, p.units, 0) <= kSmallSmemMax)
        return launch_small_t<ES, B, false>(p, StochArgs{0, 0.0, 0ull}, stream);
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, prune_kernel<ES, B>, kThreads, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorLaunchOutOfResources;
    int64_t grid = (int64_t)occ * num_sms();
    grid = std::min<int64_t>(grid, kMaxGrid);
    grid = std::min<int64_t>(grid, std::max<int64_t>(1, (p.units + kThreads / 32 - 1) / (kThreads / 32)));
    void *args[] = {&p};
    count_launch();
    return cudaLaunchCooperativeKernel((const void *)prune_kernel<ES, B>, dim3((unsigned)grid), dim3(kThreads),
                                       args, 0, stream);
}

#define BSRP_DISPATCH_B(ES, b, CALL)     \
    switch (b) {                         \
        case 4: return CALL(ES, 4);      \
        case 8: return CALL(ES, 8);      \
        case 16: return CALL(ES, 16);    \
        case 32: return CALL(ES, 32);    \
        case 64: return CALL(ES, 64);    \
        default: return cudaErrorInvalidValue; \
    }

cudaError_t launch_prune(const void *X, int64_t M, int64_t K, int b, int es, int64_t k, int32_t *rowptr,
                         int32_t *colidx, void *values, void *ws, cudaStream_t stream, int presummed) {
    PruneParams p{};
    p.presummed = presummed;
    p.pdl_trig = pdl_flags() & 1;
    p.X = X;
    p.K = K;
    p.nbr = M / b;
    p.nbc = K / b;
    p.N = p.nbr * p.nbc;
    p.k = k;
    p.rowptr = rowptr;
    p.colidx = colidx;
    p.values = values;
    const PruneWs w = prune_ws_layout(p.N);
    char *base = static_cast<char *>(ws);
    p.bar = reinterpret_cast<uint32_t *>(base + w.hdr);
    p.hist1 = reinterpret_cast<uint32_t *>(base + w.hist1);
    p.hist2 = reinterpret_cast<uint32_t *>(base + w.hist2);
    p.hist3 = reinterpret_cast<uint32_t *>(base + w.hist3);
    p.cta_cnt = reinterpret_cast<uint32_t *>(base + w.cta_cnt);
    p.sumsq = reinterpret_cast<float *>(base + w.sumsq);
    p.slot = reinterpret_cast<int32_t *>(base + w.slot);
    p.cand = reinterpret_cast<uint2 *>(base + w.cand);
#define CALL(ES_, B_) (p.upr = units_per_row<ES_, B_>(p.nbc), p.units = p.nbr * p.upr, \
                       launch_prune_t<ES_, B_>(p, stream, ws, w))
    if (es == 4) {
        BSRP_DISPATCH_B(4, b, CALL)
    } else {
        BSRP_DISPATCH_B(2, b, CALL)
    }
#undef CALL
}

cudaError_t launch_act_sumsq(const void *Z, void *X, int64_t M, int64_t K, int b, int es, int act, void *ws,
                             cudaStream_t stream) {
    const int64_t nbr = M / b, nbc = K / b;
    float *sumsq = reinterpret_cast<float *>(static_cast<char *>(ws) + prune_ws_layout(nbr * nbc).sumsq);
#define CALL(ES_, B_) ([&]() {                                                                        \
        int64_t upr = units_per_row<ES_, B_>(nbc), units = nbr * upr;                               \
        int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((units + 7) / 8, 148 * 16));           \
        act_sumsq_kernel<ES_, B_><<<(unsigned)blocks, 256, 0, stream>>>(Z, X, K, nbc, units, upr, act, sumsq); \
        count_launch();                                                                             \
        return cudaGetLastError();                                                                  \
    }())
    if (es == 4) {
        BSRP_DISPATCH_B(4, b, CALL)
    } else {
        BSRP_DISPATCH_B(2, b, CALL)
    }
#undef CALL
}

cudaError_t launch_block_sumsq(const void *X, int64_t M, int64_t K, int b, int es, float *sumsq,
                               cudaStream_t stream) {
    const int64_t nbr = M / b, nbc = K / b;
#define CALL(ES_, B_) ([&]() {                                                              \
        int64_t upr = units_per_row<ES_, B_>(nbc), units = nbr * upr;                     \
        int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((units + 7) / 8, 148 * 16)); \
        sumsq_kernel<ES_, B_><<<(unsigned)blocks, 256, 0, stream>>>(X, K, nbc, units, upr, sumsq); \
        count_launch();                                                                   \
        return cudaGetLastError();                                                        \
    }())
    if (es == 4) {
        BSRP_DISPATCH_B(4, b, CALL)
    } else {
        BSRP_DISPATCH_B(2, b, CALL)
    }
#undef CALL
}

cudaError_t launch_decompress(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t M,
                              int64_t K, int b, int es, void *Xout, cudaStream_t stream) {
    const int64_t nbr = M / b, nbc = K / b;
#define CALL(ES_, B_) ([&]() {                                                                   \
        int64_t upr = units_per_row<ES_, B_>(nbc), units = nbr * upr;                          \
        int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((units * kDecompRowParts<B_> + 7) / 8, 148 * 16)); \
        cudaError_t e_ = launch_pdl(pdl_flags() & 64, decompress_kernel<ES_, B_>, dim3((unsigned)blocks), dim3(256), 0, stream, \
                                    rowptr, colidx, values, K, nbc, units, upr, Xout);                    \
        count_launch();                                                                        \
        return e_ != cudaSuccess ? e_ : cudaGetLastError();                                    \
    }())
    if (es == 4) {
        BSRP_DISPATCH_B(4, b, CALL)
    } else {
        BSRP_DISPATCH_B(2, b, CALL)
    }
#undef CALL
}

// Structural check of a BSR (bsr_validate): block row r is bad if rowptr[0] != 0
// (r = 0), rowptr decreases at r, rowptr[nbr] != nnzb (r = nbr - 1), or its colidx
// entries are not strictly ascending or not in [0, nbc).  bad = the lowest bad row.
__global__ void validate_init_kernel(int32_t *bad) { *bad = 0x7fffffff; }
__global__ void __launch_bounds__(256) validate_kernel(const int32_t *__restrict__ rowptr,
                                                       const int32_t *__restrict__ colidx, int64_t nbr, int64_t nbc,
                                                       int64_t nnzb, int32_t *bad) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nbr; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = rowptr[r], z = rowptr[r + 1];
        bool ok = a <= z && a >= 0 && z <= nnzb;
        if (r == 0) ok = ok && a == 0;
        if (r == nbr - 1) ok = ok && z == nnzb;
        if (ok) {
            int32_t prev = -1;
            for (int32_t e = a; e < z; ++e) {
                const int32_t c = colidx[e];
                if (c <= prev || c >= nbc) {
                    ok = false;
                    break;
                }
                prev = c;
            }
        }
        if (!ok) atomicMin(bad, (int32_t)r);
    }
}
__global__ void validate_finish_kernel(int32_t *bad) {
    if (*bad == 0x7fffffff) *bad = -1;
}

cudaError_t launch_validate(const int32_t *rowptr, const int32_t *colidx, int64_t nbr, int64_t nbc, int64_t nnzb,
                            int32_t *bad, cudaStream_t stream) {
    validate_init_kernel<<<1, 1, 0, stream>>>(bad);
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nbr + 255) / 256, (int64_t)num_sms() * 8));
    validate_kernel<<<g, 256, 0, stream>>>(rowptr, colidx, nbr, nbc, nnzb, bad);
    validate_finish_kernel<<<1, 1, 0, stream>>>(bad);
    count_launch(3);
    return cudaGetLastError();
}

cudaError_t launch_prune_threshold(const void *X, int64_t M, int64_t K, int b, int es, uint32_t T, int shift,
                                   uint32_t tie_take, int64_t k, int32_t *rowptr, int32_t *colidx, void *values,
                                   void *ws, cudaStream_t stream, const uint64_t *gstate) {
    PruneParams p{};
    p.gstate = reinterpret_cast<const unsigned long long *>(gstate);
    p.X = X;
    p.K = K;
    p.nbr = M / b;
    p.nbc = K / b;
    p.N = p.nbr * p.nbc;
    p.k = k;
    p.rowptr = rowptr;
    p.colidx = colidx;
    p.values = values;
    if (k == 0 && !gstate) return cudaMemsetAsync(rowptr, 0, (size_t)(p.nbr + 1) * 4, stream);
    const PruneWs w = prune_ws_layout(p.N);
    char *base = static_cast<char *>(ws);
    p.bar = reinterpret_cast<uint32_t *>(base + w.hdr);
    p.cta_cnt = reinterpret_cast<uint32_t *>(base + w.cta_cnt);
    p.sumsq = reinterpret_cast<float *>(base + w.sumsq);
    p.slot = reinterpret_cast<int32_t *>(base + w.slot);
#define CALL(ES_, B_) ([&]() -> cudaError_t {                                                                    \
        p.upr = units_per_row<ES_, B_>(p.nbc);                                                                  \
        p.units = p.nbr * p.upr;                                                                                \
        int occ = 0;                                                                                            \
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, prune_apply_kernel<ES_, B_>, kThreads, 0); \
        if (e != cudaSuccess) return e;                                                                         \
        if (occ < 1) return cudaErrorLaunchOutOfResources;                                                      \
        int64_t grid = std::min<int64_t>((int64_t)occ * num_sms(), kMaxGrid);                                   \
        grid = std::min<int64_t>(grid, std::max<int64_t>(1, (p.units + kThreads / 32 - 1) / (kThreads / 32)));   \
        void *args[] = {&p, &T, &shift, &tie_take};                                                             \
        count_launch();                                                                                         \
        return cudaLaunchCooperativeKernel((const void *)prune_apply_kernel<ES_, B_>, dim3((unsigned)grid),      \
                                           dim3(kThreads), args, 0, stream);                                    \
    }())
    if (es == 4) {
        BSRP_DISPATCH_B(4, b, CALL)
    } else {
        BSRP_DISPATCH_B(2, b, CALL)
    }
#undef CALL
}

// ---- stochastic boundary swapping (DESIGN reading R19) --------
// "randomly swapping blocks near the top-k threshold, resulting in some blocks
// above the threshold being pruned anyway, and vice-versa below threshold"
// (P:L661-666).  Ranks follow the deterministic order (key desc, flat index asc);
// with A = k - w and B = k + w (w = min(window, k, N - k) > 0):
//   ranks [0, A)      kept,
//   ranks [A, B)      the boundary: pair i (rank k-1-i, rank k+i) swaps iff
//                     u_i < p, u_i = splitmix64(seed, i) as a 53-bit uniform,
//   ranks [B, N)      pruned.
// While every CTA can hold all keys and the boundary list in shared memory, the
// small-N pair (prune_sums_kernel + prune_finish_kernel<STOCH = true>) does it in
// two launches.  Beyond that (stream order, 9 launches, graph-capturable):
//   prune_sums_kernel  block sums + digit-0 histogram (shared with bsr_prune)
//   stoch_update x3 / stoch_hist x2   radix select of ranks A and B together
//   stoch_mark (coop)  flat-order tie scan: slot[f] = 1 for ranks < A, the
//                      2w boundary blocks appended as (key, flat index)
//   stoch_swap (1 CTA) bitonic sort of the boundary by rank, the swaps
//   stoch_pack (coop)  flat-order scan of the final marks, rowptr/colidx, copy
enum { ST_T = 0, ST_SHIFT = 1, ST_R = 2, ST_ABOVE = 3, ST_DONE = 4, ST_TGT = 5, ST_WORDS = 8 };

StochWs stoch_ws_layout(int64_t N) {
    StochWs w;
    w.base = prune_ws_layout(N);
    size_t o = w.base.total;
    w.cta2 = o;   o += align256(2 * kMaxGrid * 4);
    w.blist = o;  o += align256(2 * kStochMaxWindow * 8);
    w.total = o;
    return w;
}

// One CTA: resolve the next key digit of both selections (targets A, B) from the
// histogram, then zero the histogram (self-cleaning workspace).
__global__ void __launch_bounds__(kThreads) stoch_update_kernel(int level, uint32_t *hist, uint32_t *st,
                                                                int64_t tA, int64_t tB) {
    __shared__ uint64_t s_warp[32];
    __shared__ uint32_t s_sel[4];
    const int nb = level == 0 ? kH1 : level == 1 ? kH2 : kH3;
    const int w = level == 0 ? 12 : level == 1 ? 10 : 9;
    for (int t = 0; t < 2; ++t) {
        uint32_t *S = st + t * ST_WORDS;
        if (level == 0) {
            const uint32_t tgt = (uint32_t)(t == 0 ? tA : tB);
            if (tgt == 0) {  // empty selection: a prefix no key reaches, no ties
                if (threadIdx.x == 0) {
                    S[ST_T] = 0xffffffffu; S[ST_SHIFT] = 0; S[ST_R] = 0; S[ST_ABOVE] = 0; S[ST_DONE] = 1;
                    S[ST_TGT] = 0;
                }
                continue;
            }
            select_bin(hist, nb, tgt, s_warp, s_sel);
            if (threadIdx.x == 0) {
                S[ST_T] = s_sel[0]; S[ST_SHIFT] = 19; S[ST_ABOVE] = s_sel[1]; S[ST_R] = tgt - s_sel[1];
                S[ST_DONE] = tgt - s_sel[1] >= s_sel[2];
                S[ST_TGT] = tgt;
            }
        } else {
            const uint32_t done = __ldcg(S + ST_DONE), r = __ldcg(S + ST_R);
            if (done) continue;
            select_bin(hist + t * kH2, nb, r, s_warp, s_sel);
            if (threadIdx.x == 0) {
                const uint32_t above = S[ST_ABOVE] + s_sel[1];
                S[ST_T] = (S[ST_T] << w) | s_sel[0];
                S[ST_SHIFT] -= w;
                S[ST_ABOVE] = above;
                S[ST_R] = S[ST_TGT] - above;
                S[ST_DONE] = (S[ST_TGT] - above >= s_sel[2]) || level == 2;
            }
        }
        __syncthreads();
    }
    __syncthreads();
    const int nz = level == 0 ? kH1 : 2 * kH2;
    for (int i = threadIdx.x; i < nz; i += kThreads) hist[i] = 0;
}

// Histogram of the next digit of the keys matching each unresolved selection's prefix.
__global__ void __launch_bounds__(kThreads) stoch_hist_kernel(int level, const float *__restrict__ sumsq, int64_t N,
                                                              const uint32_t *__restrict__ st, uint32_t *hist) {
    __shared__ uint32_t s_h[2][kH2];
    const int nb = level == 1 ? kH2 : kH3, nshift = level == 1 ? 9 : 0;
    const int lane = threadIdx.x & 31;
    bool act[2];
    uint32_t T[2], sh[2];
    for (int t = 0; t < 2; ++t) {
        act[t] = st[t * ST_WORDS + ST_DONE] == 0;
        T[t] = st[t * ST_WORDS + ST_T];
        sh[t] = st[t * ST_WORDS + ST_SHIFT];
    }
    for (int i = threadIdx.x; i < 2 * kH2; i += kThreads) (&s_h[0][0])[i] = 0;
    __syncthreads();
    if (act[0] || act[1])
        for (int64_t fb = (int64_t)blockIdx.x * kThreads; fb < N; fb += (int64_t)gridDim.x * kThreads) {
            const int64_t f = fb + threadIdx.x;
            const uint32_t key = f < N ? key_of(__ldcg(sumsq + f)) : 0u;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const bool in = act[t] && f < N && (key >> sh[t]) == T[t];
                const uint32_t bin = (key >> nshift) & (uint32_t)(nb - 1);
                const uint32_t im = __ballot_sync(0xffffffffu, in);
                if (!im) continue;
                const int l0 = __ffs(im) - 1;
                const uint32_t b0 = __shfl_sync(0xffffffffu, bin, l0);
                if (__all_sync(0xffffffffu, !in || bin == b0)) {  // a warp of ties adds once
                    if (lane == l0) atomicAdd(&s_h[t][b0], (uint32_t)__popc(im));
                } else if (in) {
                    atomicAdd(&s_h[t][bin], 1u);
                }
            }
        }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * kH2; i += kThreads) {
        const uint32_t v = (&s_h[0][0])[i];
        if (v) atomicAdd(hist + i, v);
    }
}

struct StochParams {
    const float *sumsq;
    int64_t N;
    int32_t *slot;           // out: 1 for ranks < A, else 0
    const uint32_t *st;
    uint32_t *bar, *cta2;
    uint32_t *bcount, *shist;
    unsigned long long *blist;  // (key << 32) | (0xffffffff - f): descending order = rank order
};

// Cooperative: per-CTA tie counts of both selections, grid barrier, flat-order
// scan (the same tie rule as scan_and_index: the first r ties in flat order).
__global__ void __launch_bounds__(kThreads) stoch_mark_kernel(StochParams q) {
    __shared__ uint64_t s_warp[32];
    __shared__ uint32_t s_flag;
    const int lane = threadIdx.x & 31;
    const int64_t f0 = (int64_t)blockIdx.x * q.N / gridDim.x, f1 = (int64_t)(blockIdx.x + 1) * q.N / gridDim.x;
    const uint32_t TA = q.st[ST_T], shA = q.st[ST_SHIFT], rA = q.st[ST_R];
    const uint32_t TB = q.st[ST_WORDS + ST_T], shB = q.st[ST_WORDS + ST_SHIFT], rB = q.st[ST_WORDS + ST_R];
    uint32_t ta = 0, tb = 0;
    for (int64_t f = f0 + threadIdx.x; f < f1; f += kThreads) {
        const uint32_t key = key_of(q.sumsq[f]);
        ta += (key >> shA) == TA;
        tb += (key >> shB) == TB;
    }
    {
        uint64_t tot;
        block_excl_scan(((uint64_t)ta << 32) | tb, s_warp, tot);
        if (threadIdx.x == 0) {
            q.cta2[2 * blockIdx.x] = (uint32_t)(tot >> 32);
            q.cta2[2 * blockIdx.x + 1] = (uint32_t)tot;
        }
    }
    grid_barrier(q.bar, 0);
    uint64_t pre = 0;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += kThreads)
        pre += ((uint64_t)__ldcg(q.cta2 + 2 * c) << 32) | __ldcg(q.cta2 + 2 * c + 1);
    {
        uint64_t tot;
        block_excl_scan(pre, s_warp, tot);
        pre = tot;
    }
    if (threadIdx.x == 0) {  // self-cleaning barrier counter (see prune_apply_kernel)
        __threadfence();
        s_flag = atomicAdd(q.bar + 32, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_flag && threadIdx.x == 0) {
        __threadfence();
        q.bar[0] = 0;
        q.bar[32] = 0;
    }
    uint32_t baseA = (uint32_t)(pre >> 32), baseB = (uint32_t)pre;
    for (int64_t fb = f0; fb < f1; fb += kThreads) {
        const int64_t f = fb + threadIdx.x;
        const bool in = f < f1;
        const uint32_t key = in ? key_of(q.sumsq[f]) : 0u;
        const uint32_t kA = key >> shA, kB = key >> shB;
        const uint32_t tA = in && kA == TA, tB = in && kB == TB;
        uint64_t tot;
        const uint64_t ex = block_excl_scan(((uint64_t)tA << 32) | tB, s_warp, tot);
        const uint32_t bA = baseA + (uint32_t)(ex >> 32), bB = baseB + (uint32_t)ex;
        const bool inA = in && (kA > TA || (tA && bA < rA));
        const bool inB = in && (kB > TB || (tB && bB < rB));
        const bool bnd = inB && !inA;
        if (in) q.slot[f] = inA ? 1 : 0;
        const uint32_t m = __ballot_sync(0xffffffffu, bnd);
        uint32_t pos = 0;
        if (m && lane == 0) pos = atomicAdd(q.bcount, (uint32_t)__popc(m));
        pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << lane) - 1u));
        if (bnd) {
            if (pos >= 2u * kStochMaxWindow) __trap();  // cannot happen: |ranks [A, B)| = 2w
            q.blist[pos] = ((unsigned long long)key << 32) | (0xffffffffu - (uint32_t)f);
        }
        baseA += (uint32_t)(tot >> 32);
        baseB += (uint32_t)tot;
    }
}

// One CTA: sort the 2w boundary blocks by rank (bitonic, descending composite
// key), apply the swaps, mark the kept ones, reset the boundary counter.
__global__ void __launch_bounds__(1024) stoch_swap_kernel(unsigned long long *__restrict__ blist, uint32_t *bcount,
                                                          int32_t *__restrict__ slot, int w, double prob,
                                                          unsigned long long seed) {
    extern __shared__ unsigned long long s_b[];
    const int n = 2 * w;
    if (threadIdx.x == 0 && __ldcg(bcount) != (uint32_t)n) __trap();  // workspace not zero-filled
    int P = 1;
    while (P < n) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) s_b[i] = i < n ? __ldcg(blist + i) : 0ull;
    __syncthreads();
    if (threadIdx.x == 0) *bcount = 0;
    bitonic_desc(s_b, P);
    // sorted position j holds rank A + j: j < w is kept unless pair w-1-j swaps,
    // j >= w is kept iff pair j-w swaps
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const int i = j < w ? w - 1 - j : j - w;
        const bool swapped = swap_uniform(seed, (uint64_t)i) < prob;
        const bool keep = j < w ? !swapped : swapped;
        const uint32_t f = 0xffffffffu - (uint32_t)(s_b[j] & 0xffffffffull);
        if (keep) slot[f] = 1;
    }
}

// Cooperative: output slots of the marked blocks in flat order, rowptr, colidx, copy.
template <int ES, int B>
__global__ void __launch_bounds__(kThreads, (B >= 16) ? 1 : 2) stoch_pack_kernel(PruneParams p) {
    using G_ = Geo<ES, B>;
    __shared__ uint64_t s_warp[32];
    __shared__ uint32_t s_flag;
    const int64_t u0 = (int64_t)blockIdx.x * p.units / gridDim.x;
    const int64_t u1 = (int64_t)(blockIdx.x + 1) * p.units / gridDim.x;
    auto flat_start = [&](int64_t u) -> int64_t {
        return u >= p.units ? p.N : (u / p.upr) * p.nbc + (u % p.upr) * G_::G;
    };
    const int64_t f0 = flat_start(u0), f1 = flat_start(u1);
    uint32_t nk = 0;
    for (int64_t f = f0 + threadIdx.x; f < f1; f += kThreads) nk += p.slot[f] == 1;
    {
        uint64_t tot;
        block_excl_scan(nk, s_warp, tot);
        if (threadIdx.x == 0) p.cta_cnt[blockIdx.x] = (uint32_t)tot;
    }
    grid_barrier(p.bar, 0);
    uint64_t pre = 0;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += kThreads) pre += __ldcg(p.cta_cnt + c);
    {
        uint64_t tot;
        block_excl_scan(pre, s_warp, tot);
        pre = tot;
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_flag = atomicAdd(p.bar + 32, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_flag && threadIdx.x == 0) {
        __threadfence();
        p.bar[0] = 0;
        p.bar[32] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) p.rowptr[0] = 0;
    uint32_t base = (uint32_t)pre;
    for (int64_t fb = f0; fb < f1; fb += kThreads) {
        const int64_t f = fb + threadIdx.x;
        const bool in = f < f1;
        const uint32_t kp = in && p.slot[f] == 1;
        uint64_t tot;
        const uint32_t pos = base + (uint32_t)block_excl_scan(kp, s_warp, tot);
        if (in) {
            const bool kept = kp && pos < (uint64_t)p.k;
            const int64_t I = f / p.nbc, J = f - I * p.nbc;
            p.slot[f] = kept ? (int32_t)pos : -1;
            if (kept) p.colidx[pos] = (int32_t)J;
            if (J == p.nbc - 1) p.rowptr[I + 1] = (int32_t)(pos + kp);
        }
        base += (uint32_t)tot;
    }
    __syncthreads();
    pack_kept<ES, B>(p, u0, u1);
}

template <int ES, int B>
static cudaError_t launch_stoch_t(PruneParams p, StochParams q, int64_t wn, double prob,
                                  uint64_t seed, cudaStream_t stream) {
    // the two-kernel path while every CTA can hold all keys and the boundary list
    // (N up to ~43K keys: S12 fc2 at b = 16 included); the multi-kernel path beyond
    if (small_smem_bytes(p.N, p.units, wn) <= kSmallSmemMax)
        return launch_small_t<ES, B, true>(p, StochArgs{wn, prob, (unsigned long long)seed}, stream);
    const int sms = num_sms();
    const int64_t per = kThreads / 32;
    const int64_t sgrid = std::max<int64_t>(1, std::min<int64_t>((p.units + per - 1) / per, (int64_t)sms));
    cudaError_t e = launch_pdl(false, prune_sums_kernel<ES, B>, dim3((unsigned)sgrid), dim3(kThreads), 0, stream, p);
    if (e != cudaSuccess) return e;
    uint32_t *st = const_cast<uint32_t *>(q.st);
    uint32_t *shist = q.shist;
    const int64_t tA = p.k - wn, tB = p.k + wn;
    const int64_t hgrid = std::max<int64_t>(1, std::min<int64_t>((p.N + kThreads - 1) / kThreads, 2 * (int64_t)sms));
    stoch_update_kernel<<<1, kThreads, 0, stream>>>(0, p.hist1, st, tA, tB);
    for (int level = 1; level <= 2; ++level) {
        stoch_hist_kernel<<<(unsigned)hgrid, kThreads, 0, stream>>>(level, p.sumsq, p.N, q.st, shist);
        stoch_update_kernel<<<1, kThreads, 0, stream>>>(level, shist, st, tA, tB);
    }
    count_launch(6);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stoch_mark_kernel, kThreads, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorLaunchOutOfResources;
    int64_t mgrid = std::min<int64_t>((int64_t)occ * sms, kMaxGrid);
    mgrid = std::min<int64_t>(mgrid, std::max<int64_t>(1, (p.N + kThreads - 1) / kThreads));
    {
        void *args[] = {&q};
        e = cudaLaunchCooperativeKernel((const void *)stoch_mark_kernel, dim3((unsigned)mgrid), dim3(kThreads), args, 0,
                                        stream);
        count_launch();
        if (e != cudaSuccess) return e;
    }
    int P = 1;
    while (P < 2 * wn) P <<= 1;
    const size_t smem = (size_t)P * 8;
    e = cudaFuncSetAttribute(stoch_swap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    stoch_swap_kernel<<<1, 1024, smem, stream>>>(q.blist, q.bcount, p.slot, (int)wn, prob, (unsigned long long)seed);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stoch_pack_kernel<ES, B>, kThreads, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorLaunchOutOfResources;
    int64_t pgrid = std::min<int64_t>((int64_t)occ * sms, kMaxGrid);
    pgrid = std::min<int64_t>(pgrid, std::max<int64_t>(1, (p.units + per - 1) / per));
    void *args[] = {&p};
    count_launch();
    return cudaLaunchCooperativeKernel((const void *)stoch_pack_kernel<ES, B>, dim3((unsigned)pgrid), dim3(kThreads),
                                       args, 0, stream);
}

cudaError_t launch_prune_stochastic(const void *X, int64_t M, int64_t K, int b, int es, int64_t k, int64_t window,
                                    double prob, uint64_t seed, int32_t *rowptr, int32_t *colidx, void *values,
                                    void *ws, cudaStream_t stream) {
    const int64_t N = (M / b) * (K / b);
    const int64_t wn = std::min<int64_t>(window, std::min<int64_t>(k, N - k));
    if (wn <= 0) return launch_prune(X, M, K, b, es, k, rowptr, colidx, values, ws, stream, 0);
    if (wn > kStochMaxWindow) return cudaErrorInvalidValue;
    const StochWs w = stoch_ws_layout(N);
    char *base = static_cast<char *>(ws);
    PruneParams p{};
    p.X = X;
    p.K = K;
    p.nbr = M / b;
    p.nbc = K / b;
    p.N = N;
    p.k = k;
    p.rowptr = rowptr;
    p.colidx = colidx;
    p.values = values;
    p.bar = reinterpret_cast<uint32_t *>(base + w.base.hdr);
    p.hist1 = reinterpret_cast<uint32_t *>(base + w.base.hist1);
    p.cta_cnt = reinterpret_cast<uint32_t *>(base + w.base.cta_cnt);
    p.sumsq = reinterpret_cast<float *>(base + w.base.sumsq);
    p.slot = reinterpret_cast<int32_t *>(base + w.base.slot);
    StochParams q{};
    q.sumsq = p.sumsq;
    q.N = N;
    q.slot = p.slot;
    q.st = reinterpret_cast<uint32_t *>(base + w.base.sstate);
    q.bcount = reinterpret_cast<uint32_t *>(base + w.base.sstate) + 2 * ST_WORDS;
    q.bar = p.bar;
    q.cta2 = reinterpret_cast<uint32_t *>(base + w.cta2);
    q.blist = reinterpret_cast<unsigned long long *>(base + w.blist);
    q.shist = reinterpret_cast<uint32_t *>(base + w.base.shist);
#define CALL(ES_, B_) (p.upr = units_per_row<ES_, B_>(p.nbc), p.units = p.nbr * p.upr, \
                       launch_stoch_t<ES_, B_>(p, q, wn, prob, seed, stream))
    if (es == 4) {
        BSRP_DISPATCH_B(4, b, CALL)
    } else {
        BSRP_DISPATCH_B(2, b, CALL)
    }
#undef CALL
}

}  // namespace bsrp
