// prune_rows.cu -- the paper-faithful variant: 1 x b
// row-segment blocks (the Table II geometry) selected per sample
// ("Blocks are only compared locally, not among other activations in the
// mini-batch ... all activations in a mini-batch to have the same amount of
// zero and non-zero blocks").  X is M x K with M = samples x S rows;
// every sample keeps exactly k_s = nearest(keep * S * K / b) segments (R3), ties
// to the lower flat index within the sample (BJ rule).  One BSR with br = 1,
// bc = b over all rows: rowptr[M + 1], colidx[k], values[k][b].
//
//   rows_sumsq_kernel   fp32 sum of squares of every segment (fixed order: the
//                       segment's elements in index order), key = fp32 bits.
//   rows_select_kernel  one CTA per sample: exact radix select (8+8+8+7 bits,
//                       shared-memory histograms) of the sample's k_s-th key,
//                       then a flat-order scan gives each kept segment its slot
//                       s * k_s + rank; it writes colidx and rowptr.  No grid-wide
//                       step: the samples' offsets are known (every sample keeps k_s).
//   rows_pack_kernel    one warp per row over the whole GPU: the kept segments
//                       gathered from X into values (raw bits) -- the copy used to
//                       run inside the per-sample CTAs, latency-bound there.
//   rows_decompress_kernel  one warp per row: zeros, then the kept segments.
//   rows_wgrad_kernel   dW = X_bsr^T dY (fp32 FFMA, fixed order, deterministic):
//                       CTA = 128 kcols x 128 dY columns x a range of rows,
//                       16 rows per stage staged by cp.async (pruned segments
//                       zero-filled), 8 x 8 register tile per thread; split
//                       partials summed in split order.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace bsrp {
namespace rows {

constexpr int kThreads = 512;

__device__ __forceinline__ uint32_t key_of(float s) { return __float_as_uint(s) & 0x7fffffffu; }

template <int ES, int B>
__global__ void __launch_bounds__(256) rows_sumsq_kernel(const uint8_t *__restrict__ X, int64_t M, int64_t K,
                                                         float *__restrict__ sumsq) {
    const int64_t nbc = K / B, N = M * nbc;
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < N; f += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = f / nbc, J = f - r * nbc;
        const uint8_t *src = X + (r * K + J * B) * ES;
        float acc = 0.f;
        if constexpr (B * ES >= 16) {
#pragma unroll
            for (int q = 0; q < B * ES / 16; ++q) {
                const uint4 v = __ldg(reinterpret_cast<const uint4 *>(src) + q);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if constexpr (ES == 4) {
                        const float x = __uint_as_float(w[i]);
                        acc = fmaf(x, x, acc);
                    } else {
                        const float x0 = __uint_as_float(w[i] << 16), x1 = __uint_as_float(w[i] & 0xffff0000u);
                        acc = fmaf(x0, x0, acc);
                        acc = fmaf(x1, x1, acc);
                    }
                }
            }
        } else {  // bf16 b = 4: 8 bytes
            const uint2 v = __ldg(reinterpret_cast<const uint2 *>(src));
            const uint32_t w[2] = {v.x, v.y};
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const float x0 = __uint_as_float(w[i] << 16), x1 = __uint_as_float(w[i] & 0xffff0000u);
                acc = fmaf(x0, x0, acc);
                acc = fmaf(x1, x1, acc);
            }
        }
        sumsq[f] = acc;
    }
}

// Exclusive block scan of 64-bit values (blockDim.x == kThreads).
__device__ __forceinline__ uint64_t scan64(uint64_t v, uint64_t *s_warp, uint64_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = kThreads / 32;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint64_t t = lane < nw ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        s_warp[lane] = t;
    }
    __syncthreads();
    const uint64_t base = wid > 0 ? s_warp[wid - 1] : 0;
    total = s_warp[nw - 1];
    __syncthreads();
    return base + x - v;
}

// a sample's keys staged in shared memory when they fit: up to 208 KB (one CTA per
// SM; the S12 fc1 samples at every b and fc2 at b >= 8 fit; measured 12288 -> this:
// profiles/r02h/rows_*.json)
constexpr int kSmemKeys = 53248;

template <int ES, int B>
__global__ void __launch_bounds__(kThreads) rows_select_kernel(const uint8_t *__restrict__ X, int64_t K, int64_t S,
                                                               int64_t ks, const float *__restrict__ sumsq_g,
                                                               int32_t *__restrict__ rowptr,
                                                               int32_t *__restrict__ colidx,
                                                               uint8_t *__restrict__ values) {
    __shared__ uint32_t s_h[256];
    __shared__ uint64_t s_warp[32];
    __shared__ uint32_t s_sel[3];
    extern __shared__ float s_keys[];
    const int lane = threadIdx.x & 31;
    const int64_t nbc = K / B, ns = S * nbc;
    const int64_t s = blockIdx.x, f0 = s * ns;
    // the passes below re-read the sample's keys several times: from shared memory
    // when they fit (several independent loads in flight while staging them)
    const bool on_chip = ns <= kSmemKeys;
    if (on_chip) {
        for (int64_t i0 = threadIdx.x; i0 < ns; i0 += 4 * kThreads) {
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = i0 + u * kThreads < ns ? __ldcg(sumsq_g + f0 + i0 + u * kThreads) : 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u * kThreads < ns) s_keys[i0 + u * kThreads] = v[u];
        }
        __syncthreads();
    }
    auto keyat = [&](int64_t f) -> float { return on_chip ? s_keys[f] : __ldcg(sumsq_g + f0 + f); };
    const int64_t out0 = s * ks;  // this sample's first output slot
    if (s == 0 && threadIdx.x == 0) rowptr[0] = 0;
    uint32_t prefix = 0, need = (uint32_t)ks;
    int shift = 31;
    if (ks > 0 && ks < ns) {
        for (int pass = 0; pass < 4; ++pass) {
            const int w = pass < 3 ? 8 : 7, nshift = shift - w;
            if (threadIdx.x < 256) s_h[threadIdx.x] = 0;
            __syncthreads();
            for (int64_t fb0 = 0; fb0 < ns; fb0 += 4 * kThreads) {
              float kv[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                  const int64_t f = fb0 + u * kThreads + threadIdx.x;
                  kv[u] = f < ns ? keyat(f) : 0.f;  // 4 independent loads in flight (keys off chip)
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int64_t f = fb0 + u * kThreads + threadIdx.x;
                if (fb0 + u * kThreads >= ns) break;
                const uint32_t key = f < ns ? key_of(kv[u]) : 0u;
                const bool in = f < ns && (pass == 0 || (key >> shift) == prefix);
                const uint32_t bin = (key >> nshift) & ((1u << w) - 1u);
                const uint32_t im = __ballot_sync(0xffffffffu, in);
                if (!im) continue;
                const int l0 = __ffs(im) - 1;
                const uint32_t b0 = __shfl_sync(0xffffffffu, bin, l0);
                if (__all_sync(0xffffffffu, !in || bin == b0)) {  // a warp of ties adds once
                    if (lane == l0) atomicAdd(&s_h[b0], (uint32_t)__popc(im));
                } else if (in) {
                    atomicAdd(&s_h[bin], 1u);
                }
              }
            }
            __syncthreads();
            // bins in descending order: thread t owns bin 255 - t; exclusive scan = keys above
            const uint32_t cnt = threadIdx.x < 256 ? s_h[255 - threadIdx.x] : 0u;
            uint64_t tot;
            const uint32_t above = (uint32_t)scan64(cnt, s_warp, tot);
            if (threadIdx.x < 256 && above < need && above + cnt >= need) {
                s_sel[0] = 255 - threadIdx.x;
                s_sel[1] = above;
                s_sel[2] = cnt;
            }
            __syncthreads();
            prefix = (prefix << w) | s_sel[0];
            need -= s_sel[1];
            shift = nshift;
            const bool whole = need == s_sel[2];
            __syncthreads();
            if (whole) break;
        }
    } else {
        prefix = ks == 0 ? 0xffffffffu : 0u;  // keep none: nothing > / == ; keep all: every key >= 0
        shift = 0;
        need = ks == 0 ? 0u : (uint32_t)ns;
    }
    const uint32_t r = need;  // keys == prefix to keep (lowest flat index first)
    auto flags = [&](float key, uint32_t &a, uint32_t &t) {
        const uint32_t kk = key_of(key) >> shift;
        a = ks == ns ? 1u : ks > 0 ? (uint32_t)(kk > prefix) : 0u;
        t = (ks > 0 && ks < ns) ? (uint32_t)(kk == prefix) : 0u;
    };
    if (on_chip) {
        // keys on chip: thread-contiguous chunks (c odd: conflict-free), one block scan
        // of the per-thread (above, tie) counts, then each thread walks its chunk
        // again -- instead of one block-wide scan per 512 keys
        const int64_t c = ((ns + kThreads - 1) / kThreads) | 1;
        const int64_t t0 = ns < (int64_t)threadIdx.x * c ? ns : (int64_t)threadIdx.x * c;
        const int64_t t1 = ns < t0 + c ? ns : t0 + c;
        uint32_t na = 0, nt = 0;
        for (int64_t f = t0; f < t1; ++f) {
            uint32_t a, t;
            flags(s_keys[f], a, t);
            na += a;
            nt += t;
        }
        uint64_t tot;
        const uint64_t ex = scan64(((uint64_t)na << 32) | nt, s_warp, tot);
        uint32_t ab = (uint32_t)(ex >> 32), tb = (uint32_t)ex;
        for (int64_t f = t0; f < t1; ++f) {
            uint32_t a, t;
            flags(s_keys[f], a, t);
            const bool kept = a || (t && tb < r);
            const int64_t pos = out0 + ab + min(r, tb);
            const int64_t row = f / nbc, J = f - row * nbc;
            if (kept) colidx[pos] = (int32_t)J;  // the segment itself: rows_pack_kernel
            if (J == nbc - 1) rowptr[s * S + row + 1] = (int32_t)(out0 + ab + a + min(r, tb + t));
            ab += a;
            tb += t;
        }
        return;
    }
    // keys off chip: flat-order scan in 512-key chunks, the next chunk's keys in flight
    uint64_t base = 0;
    float kcur = threadIdx.x < ns ? keyat(threadIdx.x) : 0.f;
    for (int64_t fb = 0; fb < ns; fb += kThreads) {
        const int64_t f = fb + threadIdx.x;
        // the next chunk's key is in flight while this chunk is scanned (keys off chip)
        const float knext = f + kThreads < ns ? keyat(f + kThreads) : 0.f;
        uint32_t a = 0, t = 0;
        if (f < ns) {
            const uint32_t kk = key_of(kcur) >> shift;
            if (ks == ns) {
                a = 1;
            } else if (ks > 0) {
                a = kk > prefix;
                t = kk == prefix;
            }
        }
        uint64_t tot;
        const uint64_t ex = scan64(((uint64_t)a << 32) | t, s_warp, tot);
        const uint32_t ab = (uint32_t)(base >> 32) + (uint32_t)(ex >> 32), tb = (uint32_t)base + (uint32_t)ex;
        if (f < ns) {
            const bool kept = a || (t && tb < r);
            const int64_t pos = out0 + ab + min(r, tb);
            const int64_t row = f / nbc, J = f - row * nbc;
            if (kept) colidx[pos] = (int32_t)J;  // the segment itself: rows_pack_kernel
            if (J == nbc - 1) rowptr[s * S + row + 1] = (int32_t)(out0 + ab + a + min(r, tb + t));
        }
        base += tot;
        kcur = knext;
    }
}

// Copy the kept segments into values (raw bits): one warp per row, the row's
// stored entries [rowptr[r], rowptr[r+1]) gathered from X at colidx -- the
// inverse of rows_decompress_kernel, over the whole GPU (the select kernel runs
// one CTA per sample and only indexes).
template <int ES, int B>
__global__ void __launch_bounds__(256) rows_pack_kernel(const uint8_t *__restrict__ X, const int32_t *__restrict__ rowptr,
                                                        const int32_t *__restrict__ colidx, int64_t M, int64_t K,
                                                        uint8_t *__restrict__ values) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int PC = B * ES >= 16 ? 16 : B * ES, NP = B * ES / PC;
    for (int64_t r = w0; r < M; r += nw) {
        const int a = __ldg(rowptr + r), z = __ldg(rowptr + r + 1);
        for (int i0 = lane; i0 < (z - a) * NP; i0 += 4 * 32) {  // 4 segments' pieces in flight per lane
            uint4 v[4];
            uint8_t *dst[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * 32;
                dst[u] = nullptr;
                if (i < (z - a) * NP) {
                    const int e = a + i / NP, q = i % NP;
                    const uint8_t *src = X + (r * K + (int64_t)__ldg(colidx + e) * B) * ES + q * PC;
                    dst[u] = values + (int64_t)e * B * ES + q * PC;
                    if constexpr (PC == 16) v[u] = __ldcs(reinterpret_cast<const uint4 *>(src));
                    else { const uint2 t = __ldcs(reinterpret_cast<const uint2 *>(src)); v[u] = make_uint4(t.x, t.y, 0, 0); }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (!dst[u]) continue;
                if constexpr (PC == 16) __stcs(reinterpret_cast<uint4 *>(dst[u]), v[u]);
                else __stcs(reinterpret_cast<uint2 *>(dst[u]), make_uint2(v[u].x, v[u].y));
            }
        }
    }
}

template <int ES, int B>
__global__ void __launch_bounds__(256) rows_decompress_kernel(const int32_t *__restrict__ rowptr,
                                                              const int32_t *__restrict__ colidx,
                                                              const uint8_t *__restrict__ values, int64_t M, int64_t K,
                                                              uint8_t *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < M; r += nw) {
        uint4 *row = reinterpret_cast<uint4 *>(out + r * K * ES);
        const int nv = (int)(K * ES / 16);
        for (int i = lane; i < nv; i += 32) row[i] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        const int a = __ldg(rowptr + r), z = __ldg(rowptr + r + 1);
        constexpr int PC = B * ES >= 16 ? 16 : B * ES, NP = B * ES / PC;
        for (int i = lane; i < (z - a) * NP; i += 32) {
            const int e = a + i / NP, q = i % NP;
            const uint8_t *src = values + (int64_t)e * B * ES + q * PC;
            uint8_t *dst = out + (r * K + (int64_t)__ldg(colidx + e) * B) * ES + q * PC;
            if constexpr (PC == 16) *reinterpret_cast<uint4 *>(dst) = __ldg(reinterpret_cast<const uint4 *>(src));
            else *reinterpret_cast<uint2 *>(dst) = __ldg(reinterpret_cast<const uint2 *>(src));
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------------ dW
constexpr int kWT = 256;  // threads of the dW kernel
constexpr int kKT = 128, kNT = 128, kR = 16;  // kcols, dY columns, rows per stage
constexpr int kSplitCTAs = 2 * 148;

struct WParams {
    const int32_t *rowptr, *colidx;
    const uint8_t *values, *dY;
    float *out;
    int64_t M, K, N;
    int nsplit, accumulate;
};

template <int ESX, int ESY, int B>
__global__ void __launch_bounds__(kWT, 2) rows_wgrad_kernel(WParams p) {
    constexpr int XB = kR * kKT * ESX, YB = kR * kNT * ESY, STAGE = XB + YB;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint32_t s_mask[2][kR], s_base[2][kR];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tn = tid & 15, tk = tid >> 4;
    const int nkt = (int)((p.K + kKT - 1) / kKT), ntn = (int)((p.N + kNT - 1) / kNT);
    int t = blockIdx.x;
    const int nt = t % ntn;
    t /= ntn;
    const int kt = t % nkt;
    const int split = t / nkt;
    const int64_t kc0 = (int64_t)kt * kKT, n0 = (int64_t)nt * kNT;
    const int nbc = (int)(p.K / B), J0 = (int)(kc0 / B), nbJ = min(kKT / B, nbc - J0);
    const int64_t ngroups = (p.M + kR - 1) / kR;
    const int64_t Gb = (int64_t)split * ngroups / p.nsplit, Ge = (int64_t)(split + 1) * ngroups / p.nsplit;
    // this warp's kcols [16w, 16w + 16) of the range -> segment columns (range-relative)
    const int wj0 = (warp * 16) / B, wj1 = (warp * 16 + 15) / B;
    const uint32_t wmask = (wj1 >= 31 ? 0xffffffffu : ((1u << (wj1 + 1)) - 1u)) & ~((1u << wj0) - 1u);

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    const uint32_t sm0 = static_cast<uint32_t>(__cvta_generic_to_shared(smem));

    // per row of group g: kept-segment mask in [J0, J0 + nbJ) and first value index (warp 0)
    auto plan = [&](int64_t g, int buf) -> bool {
        if (warp == 0) {
            uint32_t mask = 0, base = 0;
            const int64_t r = g * kR + lane;
            if (lane < kR && r < p.M) {
                int lo = __ldg(p.rowptr + r), hi = __ldg(p.rowptr + r + 1);
                const int z = hi;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (__ldg(p.colidx + mid) < J0) lo = mid + 1; else hi = mid;
                }
                base = (uint32_t)lo;
                const int e1 = min(z, lo + nbJ);
                for (int e = lo; e < e1; ++e) {
                    const int J = __ldg(p.colidx + e) - J0;
                    if (J < nbJ) mask |= 1u << J;
                }
            }
            if (lane < kR) {
                s_mask[buf][lane] = mask;
                s_base[buf][lane] = base;
            }
        }
        __syncthreads();
        uint32_t any = 0;
        for (int i = 0; i < kR; ++i) any |= s_mask[buf][i];
        return any != 0;
    };
    auto stage = [&](int st, int64_t g, int buf) {
        const uint32_t xs = sm0 + (uint32_t)(st * STAGE), ys = xs + XB;
        constexpr int PC = (B * ESX < 16) ? B * ESX : 16;
        for (int q = tid; q < XB / PC; q += kWT) {
            const int rr = (q * PC) / (kKT * ESX), cbyte = (q * PC) % (kKT * ESX);
            const int j = cbyte / (B * ESX), off = cbyte % (B * ESX);
            const uint32_t mask = s_mask[buf][rr];
            const bool kept = j < nbJ && ((mask >> j) & 1u);
            const uint32_t idx = kept ? s_base[buf][rr] + __popc(mask & ((1u << j) - 1u)) : 0u;
            const uint8_t *src = p.values + (int64_t)idx * B * ESX + off;
            if constexpr (PC == 16)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(xs + (uint32_t)(q * PC)), "l"(src),
                             "r"(kept ? 16 : 0)
                             : "memory");
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(xs + (uint32_t)(q * PC)), "l"(src),
                             "n"(PC), "r"(kept ? PC : 0)
                             : "memory");
        }
        for (int q = tid; q < YB / 16; q += kWT) {
            const int rr = (q * 16) / (kNT * ESY), cbyte = (q * 16) % (kNT * ESY);
            const int64_t row = g * kR + rr, n = n0 + cbyte / ESY;
            const bool ok = row < p.M && n < p.N;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ys + (uint32_t)(q * 16)),
                         "l"(p.dY + ((ok ? row : 0) * p.N + (ok ? n : 0)) * ESY), "r"(ok ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    int cur = 0, buf = 0;
    bool have = false;
    int64_t g = Gb;
    while (true) {
        // next group with a kept segment in range
        bool next = false;
        while (g < Ge) {
            const bool any = plan(g, buf ^ (have ? 1 : 0));
            ++g;
            if (any) {
                next = true;
                break;
            }
        }
        if (next) stage(cur ^ (have ? 1 : 0), g - 1, buf ^ (have ? 1 : 0));
        if (have) {
            if (next) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            const uint8_t *xs = smem + cur * STAGE, *ys = xs + XB;
#pragma unroll 4
            for (int r = 0; r < kR; ++r) {
                if (!(s_mask[buf][r] & wmask)) continue;  // this row keeps no segment in the warp's 16 kcols
                float xv[8], yv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if constexpr (ESX == 4) xv[i] = reinterpret_cast<const float *>(xs)[r * kKT + tk * 8 + i];
                    else xv[i] = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(xs)[r * kKT + tk * 8 + i] << 16);
                    if constexpr (ESY == 4) yv[i] = reinterpret_cast<const float *>(ys)[r * kNT + tn * 8 + i];
                    else yv[i] = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t *>(ys)[r * kNT + tn * 8 + i] << 16);
                }
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(xv[i], yv[j], acc[i][j]);
            }
            __syncthreads();
            cur ^= 1;
            buf ^= 1;
        }
        if (!next) break;
        have = true;
    }
    (void)lane;
    float *out = p.out + (p.nsplit > 1 ? (int64_t)split * p.K * p.N : 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t row = kc0 + tk * 8 + i;
        if (row >= p.K) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t n = n0 + tn * 8 + 4 * h;
            if (n >= p.N) continue;
            float4 *o = reinterpret_cast<float4 *>(out + row * p.N + n);
            float4 v = make_float4(acc[i][4 * h], acc[i][4 * h + 1], acc[i][4 * h + 2], acc[i][4 * h + 3]);
            if (p.nsplit == 1 && p.accumulate) {
                const float4 old = *o;
                v.x += old.x; v.y += old.y; v.z += old.z; v.w += old.w;
            }
            *o = v;
        }
    }
}

static int sms() {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

static int nsplit_for(int64_t M, int64_t K, int64_t N) {
    const int64_t tiles = ((K + kKT - 1) / kKT) * ((N + kNT - 1) / kNT);
    const int64_t groups = (M + kR - 1) / kR;
    return (int)std::max<int64_t>(1, std::min<int64_t>(groups / 4, kSplitCTAs / std::max<int64_t>(1, tiles)));
}

}  // namespace rows

#define BSRP_ROWS_B(ES, b, CALL)          \
    switch (b) {                          \
        case 4: return CALL(ES, 4);       \
        case 8: return CALL(ES, 8);       \
        case 16: return CALL(ES, 16);     \
        case 32: return CALL(ES, 32);     \
        case 64: return CALL(ES, 64);     \
        default: return cudaErrorInvalidValue; \
    }

cudaError_t launch_prune_rows(const void *X, int64_t M, int64_t K, int b, int es, int64_t S, int64_t ks,
                              int32_t *rowptr, int32_t *colidx, void *values, void *ws, cudaStream_t stream) {
    float *sumsq = static_cast<float *>(ws);
    const int64_t N = M * (K / b);
    const unsigned g1 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, (int64_t)rows::sms() * 16));
#define CALL(ES_, B_) ([&]() -> cudaError_t {                                                                      \
        rows::rows_sumsq_kernel<ES_, B_><<<g1, 256, 0, stream>>>(static_cast<const uint8_t *>(X), M, K, sumsq);    \
        count_launch();                                                                                           \
        const int64_t ns_ = S * (K / B_);                                                                         \
        const size_t smem_ = ns_ <= rows::kSmemKeys ? (size_t)ns_ * 4 : 0;                                        \
        /* 48 KB of keys + the static shared arrays exceed the default 48 KB dynamic limit: opt in */            \
        if (smem_) {                                                                                              \
            const cudaError_t ea_ = cudaFuncSetAttribute(rows::rows_select_kernel<ES_, B_>,                         \
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_); \
            if (ea_ != cudaSuccess) return ea_;                                                                   \
        }                                                                                                         \
        rows::rows_select_kernel<ES_, B_><<<(unsigned)(M / S), rows::kThreads, smem_, stream>>>(                   \
            static_cast<const uint8_t *>(X), K, S, ks, sumsq, rowptr, colidx, static_cast<uint8_t *>(values));     \
        count_launch();                                                                                           \
        if (ks > 0) {                                                                                             \
            const unsigned g3 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((M + 7) / 8, (int64_t)rows::sms() * 16)); \
            rows::rows_pack_kernel<ES_, B_><<<g3, 256, 0, stream>>>(static_cast<const uint8_t *>(X), rowptr, colidx, \
                                                                  M, K, static_cast<uint8_t *>(values));          \
            count_launch();                                                                                       \
        }                                                                                                         \
        return cudaGetLastError();                                                                                \
    }())
    if (es == 4) {
        BSRP_ROWS_B(4, b, CALL)
    } else {
        BSRP_ROWS_B(2, b, CALL)
    }
#undef CALL
}

cudaError_t launch_decompress_rows(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t M,
                                   int64_t K, int b, int es, void *out, cudaStream_t stream) {
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((M + 7) / 8, (int64_t)rows::sms() * 16));
#define CALL(ES_, B_) ([&]() -> cudaError_t {                                                                     \
        rows::rows_decompress_kernel<ES_, B_><<<g, 256, 0, stream>>>(rowptr, colidx,                              \
                                                                     static_cast<const uint8_t *>(values), M, K, \
                                                                     static_cast<uint8_t *>(out));                \
        count_launch();                                                                                          \
        return cudaGetLastError();                                                                               \
    }())
    if (es == 4) {
        BSRP_ROWS_B(4, b, CALL)
    } else {
        BSRP_ROWS_B(2, b, CALL)
    }
#undef CALL
}

size_t wgrad_rows_ws_bytes(int64_t M, int64_t K, int64_t N) {
    const int ns = rows::nsplit_for(M, K, N);
    return ns > 1 ? (size_t)ns * K * N * sizeof(float) : 0;
}

cudaError_t launch_wgrad_rows(const int32_t *rowptr, const int32_t *colidx, const void *values, int es_x, int64_t M,
                              int64_t K, int b, const void *dY, int es_y, int64_t N, float *dW, int accumulate,
                              void *ws, cudaStream_t stream) {
    rows::WParams p{};
    p.rowptr = rowptr;
    p.colidx = colidx;
    p.values = static_cast<const uint8_t *>(values);
    p.dY = static_cast<const uint8_t *>(dY);
    p.M = M;
    p.K = K;
    p.N = N;
    p.accumulate = accumulate;
    p.nsplit = rows::nsplit_for(M, K, N);
    p.out = p.nsplit > 1 ? static_cast<float *>(ws) : dW;
    if (!values) return accumulate ? cudaSuccess : cudaMemsetAsync(dW, 0, (size_t)K * N * sizeof(float), stream);
    const int64_t tiles = ((K + rows::kKT - 1) / rows::kKT) * ((N + rows::kNT - 1) / rows::kNT);
    const unsigned grid = (unsigned)(tiles * p.nsplit);
#define LAUNCH(EX, EY, B_) ([&]() -> cudaError_t {                                                               \
        constexpr int smem = 2 * (rows::kR * rows::kKT * EX + rows::kR * rows::kNT * EY);                         \
        cudaError_t e = cudaFuncSetAttribute(rows::rows_wgrad_kernel<EX, EY, B_>,                                 \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);                  \
        if (e != cudaSuccess) return e;                                                                          \
        rows::rows_wgrad_kernel<EX, EY, B_><<<grid, rows::kWT, smem, stream>>>(p);                               \
        count_launch();                                                                                          \
        e = cudaGetLastError();                                                                                  \
        if (e != cudaSuccess || p.nsplit == 1) return e;                                                         \
        return launch_splitk_reduce(static_cast<const float *>(ws), dW, K * N, p.nsplit, accumulate, stream);     \
    }())
#define BCASE(EX, EY)                                 \
    switch (b) {                                      \
        case 4: return LAUNCH(EX, EY, 4);             \
        case 8: return LAUNCH(EX, EY, 8);             \
        case 16: return LAUNCH(EX, EY, 16);           \
        case 32: return LAUNCH(EX, EY, 32);           \
        case 64: return LAUNCH(EX, EY, 64);           \
        default: return cudaErrorInvalidValue;        \
    }
    if (es_x == 4 && es_y == 4) BCASE(4, 4)
    if (es_x == 4 && es_y == 2) BCASE(4, 2)
    if (es_x == 2 && es_y == 4) BCASE(2, 4)
    BCASE(2, 2)
#undef BCASE
#undef LAUNCH
}

}  // namespace bsrp
