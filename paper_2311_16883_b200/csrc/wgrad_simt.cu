// wgrad_simt.cu -- the FP32 path of the BSR weight gradient (row a6).
//
//   dW[J*b + c][n] = sum over stored blocks (I, J), sum over r < b of
//                    values(I,J)[r][c] * dY[I*b + r][n]          (BJ)
//
// fp32 FFMA with round-to-nearest in a FIXED order (ascending block row I within
// a split, ascending r; splits summed in split order), so the result is
// deterministic and, within ~2e-6..5e-6 relative Frobenius
// error of the fp64 oracle (the 1e-5 bar; plain TF32 cannot meet it).  This is
// the path for every b (4..64) and for fp32 storage at b < 32, where the tf32
// tensor-core operands do not exist (R16).
//
// CTA = 128 kcols (dW rows) x 128 dY columns x a range of block rows (split-K).
// 256 threads, each an 8 x 8 register tile; a warp owns 16 consecutive kcols, so
// a warp whose kcols are all in pruned blocks of a block row skips that row's
// FMAs (warp-uniform).  Per block row with at least one stored block in the
// CTA's kcol range: the b x 128 slab of dY and the b x 128 strip of X (stored
// blocks copied, pruned blocks zero-filled) are staged in shared memory by
// 16-byte cp.async, double-buffered so the next row's copies overlap this row's
// FFMAs.  Block rows without a stored block in range are never read.  Warp 0
// plans 32 block rows at a time (kept-block mask + first value index per row).
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace bsrp {
namespace simt {

constexpr int kThreads = 256;
constexpr int kKT = 128;  // kcols per CTA
constexpr int kNT = 128;  // dY columns per CTA
constexpr int kSplitCTAs = 2 * 148;  // target CTAs (2 per SM) when splitting block rows

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}

// 4 consecutive elements as fp32 (bf16: exact widening).
template <int ES>
__device__ __forceinline__ float4 to_f4(const uint4 &w, int half) {
    if constexpr (ES == 4) {
        return make_float4(__uint_as_float(w.x), __uint_as_float(w.y), __uint_as_float(w.z), __uint_as_float(w.w));
    } else {
        const uint32_t a = half ? w.z : w.x, c = half ? w.w : w.y;
        return make_float4(__uint_as_float(a << 16), __uint_as_float(a & 0xffff0000u), __uint_as_float(c << 16),
                           __uint_as_float(c & 0xffff0000u));
    }
}

struct Params {
    const int32_t *rowptr, *colidx;
    const uint8_t *values, *dY;
    float *out;  // dW (nsplit == 1) or the split-K workspace
    int64_t nbr, K, N;
    int nsplit, accumulate;
};

// Shared memory per stage: X strip [b][kKT] and dY slab [b][kNT], in element
// bytes of the inputs (bf16 stays bf16 in shared memory; widened when read).
template <int ESX, int ESY, int B>
struct Smem {
    static constexpr int X_BYTES = B * kKT * ESX;
    static constexpr int Y_BYTES = B * kNT * ESY;
    static constexpr int STAGE = X_BYTES + Y_BYTES;
};

template <int ESX, int ESY, int B>
__global__ void __launch_bounds__(kThreads, 2) wgrad_simt_kernel(Params p) {
    using S = Smem<ESX, ESY, B>;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint32_t s_mask[32], s_base[32], s_row[32];
    __shared__ int s_cnt;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tn = tid & 15, tk = tid >> 4;  // 8 dY columns x 8 kcols per thread
    const int nkt = (int)((p.K + kKT - 1) / kKT);
    const int ntn = (int)((p.N + kNT - 1) / kNT);
    int t = blockIdx.x;
    const int nt = t % ntn;
    t /= ntn;
    const int kt = t % nkt;
    const int split = t / nkt;
    const int64_t kc0 = (int64_t)kt * kKT, n0 = (int64_t)nt * kNT;
    const int nbc = (int)(p.K / B);
    const int J0 = (int)(kc0 / B);                       // first block column of the range
    const int nbJ = min(kKT / B > 0 ? kKT / B : 1, nbc - J0);  // block columns in range (kKT >= B)
    const int64_t Ib = (int64_t)split * p.nbr / p.nsplit, Ie = (int64_t)(split + 1) * p.nbr / p.nsplit;
    // this warp's kcols [16w, 16w + 16) of the range -> block columns (range-relative)
    const int wj0 = (warp * 16) / B, wj1 = (warp * 16 + 15) / B;
    const uint32_t wmask = (wj1 >= 31 ? 0xffffffffu : ((1u << (wj1 + 1)) - 1u)) & ~((1u << wj0) - 1u);

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    const uint32_t sm0 = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    // Stage the X strip and the dY slab of block row I (mask/base: stored blocks in range).
    auto stage_row = [&](int st, int64_t I, uint32_t mask, uint32_t base) {
        const uint32_t xs = sm0 + (uint32_t)(st * S::STAGE), ys = xs + S::X_BYTES;
        // X strip: row r of block column j -> bytes [r][j*B .. (j+1)*B) of a [B][kKT] tile,
        // in pieces that never cross a block row (8 bytes for bf16 b = 4)
        constexpr int PC = (B * ESX < 16) ? B * ESX : 16;
        constexpr int XP = S::X_BYTES / PC;
        for (int q = tid; q < XP; q += kThreads) {
            const int r = (q * PC) / (kKT * ESX);
            const int cbyte = (q * PC) % (kKT * ESX);
            const int j = cbyte / (B * ESX), off = cbyte % (B * ESX);
            const bool kept = j < nbJ && ((mask >> j) & 1u);
            const uint32_t idx = kept ? base + __popc(mask & ((1u << j) - 1u)) : 0u;
            const uint8_t *src = p.values + ((int64_t)idx * B * B * ESX + (int64_t)r * B * ESX + off);
            if constexpr (PC == 16) {
                cp_async16(xs + (uint32_t)(q * PC), src, kept);
            } else {
                asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(xs + (uint32_t)(q * PC)), "l"(src),
                             "n"(PC), "r"(kept ? PC : 0)
                             : "memory");
            }
        }
        constexpr int YP = S::Y_BYTES / 16;
        for (int q = tid; q < YP; q += kThreads) {
            const int r = (q * 16) / (kNT * ESY);
            const int cbyte = (q * 16) % (kNT * ESY);
            const int64_t n = n0 + cbyte / ESY;
            const bool ok = n < p.N;
            cp_async16(ys + (uint32_t)(q * 16), p.dY + ((I * B + r) * p.N + (ok ? n : 0)) * ESY, ok);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    // rows are planned 32 at a time by warp 0 (kept-block mask in range + first value index)
    int64_t I0 = Ib;
    int cnt = 0, pos = 0;
    auto plan = [&]() {
        __syncthreads();  // previous plan fully consumed
        if (warp == 0) {
            const int64_t I = I0 + lane;
            uint32_t mask = 0, base = 0;
            if (I < Ie) {
                int lo = __ldg(p.rowptr + I), hi = __ldg(p.rowptr + I + 1);
                const int z = hi;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (__ldg(p.colidx + mid) < J0) lo = mid + 1; else hi = mid;
                }
                base = (uint32_t)lo;
                // at most nbJ stored blocks lie in range: independent loads, no early exit
                const int e1 = min(z, lo + nbJ);
#pragma unroll 8
                for (int e = lo; e < e1; ++e) {
                    const int J = __ldg(p.colidx + e) - J0;
                    if (J < nbJ) mask |= 1u << J;
                }
            }
            const uint32_t rows = __ballot_sync(0xffffffffu, mask != 0);
            if (mask) {
                const int k = __popc(rows & ((1u << lane) - 1u));
                s_mask[k] = mask;
                s_base[k] = base;
                s_row[k] = (uint32_t)(I - I0);
            }
            if (lane == 0) s_cnt = __popc(rows);
        }
        __syncthreads();
        cnt = s_cnt;
        pos = 0;
    };

    plan();
    // software pipeline: the row in stage `cur` is computed while the next one lands
    int cur = 0;
    bool have = false;
    uint32_t cmask = 0;
    while (true) {
        // find the next row to stage (possibly planning the next 32 rows)
        while (pos >= cnt && I0 + 32 < Ie) {
            I0 += 32;
            // the plan buffers are rewritten: the staged row's mask was copied to cmask
            plan();
        }
        const bool next = pos < cnt;
        uint32_t nmask = 0;
        if (next) {
            nmask = s_mask[pos];
            stage_row(cur ^ (have ? 1 : 0), I0 + s_row[pos], nmask, s_base[pos]);
            ++pos;
        }
        if (have) {
            // wait for the current row's copies (the next row's group may stay in flight)
            if (next) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            if (cmask & wmask) {
                const uint8_t *xs = smem + cur * S::STAGE, *ys = xs + S::X_BYTES;
#pragma unroll 4
                for (int r = 0; r < B; ++r) {
                    float xv[8], yv[8];
                    if constexpr (ESX == 4) {
                        const float4 a = *reinterpret_cast<const float4 *>(xs + (r * kKT + tk * 8) * 4);
                        const float4 c = *reinterpret_cast<const float4 *>(xs + (r * kKT + tk * 8 + 4) * 4);
                        xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
                        xv[4] = c.x; xv[5] = c.y; xv[6] = c.z; xv[7] = c.w;
                    } else {
                        const uint4 w = *reinterpret_cast<const uint4 *>(xs + (r * kKT + tk * 8) * 2);
                        const float4 a = to_f4<2>(w, 0), c = to_f4<2>(w, 1);
                        xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
                        xv[4] = c.x; xv[5] = c.y; xv[6] = c.z; xv[7] = c.w;
                    }
                    if constexpr (ESY == 4) {
                        const float4 a = *reinterpret_cast<const float4 *>(ys + (r * kNT + tn * 8) * 4);
                        const float4 c = *reinterpret_cast<const float4 *>(ys + (r * kNT + tn * 8 + 4) * 4);
                        yv[0] = a.x; yv[1] = a.y; yv[2] = a.z; yv[3] = a.w;
                        yv[4] = c.x; yv[5] = c.y; yv[6] = c.z; yv[7] = c.w;
                    } else {
                        const uint4 w = *reinterpret_cast<const uint4 *>(ys + (r * kNT + tn * 8) * 2);
                        const float4 a = to_f4<2>(w, 0), c = to_f4<2>(w, 1);
                        yv[0] = a.x; yv[1] = a.y; yv[2] = a.z; yv[3] = a.w;
                        yv[4] = c.x; yv[5] = c.y; yv[6] = c.z; yv[7] = c.w;
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(xv[i], yv[j], acc[i][j]);
                }
            }
            __syncthreads();  // stage `cur` may be overwritten from here on
            cur ^= 1;
        }
        if (!next) break;
        have = true;
        cmask = nmask;
    }

    // epilogue: rows kc0 + tk*8 + i, columns n0 + tn*8 .. +8
    float *out = p.out + (p.nsplit > 1 ? (int64_t)split * p.K * p.N : 0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t row = kc0 + tk * 8 + i;
        if (row >= p.K) continue;
        const int64_t n = n0 + tn * 8;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (n + 4 * h >= p.N) continue;
            float4 *o = reinterpret_cast<float4 *>(out + row * p.N + n + 4 * h);
            float4 v = make_float4(acc[i][4 * h], acc[i][4 * h + 1], acc[i][4 * h + 2], acc[i][4 * h + 3]);
            if (p.nsplit == 1 && p.accumulate) {
                const float4 old = *o;
                v.x += old.x; v.y += old.y; v.z += old.z; v.w += old.w;
            }
            *o = v;
        }
    }
}

static int nsplit_for(int64_t M, int64_t K, int b, int64_t N) {
    const int64_t tiles = ((K + kKT - 1) / kKT) * ((N + kNT - 1) / kNT);
    const int64_t nbr = M / b;
    return (int)std::max<int64_t>(1, std::min<int64_t>(nbr / 8, kSplitCTAs / std::max<int64_t>(1, tiles)));
}

template <int ESX, int ESY, int B>
static cudaError_t launch_t(const Params &p0, int64_t M, cudaStream_t stream, void *ws) {
    using S = Smem<ESX, ESY, B>;
    Params p = p0;
    p.nsplit = nsplit_for(M, p.K, B, p.N);
    float *dW = p.out;
    if (p.nsplit > 1) p.out = static_cast<float *>(ws);
    auto kern = wgrad_simt_kernel<ESX, ESY, B>;
    const int smem = 2 * S::STAGE;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int64_t tiles = ((p.K + kKT - 1) / kKT) * ((p.N + kNT - 1) / kNT);
    kern<<<(unsigned)(tiles * p.nsplit), kThreads, smem, stream>>>(p);
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess || p.nsplit == 1) return e;
    return launch_splitk_reduce(static_cast<const float *>(ws), dW, p.K * p.N, p.nsplit, p.accumulate, stream);
}

template <int ESX, int ESY>
static cudaError_t launch_es(const Params &p, int64_t M, int b, cudaStream_t stream, void *ws) {
    switch (b) {
        case 4: return launch_t<ESX, ESY, 4>(p, M, stream, ws);
        case 8: return launch_t<ESX, ESY, 8>(p, M, stream, ws);
        case 16: return launch_t<ESX, ESY, 16>(p, M, stream, ws);
        case 32: return launch_t<ESX, ESY, 32>(p, M, stream, ws);
        case 64: return launch_t<ESX, ESY, 64>(p, M, stream, ws);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace simt

size_t wgrad_simt_ws_bytes(int64_t M, int64_t K, int b, int64_t N) {
    const int ns = simt::nsplit_for(M, K, b, N);
    return ns > 1 ? (size_t)ns * K * N * sizeof(float) : 0;
}

cudaError_t launch_wgrad_simt(const int32_t *rowptr, const int32_t *colidx, const void *values, int es_x,
                              int64_t M, int64_t K, int b, const void *dY, int es_y, int64_t N, float *dW,
                              int accumulate, void *ws, cudaStream_t stream) {
    simt::Params p{};
    p.rowptr = rowptr;
    p.colidx = colidx;
    p.values = static_cast<const uint8_t *>(values);
    p.dY = static_cast<const uint8_t *>(dY);
    p.out = dW;
    p.nbr = M / b;
    p.K = K;
    p.N = N;
    p.accumulate = accumulate;
    if (!values) {  // no stored block (k = 0): dW = 0 (or unchanged)
        return accumulate ? cudaSuccess : cudaMemsetAsync(dW, 0, (size_t)K * N * sizeof(float), stream);
    }
    if (es_x == 4 && es_y == 4) return simt::launch_es<4, 4>(p, M, b, stream, ws);
    if (es_x == 4 && es_y == 2) return simt::launch_es<4, 2>(p, M, b, stream, ws);
    if (es_x == 2 && es_y == 4) return simt::launch_es<2, 4>(p, M, b, stream, ws);
    return simt::launch_es<2, 2>(p, M, b, stream, ws);
}

}  // namespace bsrp
