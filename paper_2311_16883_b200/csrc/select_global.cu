// select_global.cu -- cross-rank global top-k.
//
// Under data parallelism each rank holds a shard of the batch rows of X.  With
// per-rank scope (reading R2, the default) every rank keeps keep * N_rank blocks.
// The global variant keeps the k = nearest(keep * N_total) largest blocks of the
// CONCATENATED X (rank order = flat order), so the kept set is the one a single
// GPU would select on the whole batch (P:L413-418 applied to the full X; tie
// rule BJ: lower flat index first, i.e. lower rank first).
//
// The library does no communication.  It exposes the three local steps the
// caller interleaves with two collectives (all-reduce of digit histograms,
// all-gather of tie counts), see paper_2311_16883_b200.prune_global:
//   1. bsr_select_hist   level 0: block sums of squares (kept in the prune
//                        workspace) + histogram of key bits 30..19;
//                        level 1 / 2: histogram of bits 18..9 / 8..0 of the
//                        keys matching a prefix.
//   2. bsr_select_counts (keys > T, keys == T) of this rank at a digit shift.
//   3. bsr_prune_threshold  pack: keep keys > T and the first `tie_take` keys
//                        == T in flat order (one cooperative kernel: per-CTA
//                        counts, grid barrier, flat-order scan, raw-bit copy).
// Same fp32 keys, scan and pack code as bsr_prune (prune.cu), so with one rank
// the result is bit-identical to bsr_prune_k.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace bsrp {
namespace sel {

constexpr int kThreads = 512;
constexpr int kH1 = 4096, kH2 = 1024, kH3 = 512;

__device__ __forceinline__ uint32_t key_of(float s) { return __float_as_uint(s) & 0x7fffffffu; }

// Histogram of one key digit: level 0 = bits 30..19 (all keys), 1 = bits 18..9
// of keys with bits 30..19 == prefix, 2 = bits 8..0 of keys with bits 30..9 == prefix.
__global__ void __launch_bounds__(kThreads) digit_hist_kernel(const float *__restrict__ sumsq, int64_t N, int level,
                                                              uint32_t prefix, uint32_t *__restrict__ hist) {
    __shared__ uint32_t s_h[kH1];
    const int nb = level == 0 ? kH1 : level == 1 ? kH2 : kH3;
    const int sh_pre = level == 0 ? 31 : level == 1 ? 19 : 9;
    const int sh = level == 0 ? 19 : level == 1 ? 9 : 0;
    for (int i = threadIdx.x; i < nb; i += kThreads) s_h[i] = 0;
    __syncthreads();
    for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < N; f += (int64_t)gridDim.x * kThreads) {
        const uint32_t key = key_of(__ldg(sumsq + f));
        if (level == 0 || (key >> sh_pre) == prefix) atomicAdd(&s_h[(key >> sh) & (nb - 1)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += kThreads)
        if (s_h[i]) atomicAdd(hist + i, s_h[i]);
}

// counts[0] += #(key >> shift > T), counts[1] += #(key >> shift == T)
__global__ void __launch_bounds__(kThreads) count_kernel(const float *__restrict__ sumsq, int64_t N, uint32_t T,
                                                         int shift, unsigned long long *__restrict__ counts) {
    uint32_t a = 0, t = 0;
    for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < N; f += (int64_t)gridDim.x * kThreads) {
        const uint32_t kk = key_of(__ldg(sumsq + f)) >> shift;
        a += kk > T;
        t += kk == T;
    }
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (a) atomicAdd(counts, (unsigned long long)a);
        if (t) atomicAdd(counts + 1, (unsigned long long)t);
    }
}

// ---- device-side protocol (no host round trip between the collectives) ----
// State words (uint64, caller-owned device memory, kGStateWords):
//   0 k_total  1 prefix T  2 shift  3 above (all ranks, strictly above the current
//   prefix)  4 r = k_total - above  5 done (the boundary digit is resolved)
//   6 tie_take (this rank)  7 k_rank (this rank's kept blocks)  8 bin count
enum { GS_K = 0, GS_T = 1, GS_SHIFT = 2, GS_ABOVE = 3, GS_R = 4, GS_DONE = 5, GS_TAKE = 6, GS_KRANK = 7, GS_CNT = 8 };

__global__ void gselect_init_kernel(unsigned long long k_total, unsigned long long *st) {
    if (threadIdx.x < 16) st[threadIdx.x] = 0;
    __syncwarp();
    if (threadIdx.x == 0) {
        st[GS_K] = k_total;
        st[GS_R] = k_total;
        if (k_total == 0) {  // nothing kept: a threshold no key exceeds, no ties to take
            st[GS_T] = 0xffffffffull;
            st[GS_DONE] = 1;
        }
    }
}

// Histogram of the next key digit of this rank's keys, or all zeros once the
// boundary is resolved (the collective sequence stays fixed: 3 all-reduces).
__global__ void __launch_bounds__(kThreads) gselect_hist_kernel(const float *__restrict__ sumsq, int64_t N, int level,
                                                                const unsigned long long *__restrict__ st,
                                                                uint32_t *__restrict__ hist) {
    __shared__ uint32_t s_h[kH1];
    const int nb = level == 0 ? kH1 : level == 1 ? kH2 : kH3;
    const int sh_pre = level == 0 ? 31 : level == 1 ? 19 : 9;
    const int sh = level == 0 ? 19 : level == 1 ? 9 : 0;
    const bool done = st[GS_DONE] != 0;
    const uint32_t prefix = (uint32_t)st[GS_T];
    for (int i = threadIdx.x; i < nb; i += kThreads) s_h[i] = 0;
    __syncthreads();
    if (!done)
        for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < N; f += (int64_t)gridDim.x * kThreads) {
            const uint32_t key = key_of(__ldg(sumsq + f));
            if (level == 0 || (key >> sh_pre) == prefix) atomicAdd(&s_h[(key >> sh) & (nb - 1)], 1u);
        }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += kThreads)
        if (s_h[i]) atomicAdd(hist + i, s_h[i]);
}

// One CTA: the bin of the all-reduced histogram that holds the r-th largest key
// (bins scanned from the top), appended to the prefix (P:L415-417 + BJ tie rule).
__global__ void __launch_bounds__(kThreads) gselect_update_kernel(const uint32_t *__restrict__ hist, int level,
                                                                  unsigned long long *__restrict__ st) {
    __shared__ unsigned long long s_part[kThreads];
    __shared__ unsigned long long s_sel[3];
    if (st[GS_DONE]) return;
    const int nb = level == 0 ? kH1 : level == 1 ? kH2 : kH3;
    const int bits = level == 0 ? 12 : level == 1 ? 10 : 9;
    const unsigned long long target = st[GS_R];
    const int per = nb / kThreads;  // 8, 2, 1; thread 0 owns the top bins
    unsigned long long loc = 0;
    for (int i = 0; i < per; ++i) loc += hist[nb - 1 - (threadIdx.x * per + i)];
    s_part[threadIdx.x] = loc;
    __syncthreads();
    if (threadIdx.x == 0) {  // sequential exclusive scan over 512 partials (one-off, tiny)
        unsigned long long run = 0;
        for (int t = 0; t < kThreads; ++t) {
            const unsigned long long v = s_part[t];
            s_part[t] = run;
            run += v;
        }
    }
    __syncthreads();
    unsigned long long run = s_part[threadIdx.x];
    for (int i = 0; i < per; ++i) {
        const int bin = nb - 1 - (threadIdx.x * per + i);
        const unsigned long long h = hist[bin];
        if (run < target && run + h >= target) {
            s_sel[0] = (unsigned long long)bin;
            s_sel[1] = run;
            s_sel[2] = h;
        }
        run += h;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long prefix = level == 0 ? s_sel[0] : (st[GS_T] << bits) | s_sel[0];
        st[GS_T] = prefix;
        st[GS_SHIFT] = level == 0 ? 19 : level == 1 ? 9 : 0;
        st[GS_ABOVE] += s_sel[1];
        st[GS_R] = st[GS_K] - st[GS_ABOVE];
        st[GS_CNT] = s_sel[2];
        if (st[GS_R] >= s_sel[2] || level == 2) st[GS_DONE] = 1;  // the whole bin is kept, or the key is exact
    }
}

// This rank's (#keys > T, #keys == T) at the resolved digit.
__global__ void __launch_bounds__(kThreads) gselect_count_kernel(const float *__restrict__ sumsq, int64_t N,
                                                                 const unsigned long long *__restrict__ st,
                                                                 unsigned long long *__restrict__ counts) {
    const uint32_t T = (uint32_t)st[GS_T];
    const int shift = (int)st[GS_SHIFT];
    uint32_t a = 0, t = 0;
    for (int64_t f = (int64_t)blockIdx.x * kThreads + threadIdx.x; f < N; f += (int64_t)gridDim.x * kThreads) {
        const uint32_t kk = key_of(__ldg(sumsq + f)) >> shift;
        a += kk > T;
        t += kk == T;
    }
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (a) atomicAdd(counts, (unsigned long long)a);
        if (t) atomicAdd(counts + 1, (unsigned long long)t);
    }
}

// Tie quota of this rank from every rank's (above, tie) counts (lower ranks
// first = lower flat index first in the concatenated X, BJ tie rule).
__global__ void gselect_take_kernel(const unsigned long long *__restrict__ all, int world, int rank,
                                    unsigned long long *__restrict__ st) {
    if (threadIdx.x != 0) return;
    unsigned long long before = 0;
    for (int q = 0; q < rank; ++q) before += all[2 * q + 1];
    const unsigned long long r = st[GS_R], mine = all[2 * rank + 1];
    const unsigned long long take = r > before ? (r - before < mine ? r - before : mine) : 0ull;
    st[GS_TAKE] = take;
    st[GS_KRANK] = all[2 * rank] + take;
}

}  // namespace sel

static int grid_for(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + sel::kThreads - 1) / sel::kThreads, (int64_t)sms * 4));
}

cudaError_t launch_select_hist(const void *X, int64_t M, int64_t K, int b, int es, int level, uint32_t prefix,
                               uint32_t *hist, void *ws, cudaStream_t stream) {
    const int64_t N = (M / b) * (K / b);
    const PruneWs w = prune_ws_layout(N);
    float *sumsq = reinterpret_cast<float *>(static_cast<char *>(ws) + w.sumsq);
    if (level == 0) {
        cudaError_t e = launch_block_sumsq(X, M, K, b, es, sumsq, stream);
        if (e != cudaSuccess) return e;
    }
    const int nb = level == 0 ? sel::kH1 : level == 1 ? sel::kH2 : sel::kH3;
    cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)nb * 4, stream);
    if (e != cudaSuccess) return e;
    sel::digit_hist_kernel<<<grid_for(N), sel::kThreads, 0, stream>>>(sumsq, N, level, prefix, hist);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_select_counts(int64_t M, int64_t K, int b, uint32_t T, int shift, uint64_t *counts, void *ws,
                                 cudaStream_t stream) {
    const int64_t N = (M / b) * (K / b);
    const PruneWs w = prune_ws_layout(N);
    const float *sumsq = reinterpret_cast<const float *>(static_cast<const char *>(ws) + w.sumsq);
    cudaError_t e = cudaMemsetAsync(counts, 0, 2 * sizeof(uint64_t), stream);
    if (e != cudaSuccess) return e;
    sel::count_kernel<<<grid_for(N), sel::kThreads, 0, stream>>>(sumsq, N, T, shift,
                                                                  reinterpret_cast<unsigned long long *>(counts));
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gselect_init(int64_t k_total, uint64_t *state, cudaStream_t stream) {
    sel::gselect_init_kernel<<<1, 32, 0, stream>>>((unsigned long long)k_total,
                                                   reinterpret_cast<unsigned long long *>(state));
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gselect_hist(const void *X, int64_t M, int64_t K, int b, int es, int level, const uint64_t *state,
                                uint32_t *hist, void *ws, cudaStream_t stream) {
    const int64_t N = (M / b) * (K / b);
    const PruneWs w = prune_ws_layout(N);
    float *sumsq = reinterpret_cast<float *>(static_cast<char *>(ws) + w.sumsq);
    if (level == 0) {
        cudaError_t e = launch_block_sumsq(X, M, K, b, es, sumsq, stream);
        if (e != cudaSuccess) return e;
    }
    const int nb = level == 0 ? sel::kH1 : level == 1 ? sel::kH2 : sel::kH3;
    cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)nb * 4, stream);
    if (e != cudaSuccess) return e;
    sel::gselect_hist_kernel<<<grid_for(N), sel::kThreads, 0, stream>>>(
        sumsq, N, level, reinterpret_cast<const unsigned long long *>(state), hist);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gselect_update(const uint32_t *hist_total, int level, uint64_t *state, cudaStream_t stream) {
    sel::gselect_update_kernel<<<1, sel::kThreads, 0, stream>>>(hist_total, level,
                                                                reinterpret_cast<unsigned long long *>(state));
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gselect_counts(int64_t M, int64_t K, int b, const uint64_t *state, uint64_t *counts, void *ws,
                                  cudaStream_t stream) {
    const int64_t N = (M / b) * (K / b);
    const PruneWs w = prune_ws_layout(N);
    const float *sumsq = reinterpret_cast<const float *>(static_cast<const char *>(ws) + w.sumsq);
    cudaError_t e = cudaMemsetAsync(counts, 0, 2 * sizeof(uint64_t), stream);
    if (e != cudaSuccess) return e;
    sel::gselect_count_kernel<<<grid_for(N), sel::kThreads, 0, stream>>>(
        sumsq, N, reinterpret_cast<const unsigned long long *>(state), reinterpret_cast<unsigned long long *>(counts));
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gselect_take(const uint64_t *all_counts, int world, int rank, uint64_t *state, cudaStream_t stream) {
    sel::gselect_take_kernel<<<1, 32, 0, stream>>>(reinterpret_cast<const unsigned long long *>(all_counts), world, rank,
                                                   reinterpret_cast<unsigned long long *>(state));
    count_launch();
    return cudaGetLastError();
}

}  // namespace bsrp
