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

}  // namespace bsrp
