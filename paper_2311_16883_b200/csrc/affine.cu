// affine.cu -- weight gradient of the block-sparse affine scaling layer
// ("A block-sparse version of the affine scaling layer found
// in ResMLP is now also available, potentially allowing for further memory
// savings").
//
// ResMLP's Aff(x) = alpha * x + beta acts per channel c on the M x K residual
// stream.  Its only activation-dependent gradient is
//   dalpha[c] = sum over rows m of x[m][c] * dY[m][c]
// (dbeta = column sums of dY and dX = alpha * dY need no activation, like the
// dense dX / db of the linear layer).  With x saved as the BSR of its
// top-k b x b blocks, the sum runs over the kept blocks only:
//   dalpha[J*b + c] = sum over kept (I, J), sum over r < b of
//                     values(I,J)[r][c] * dY[I*b + r][J*b + c]
// Pruned blocks are never read, neither their X nor their dY.
//
// Layout: CTA = (block column J, range of block rows = split).  Its 128 threads
// own (column c = t % b, row group t / b); each walks the kept blocks of its
// rows that sit in column J (colidx ascending per row: one coalesced scan of the
// row's entries) and accumulates x * dY in fp32 with round-to-nearest FMAs in
// row order.  The row groups are combined by a fixed shared-memory tree and the
// split partials are summed in split order by the same deterministic reduce as
// the dW (launch_splitk_reduce), so the result does not depend on timing.
// HBM-bound: reads keep * (|X| + |dY|), writes K floats per split.
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace bsrp {
namespace aff {

constexpr int kThreads = 128;

template <int ESX, int ESY, int B>
__global__ void __launch_bounds__(kThreads) affine_wgrad_kernel(const int32_t *__restrict__ rowptr,
                                                                const int32_t *__restrict__ colidx,
                                                                const uint8_t *__restrict__ values,
                                                                const uint8_t *__restrict__ dY, int64_t nbr,
                                                                int64_t K, int nsplit, float *__restrict__ out) {
    constexpr int RG = kThreads / B;  // row groups (B <= 64 -> >= 2)
    __shared__ float s_red[kThreads];
    __shared__ int s_hit[32];
    const int J = blockIdx.x % (int)(K / B);
    const int split = blockIdx.x / (int)(K / B);
    const int64_t I0 = nbr * split / nsplit, I1 = nbr * (split + 1) / nsplit;
    const int t = threadIdx.x, c = t % B, g = t / B;
    const int lane = t & 31, warp = t >> 5;
    float acc = 0.f;
    for (int64_t I = I0; I < I1; ++I) {
        // the position of column J in row I (warp 0 scans the row's colidx 32 at a time)
        if (warp == 0) {
            const int rb = __ldg(rowptr + I), re = __ldg(rowptr + I + 1);
            int hit = -1;
            for (int e = rb; e < re && hit < 0; e += 32) {
                const int idx = e + lane;
                const int col = idx < re ? __ldg(colidx + idx) : -1;
                const unsigned m = __ballot_sync(0xffffffffu, col == J);
                if (m) hit = e + __ffs(m) - 1;
                if (__shfl_sync(0xffffffffu, col, 31) > J) break;  // ascending: J is not further on
            }
            if (lane == 0) s_hit[0] = hit;
        }
        __syncthreads();
        const int p = s_hit[0];
        __syncthreads();
        if (p < 0) continue;
        for (int r = g; r < B; r += RG) {
            const int64_t vi = ((int64_t)p * B + r) * B + c;
            const int64_t yi = (I * B + r) * K + (int64_t)J * B + c;
            float x, y;
            if constexpr (ESX == 4) x = __ldg(reinterpret_cast<const float *>(values) + vi);
            else x = __uint_as_float((uint32_t)__ldg(reinterpret_cast<const unsigned short *>(values) + vi) << 16);
            if constexpr (ESY == 4) y = __ldg(reinterpret_cast<const float *>(dY) + yi);
            else y = __uint_as_float((uint32_t)__ldg(reinterpret_cast<const unsigned short *>(dY) + yi) << 16);
            acc = __fmaf_rn(x, y, acc);
        }
    }
    // fixed tree over the row groups of column c
    s_red[t] = acc;
    __syncthreads();
    for (int h = RG / 2; h >= 1; h >>= 1) {
        if (g < h) s_red[t] = __fadd_rn(s_red[t], s_red[t + h * B]);
        __syncthreads();
    }
    if (g == 0) out[(int64_t)split * K + (int64_t)J * B + c] = s_red[c];
}

static int splits_for(int64_t nbr, int64_t K, int b) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t cols = K / b;
    const int64_t want = std::max<int64_t>(1, (int64_t)sms * 8 / cols);
    return (int)std::min<int64_t>({want, nbr, 4096});
}

}  // namespace aff

size_t affine_wgrad_ws_bytes(int64_t M, int64_t K, int b) {
    return (size_t)aff::splits_for(M / b, K, b) * K * sizeof(float);
}

cudaError_t launch_affine_wgrad(const int32_t *rowptr, const int32_t *colidx, const void *values, int es_x,
                                int64_t M, int64_t K, int b, const void *dY, int es_y, float *dalpha,
                                int accumulate, void *ws, cudaStream_t stream) {
    const int64_t nbr = M / b;
    const int ns = aff::splits_for(nbr, K, b);
    float *part = static_cast<float *>(ws);
    const unsigned grid = (unsigned)(ns * (K / b));
#define AFF_CASE(EX, EY, B_)                                                                                      \
    if (es_x == EX && es_y == EY && b == B_) {                                                                    \
        aff::affine_wgrad_kernel<EX, EY, B_><<<grid, aff::kThreads, 0, stream>>>(                                \
            rowptr, colidx, static_cast<const uint8_t *>(values), static_cast<const uint8_t *>(dY), nbr, K, ns, part); \
        count_launch();                                                                                           \
    } else
#define AFF_B(EX, EY) AFF_CASE(EX, EY, 4) AFF_CASE(EX, EY, 8) AFF_CASE(EX, EY, 16) AFF_CASE(EX, EY, 32) AFF_CASE(EX, EY, 64)
    AFF_B(4, 4) AFF_B(4, 2) AFF_B(2, 4) AFF_B(2, 2) { return cudaErrorInvalidValue; }
#undef AFF_B
#undef AFF_CASE
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_splitk_reduce(part, dalpha, K, ns, accumulate, stream);
}

}  // namespace bsrp
