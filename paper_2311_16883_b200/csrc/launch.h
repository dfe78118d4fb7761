// launch.h -- internal host-side launchers behind the C ABI (not exported).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <utility>

namespace bsrp {

// Process-wide count of kernels this library has launched (bsr_kernel_launches).
void count_launch(uint64_t n = 1);

// PDL launches.  pdl_flags() = the bsr_set_pdl bit mask (0: plain stream order):
//   1 prune triggers before its pack phase, 2 wgrad triggers at its start,
//   4 wgrad triggers at its epilogue, 8 split-K reduce triggers at its start,
//   16 / 32 / 64 PDL attribute on the wgrad / reduce / decompress launches,
//   128 PDL attribute on the small-N prune's first kernel (its second kernel always
//   chains to the first with PDL: they form one operation).
constexpr int kPdlDefault = 1 | 4 | 16 | 32 | 64 | 128;  // measured; bit 8 was slower
int pdl_flags();
// Launch `kern` with programmatic stream serialization: the kernel MUST call
// pdl_wait() (common.cuh) before touching global memory.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(bool on, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = on ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Workspace layout of bsr_prune (byte offsets; all 256-aligned).
struct PruneWs {
    size_t hdr, hist1, hist2, hist3, sstate, shist, cta_cnt, sumsq, slot, cand, total, zero_bytes;
};
constexpr int kMaxGrid = 2048;
PruneWs prune_ws_layout(int64_t N);
// bsr_prune_stochastic: the bsr_prune layout followed by the selection state,
// the refinement histograms, per-CTA tie counts and the boundary list.
constexpr int kStochMaxWindow = 4096;  // boundary pairs (the 2w boundary blocks are sorted in one CTA)
struct StochWs {
    PruneWs base;
    size_t state, shist, cta2, blist, total;
};
StochWs stoch_ws_layout(int64_t N);
cudaError_t launch_prune_stochastic(const void *X, int64_t M, int64_t K, int b, int es, int64_t k, int64_t window,
                                    double prob, uint64_t seed, int32_t *rowptr, int32_t *colidx, void *values,
                                    void *ws, cudaStream_t stream);

// Returns cudaSuccess or the launch error.
cudaError_t launch_prune(const void *X, int64_t M, int64_t K, int b, int es, int64_t k,
                         int32_t *rowptr, int32_t *colidx, void *values, void *ws,
                         cudaStream_t stream, int presummed = 0);
// Producer fusion: X = act(Z) and the block sums (into the prune workspace) in one pass.
cudaError_t launch_act_sumsq(const void *Z, void *X, int64_t M, int64_t K, int b, int es, int act, void *ws,
                             cudaStream_t stream);
cudaError_t launch_block_sumsq(const void *X, int64_t M, int64_t K, int b, int es, float *sumsq,
                               cudaStream_t stream);
cudaError_t launch_decompress(const int32_t *rowptr, const int32_t *colidx, const void *values,
                              int64_t M, int64_t K, int b, int es, void *Xout, cudaStream_t stream);

// Cross-rank global top-k steps (select_global.cu, prune.cu).
cudaError_t launch_select_hist(const void *X, int64_t M, int64_t K, int b, int es, int level, uint32_t prefix,
                               uint32_t *hist, void *ws, cudaStream_t stream);
cudaError_t launch_select_counts(int64_t M, int64_t K, int b, uint32_t T, int shift, uint64_t *counts, void *ws,
                                 cudaStream_t stream);
cudaError_t launch_prune_threshold(const void *X, int64_t M, int64_t K, int b, int es, uint32_t T, int shift,
                                   uint32_t tie_take, int64_t k, int32_t *rowptr, int32_t *colidx, void *values,
                                   void *ws, cudaStream_t stream, const uint64_t *gstate = nullptr);
// Device-side global selection (select_global.cu): the protocol state lives in device memory.
constexpr int kGStateWords = 16;
cudaError_t launch_gselect_init(int64_t k_total, uint64_t *state, cudaStream_t stream);
cudaError_t launch_gselect_hist(const void *X, int64_t M, int64_t K, int b, int es, int level, const uint64_t *state,
                                uint32_t *hist, void *ws, cudaStream_t stream);
cudaError_t launch_gselect_update(const uint32_t *hist_total, int level, uint64_t *state, cudaStream_t stream);
cudaError_t launch_gselect_counts(int64_t M, int64_t K, int b, const uint64_t *state, uint64_t *counts, void *ws,
                                  cudaStream_t stream);
cudaError_t launch_gselect_take(const uint64_t *all_counts, int world, int rank, uint64_t *state, cudaStream_t stream);

// Paper-faithful 1 x b per-sample variant (prune_rows.cu).
cudaError_t launch_prune_rows(const void *X, int64_t M, int64_t K, int b, int es, int64_t S, int64_t ks,
                              int32_t *rowptr, int32_t *colidx, void *values, void *ws, cudaStream_t stream);
cudaError_t launch_decompress_rows(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t M,
                                   int64_t K, int b, int es, void *out, cudaStream_t stream);
size_t wgrad_rows_ws_bytes(int64_t M, int64_t K, int64_t N);
cudaError_t launch_wgrad_rows(const int32_t *rowptr, const int32_t *colidx, const void *values, int es_x, int64_t M,
                              int64_t K, int b, const void *dY, int es_y, int64_t N, float *dW, int accumulate,
                              void *ws, cudaStream_t stream);

// dW = X_bsr^T dY, fp32 SIMT path (deterministic); split-K partials in ws.
size_t wgrad_simt_ws_bytes(int64_t M, int64_t K, int b, int64_t N);
cudaError_t launch_wgrad_simt(const int32_t *rowptr, const int32_t *colidx, const void *values,
                              int es_x, int64_t M, int64_t K, int b, const void *dY, int es_y,
                              int64_t N, float *dW, int accumulate, void *ws, cudaStream_t stream);

// dW = X_bsr^T dY on tcgen05 tensor cores.  kind: 0 = tf32 (fp32 operands),
// 1 = f16 (bf16 operands), 2 = FP32 grade (3xTF32, fp32 operands).
// algo: 0 auto, 1 per-run kernel, 2 span kernel (bsr_algo_t).
size_t wgrad_tc_ws_bytes(int64_t M, int64_t K, int b, int64_t N);
size_t wgrad_x3_ws_bytes(int64_t M, int64_t K, int b, int64_t N);
bool wgrad_tc_supported(int kind, int algo, int b, int64_t K, int64_t N);
cudaError_t launch_wgrad_tc(const int32_t *rowptr, const int32_t *colidx, const void *values,
                            int64_t nnzb, int kind, int algo, int64_t M, int64_t K, int b, const void *dY,
                            int64_t N, float *dW, int accumulate, void *ws, cudaStream_t stream,
                            float *mc = nullptr, int nk = 0, int mc_unicast = 0);
// dW^T (N x K) (+)= sum over nsplit K x N partials in ws, in split order (BSR_DW_NK layout).
cudaError_t launch_transpose_reduce(const float *ws, float *dWt, int64_t K, int64_t N, int nsplit, int accumulate,
                                    cudaStream_t stream);
bool wgrad_x3_native_nk(int64_t M, int64_t K, int b, int64_t N);
// bsr_validate: *bad = -1, or the lowest block row breaking the BSR invariants.
cudaError_t launch_validate(const int32_t *rowptr, const int32_t *colidx, int64_t nbr, int64_t nbc, int64_t nnzb,
                            int32_t *bad, cudaStream_t stream);

// Span kernel (wgrad_span.cu): dense-padded per-row spans, CTA-pair MMAs.
size_t wgrad_span_ws_bytes(int64_t M, int64_t K, int b, int64_t N);
cudaError_t launch_wgrad_span(const int32_t *rowptr, const int32_t *colidx, const void *values,
                              int64_t nnzb, int kind, int64_t M, int64_t K, int b, const void *dY,
                              int64_t N, float *dW, int accumulate, void *ws, cudaStream_t stream);
// Block-sparse affine layer (affine.cu): dalpha[c] = sum over kept blocks of x * dY in column c.
size_t affine_wgrad_ws_bytes(int64_t M, int64_t K, int b);
cudaError_t launch_affine_wgrad(const int32_t *rowptr, const int32_t *colidx, const void *values, int es_x,
                                int64_t M, int64_t K, int b, const void *dY, int es_y, float *dalpha,
                                int accumulate, void *ws, cudaStream_t stream);
// dW (+)= sum over nsplit partial K x N tiles in split order (deterministic).
cudaError_t launch_splitk_reduce(const float *ws, float *dW, int64_t n, int nsplit, int accumulate,
                                 cudaStream_t stream);

}  // namespace bsrp
