// abi.cu -- the exported C ABI (include/bsrprune.h): host-side validation,
// size queries, error reporting and dispatch to the sm_100a kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/bsrprune.h"
#include "launch.h"

namespace bsrp {
static std::atomic<uint64_t> g_launches{0};
static std::atomic<uint32_t> g_pdl{(uint32_t)kPdlDefault};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int pdl_flags() { return (int)g_pdl.load(std::memory_order_relaxed); }
}  // namespace bsrp

namespace {

thread_local std::string g_last_error;

bsr_status_t fail(bsr_status_t st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

bsr_status_t ok() {
    g_last_error.clear();
    return BSR_OK;
}

bsr_status_t cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return ok();
    return fail(BSR_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool supported_b(int32_t b) { return b == 4 || b == 8 || b == 16 || b == 32 || b == 64; }
int elem_size(int32_t dt) { return dt == BSR_DT_F32 ? 4 : dt == BSR_DT_BF16 ? 2 : 0; }
bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Byte ranges [a, a+na) and [b, b+nb) overlap.
bool overlap(const void *a, size_t na, const void *b, size_t nb) {
    if (!a || !b || na == 0 || nb == 0) return false;
    auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
    return x < y + nb && y < x + na;
}

bsr_status_t check_shape(int64_t M, int64_t K, int32_t b, int32_t dtype) {
    if (elem_size(dtype) == 0) return fail(BSR_ERR_INVALID_ARG, "dtype %d is not BSR_DT_F32 or BSR_DT_BF16", dtype);
    if (!supported_b(b)) return fail(BSR_ERR_UNSUPPORTED, "block size b=%d not in {4,8,16,32,64}", b);
    if (M <= 0 || K <= 0) return fail(BSR_ERR_SHAPE, "M=%lld and K=%lld must be positive", (long long)M, (long long)K);
    if (M % b != 0 || K % b != 0)
        return fail(BSR_ERR_SHAPE, "b=%d must divide M=%lld and K=%lld", b, (long long)M, (long long)K);
    if ((K * elem_size(dtype)) % 16 != 0)
        return fail(BSR_ERR_ALIGNMENT, "row pitch K*sizeof(elem)=%lld bytes is not a multiple of 16",
                    (long long)(K * elem_size(dtype)));
    const int64_t N = (M / b) * (K / b);
    if (N >= (int64_t(1) << 31) || M / b >= (int64_t(1) << 31) || M > (int64_t(1) << 40) || K > (int64_t(1) << 30))
        return fail(BSR_ERR_SHAPE, "shape too large (block count %lld must stay below 2^31)", (long long)N);
    return BSR_OK;
}

/* Dense rebuild for the tensor cores (block sizes the tcgen05 kernels cannot skip at,
 * and the 1 x b variant): the masked X is rebuilt densely in the workspace, viewed as a
 * keep-all 32 x 32 BSR (one copy pass) and contracted by the per-run tcgen05 kernel.
 * Workspace: [masked X: M*K elems][32x32 values: M*K elems][rowptr][colidx][TC partials]. */
constexpr int kDenseB = 32;
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
struct DenseTcWs {
    size_t xm, vals, rp, ci, tc, total;
};
bool dense_tc_shape_ok(int64_t M, int64_t K, int64_t N) {
    return M > 0 && K > 0 && N > 0 && M % kDenseB == 0 && K % kDenseB == 0 && N % 128 == 0 && K / kDenseB < 65536;
}
DenseTcWs dense_tc_layout(int64_t M, int64_t K, int64_t N, int es, int kind) {
    DenseTcWs w{};
    const int64_t nb = (M / kDenseB) * (K / kDenseB);
    size_t o = 0;
    w.xm = o;   o += align256((size_t)M * K * es);
    w.vals = o; o += align256((size_t)M * K * es);
    w.rp = o;   o += align256((size_t)(M / kDenseB + 1) * 4);
    w.ci = o;   o += align256((size_t)nb * 4);
    w.tc = o;
    o += align256(kind == 2 ? bsrp::wgrad_x3_ws_bytes(M, K, kDenseB, N) : bsrp::wgrad_tc_ws_bytes(M, K, kDenseB, N));
    w.total = o;
    return w;
}
// The masked X is in ws at w.xm: re-block it and run the tensor cores.
cudaError_t dense_tc_finish(int64_t M, int64_t K, int es, int kind, const void *dY, int64_t N, float *dW,
                            int accumulate, void *ws, const DenseTcWs &w, cudaStream_t s) {
    char *base = static_cast<char *>(ws);
    const int64_t nbk = (M / kDenseB) * (K / kDenseB);
    int32_t *rp = reinterpret_cast<int32_t *>(base + w.rp), *ci = reinterpret_cast<int32_t *>(base + w.ci);
    cudaError_t e = bsrp::launch_prune(base + w.xm, M, K, kDenseB, es, nbk, rp, ci, base + w.vals, nullptr, s);  // k = N
    if (e != cudaSuccess) return e;
    return bsrp::launch_wgrad_tc(rp, ci, base + w.vals, nbk, kind, BSR_ALGO_TC_RUNS, M, K, kDenseB, dY, N, dW, accumulate,
                                 base + w.tc, s);
}

bsr_status_t check_bsr(const bsr_t *A) {
    if (!A) return fail(BSR_ERR_INVALID_ARG, "BSR descriptor is NULL");
    bsr_status_t st = check_shape(A->M, A->K, A->b, A->dtype);
    if (st != BSR_OK) return st;
    const int64_t N = (A->M / A->b) * (A->K / A->b);
    if (A->nnzb < 0 || A->nnzb > N)
        return fail(BSR_ERR_INVALID_ARG, "nnzb=%lld outside [0, %lld]", (long long)A->nnzb, (long long)N);
    if (!A->rowptr) return fail(BSR_ERR_INVALID_ARG, "rowptr is NULL");
    if (A->nnzb > 0 && (!A->colidx || !A->values))
        return fail(BSR_ERR_INVALID_ARG, "colidx/values are NULL with nnzb=%lld", (long long)A->nnzb);
    if (A->values && !aligned16(A->values)) return fail(BSR_ERR_ALIGNMENT, "values is not 16-byte aligned");
    return BSR_OK;
}

}  // namespace

extern "C" {

int64_t bsr_num_blocks(int64_t M, int64_t K, int32_t b) {
    if (M <= 0 || K <= 0 || b <= 0 || M % b != 0 || K % b != 0) return -1;
    return (M / b) * (K / b);
}

int64_t bsr_keep_count(int64_t nblocks, double keep) {
    if (nblocks < 0 || !(keep >= 0.0 && keep <= 1.0)) return -1;
    int64_t k = (int64_t)std::floor(keep * (double)nblocks + 0.5);
    return k < 0 ? 0 : (k > nblocks ? nblocks : k);
}

size_t bsr_storage_bytes(int64_t M, int32_t b, int64_t k, int32_t dtype) {
    const int es = elem_size(dtype);
    if (M <= 0 || b <= 0 || M % b != 0 || k < 0 || es == 0) return 0;
    return (size_t)k * b * b * es + (size_t)k * 4 + (size_t)(M / b + 1) * 4;
}

size_t bsr_prune_workspace_bytes(int64_t M, int64_t K, int32_t b) {
    const int64_t N = bsr_num_blocks(M, K, b);
    if (N < 0 || !supported_b(b)) return 0;
    return bsrp::prune_ws_layout(N).total;
}

size_t bsr_wgrad_algo_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N, int32_t prec, int32_t algo) {
    if (bsr_num_blocks(M, K, b) < 0 || N <= 0) return 0;
    // the dense-rebuild tensor-core path: requested, or AUTO's choice below the native block sizes
    const bool dense = dense_tc_shape_ok(M, K, N) &&
                       (algo == BSR_ALGO_TC_DENSE || (algo == BSR_ALGO_AUTO && (prec == BSR_PREC_FP32 ? b < 32 : b < 16)));
    const int kind = prec == BSR_PREC_FP32 ? 2 : prec == BSR_PREC_TF32 ? 0 : 1;
    const size_t dws = dense ? dense_tc_layout(M, K, N, prec == BSR_PREC_BF16 ? 2 : 4, kind).total : 0;
    if (prec == BSR_PREC_FP32)
        return std::max({bsrp::wgrad_simt_ws_bytes(M, K, b, N), bsrp::wgrad_x3_ws_bytes(M, K, b, N), dws});
    return std::max(bsrp::wgrad_tc_ws_bytes(M, K, b, N), dws);
}

size_t bsr_wgrad_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N, int32_t prec) {
    return bsr_wgrad_algo_workspace_bytes(M, K, b, N, prec, BSR_ALGO_AUTO);
}

static bsr_status_t prune_impl(const void *X, int64_t M, int64_t K, int32_t b, int64_t k, int32_t dtype,
                               bsr_t *out, void *ws, size_t ws_bytes, void *stream, int presummed = 0) {
    bsr_status_t st = check_shape(M, K, b, dtype);
    if (st != BSR_OK) return st;
    const int64_t N = (M / b) * (K / b);
    if (k < 0 || k > N) return fail(BSR_ERR_INVALID_ARG, "k=%lld outside [0, N=%lld]", (long long)k, (long long)N);
    if (!X) return fail(BSR_ERR_INVALID_ARG, "X is NULL");
    if (!out) return fail(BSR_ERR_INVALID_ARG, "output BSR descriptor is NULL");
    if (!out->rowptr) return fail(BSR_ERR_INVALID_ARG, "out->rowptr is NULL");
    if (k > 0 && (!out->colidx || !out->values))
        return fail(BSR_ERR_INVALID_ARG, "out->colidx / out->values are NULL with k=%lld", (long long)k);
    if (!aligned16(X)) return fail(BSR_ERR_ALIGNMENT, "X is not 16-byte aligned");
    if (k > 0 && !aligned16(out->values)) return fail(BSR_ERR_ALIGNMENT, "out->values is not 16-byte aligned");
    const int es = elem_size(dtype);
    const size_t xbytes = (size_t)M * K * es;
    if (overlap(X, xbytes, out->values, (size_t)k * b * b * es) || overlap(X, xbytes, out->colidx, (size_t)k * 4) ||
        overlap(X, xbytes, out->rowptr, (size_t)(M / b + 1) * 4))
        return fail(BSR_ERR_INVALID_ARG, "X overlaps an output array");
    const size_t need = bsrp::prune_ws_layout(N).total;
    if (0 < k && k < N) {
        if (!ws || ws_bytes < need)
            return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, need);
        if (!aligned16(ws)) return fail(BSR_ERR_ALIGNMENT, "workspace is not 16-byte aligned");
    }
    if (presummed && !(ws && ws_bytes >= need)) return fail(BSR_ERR_WORKSPACE, "presummed prune needs the workspace");
    cudaError_t e = bsrp::launch_prune(X, M, K, b, es, k, out->rowptr, out->colidx, out->values, ws,
                                       static_cast<cudaStream_t>(stream), presummed);
    if (e != cudaSuccess) return cuda_status(e, "bsr_prune launch");
    out->M = M;
    out->K = K;
    out->b = b;
    out->dtype = dtype;
    out->nnzb = k;
    return ok();
}

bsr_status_t bsr_prune(const void *X, int64_t M, int64_t K, int32_t b, double keep, int32_t dtype, bsr_t *out,
                       void *ws, size_t ws_bytes, void *stream) {
    if (!(keep >= 0.0 && keep <= 1.0)) return fail(BSR_ERR_INVALID_ARG, "keep=%g must be in [0, 1]", keep);
    bsr_status_t st = check_shape(M, K, b, dtype);
    if (st != BSR_OK) return st;
    return prune_impl(X, M, K, b, bsr_keep_count((M / b) * (K / b), keep), dtype, out, ws, ws_bytes, stream);
}

bsr_status_t bsr_prune_k(const void *X, int64_t M, int64_t K, int32_t b, int64_t k, int32_t dtype, bsr_t *out,
                         void *ws, size_t ws_bytes, void *stream) {
    return prune_impl(X, M, K, b, k, dtype, out, ws, ws_bytes, stream);
}

size_t bsr_prune_stochastic_workspace_bytes(int64_t M, int64_t K, int32_t b) {
    const int64_t N = bsr_num_blocks(M, K, b);
    if (N < 0 || !supported_b(b)) return 0;
    return bsrp::stoch_ws_layout(N).total;
}

bsr_status_t bsr_prune_stochastic(const void *X, int64_t M, int64_t K, int32_t b, int64_t k, int64_t window,
                                  double p, uint64_t seed, int32_t dtype, bsr_t *out, void *ws, size_t ws_bytes,
                                  void *stream) {
    bsr_status_t st = check_shape(M, K, b, dtype);
    if (st != BSR_OK) return st;
    const int64_t N = (M / b) * (K / b);
    if (window < 0) return fail(BSR_ERR_INVALID_ARG, "window=%lld is negative", (long long)window);
    if (!(p >= 0.0 && p <= 1.0)) return fail(BSR_ERR_INVALID_ARG, "p=%g must be in [0, 1]", p);
    if (k < 0 || k > N) return fail(BSR_ERR_INVALID_ARG, "k=%lld outside [0, N=%lld]", (long long)k, (long long)N);
    const int64_t w = std::min<int64_t>(window, std::min<int64_t>(k, N - k));
    if (w > bsrp::kStochMaxWindow)
        return fail(BSR_ERR_INVALID_ARG, "window: min(window, k, N-k)=%lld exceeds %d", (long long)w,
                    bsrp::kStochMaxWindow);
    if (w == 0) return prune_impl(X, M, K, b, k, dtype, out, ws, ws_bytes, stream);
    if (!X) return fail(BSR_ERR_INVALID_ARG, "X is NULL");
    if (!out || !out->rowptr || !out->colidx || !out->values)
        return fail(BSR_ERR_INVALID_ARG, "output BSR descriptor or one of its arrays is NULL");
    if (!aligned16(X)) return fail(BSR_ERR_ALIGNMENT, "X is not 16-byte aligned");
    if (!aligned16(out->values)) return fail(BSR_ERR_ALIGNMENT, "out->values is not 16-byte aligned");
    const int es = elem_size(dtype);
    const size_t xbytes = (size_t)M * K * es;
    if (overlap(X, xbytes, out->values, (size_t)k * b * b * es) || overlap(X, xbytes, out->colidx, (size_t)k * 4) ||
        overlap(X, xbytes, out->rowptr, (size_t)(M / b + 1) * 4))
        return fail(BSR_ERR_INVALID_ARG, "X overlaps an output array");
    const size_t need = bsrp::stoch_ws_layout(N).total;
    if (!ws || ws_bytes < need)
        return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, need);
    if (!aligned16(ws)) return fail(BSR_ERR_ALIGNMENT, "workspace is not 16-byte aligned");
    cudaError_t e = bsrp::launch_prune_stochastic(X, M, K, b, es, k, window, p, seed, out->rowptr, out->colidx,
                                                  out->values, ws, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_status(e, "bsr_prune_stochastic launch");
    out->M = M;
    out->K = K;
    out->b = b;
    out->dtype = dtype;
    out->nnzb = k;
    return ok();
}

bsr_status_t bsr_block_sumsq(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype, float *sumsq,
                             void *stream) {
    bsr_status_t st = check_shape(M, K, b, dtype);
    if (st != BSR_OK) return st;
    if (!X || !sumsq) return fail(BSR_ERR_INVALID_ARG, "X or sumsq is NULL");
    if (!aligned16(X)) return fail(BSR_ERR_ALIGNMENT, "X is not 16-byte aligned");
    return cuda_status(bsrp::launch_block_sumsq(X, M, K, b, elem_size(dtype), sumsq, static_cast<cudaStream_t>(stream)),
                       "bsr_block_sumsq launch");
}

/* ---- cross-rank global top-k (select_global.cu) ---- */
static bsr_status_t check_ws(int64_t N, void *ws, size_t ws_bytes) {
    const size_t need = bsrp::prune_ws_layout(N).total;
    if (!ws || ws_bytes < need)
        return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, need);
    if (!aligned16(ws)) return fail(BSR_ERR_ALIGNMENT, "workspace is not 16-byte aligned");
    return BSR_OK;
}

bsr_status_t bsr_select_hist(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype, int32_t level,
                             uint32_t prefix, uint32_t *hist, void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_shape(M, K, b, dtype);
    if (st != BSR_OK) return st;
    if (level < 0 || level > 2) return fail(BSR_ERR_INVALID_ARG, "level=%d must be 0, 1 or 2", level);
    if (!hist) return fail(BSR_ERR_INVALID_ARG, "hist is NULL");
    if (level == 0 && !X) return fail(BSR_ERR_INVALID_ARG, "X is NULL");
    if (level == 0 && !aligned16(X)) return fail(BSR_ERR_ALIGNMENT, "X is not 16-byte aligned");
    st = check_ws((M / b) * (K / b), ws, ws_bytes);
    if (st != BSR_OK) return st;
    return cuda_status(bsrp::launch_select_hist(X, M, K, b, elem_size(dtype), level, prefix, hist, ws,
                                                static_cast<cudaStream_t>(stream)),
                       "bsr_select_hist launch");
}

bsr_status_t bsr_select_counts(int64_t M, int64_t K, int32_t b, uint32_t threshold, int32_t shift, uint64_t *counts,
                               void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_shape(M, K, b, BSR_DT_F32);
    if (st != BSR_OK) return st;
    if (shift != 0 && shift != 9 && shift != 19) return fail(BSR_ERR_INVALID_ARG, "shift=%d must be 0, 9 or 19", shift);
    if (!counts) return fail(BSR_ERR_INVALID_ARG, "counts is NULL");
    st = check_ws((M / b) * (K / b), ws, ws_bytes);
    if (st != BSR_OK) return st;
    return cuda_status(bsrp::launch_select_counts(M, K, b, threshold, shift, counts, ws,
                                                  static_cast<cudaStream_t>(stream)),
                       "bsr_select_counts launch");
}

bsr_status_t bsr_prune_threshold(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype, uint32_t threshold,
                                 int32_t shift, int64_t tie_take, int64_t k, bsr_t *out, void *ws, size_t ws_bytes,
                                 void *stream) {
    bsr_status_t st = check_shape(M, K, b, dtype);
    if (st != BSR_OK) return st;
    const int64_t N = (M / b) * (K / b);
    if (shift != 0 && shift != 9 && shift != 19) return fail(BSR_ERR_INVALID_ARG, "shift=%d must be 0, 9 or 19", shift);
    if (k < 0 || k > N) return fail(BSR_ERR_INVALID_ARG, "k=%lld outside [0, N=%lld]", (long long)k, (long long)N);
    if (tie_take < 0 || tie_take > k) return fail(BSR_ERR_INVALID_ARG, "tie_take=%lld outside [0, k]", (long long)tie_take);
    if (!X) return fail(BSR_ERR_INVALID_ARG, "X is NULL");
    if (!out || !out->rowptr) return fail(BSR_ERR_INVALID_ARG, "output BSR descriptor / rowptr is NULL");
    if (k > 0 && (!out->colidx || !out->values))
        return fail(BSR_ERR_INVALID_ARG, "out->colidx / out->values are NULL with k=%lld", (long long)k);
    if (!aligned16(X)) return fail(BSR_ERR_ALIGNMENT, "X is not 16-byte aligned");
    if (k > 0 && !aligned16(out->values)) return fail(BSR_ERR_ALIGNMENT, "out->values is not 16-byte aligned");
    st = check_ws(N, ws, ws_bytes);
    if (st != BSR_OK) return st;
    cudaError_t e = bsrp::launch_prune_threshold(X, M, K, b, elem_size(dtype), threshold, shift, (uint32_t)tie_take, k,
                                                 out->rowptr, out->colidx, out->values, ws,
                                                 static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_status(e, "bsr_prune_threshold launch");
    out->M = M;
    out->K = K;
    out->b = b;
    out->dtype = dtype;
    out->nnzb = k;
    return ok();
}

/* ---- device-side global selection (no host round trips; select_global.cu) ---- */
size_t bsr_gselect_state_bytes(void) { return bsrp::kGStateWords * sizeof(uint64_t); }

bsr_status_t bsr_gselect_init(int64_t k_total, uint64_t *state, void *stream) {
    if (k_total < 0) return fail(BSR_ERR_INVALID_ARG, "k_total=%lld < 0", (long long)k_total);
    if (!state) return fail(BSR_ERR_INVALID_ARG, "state is NULL");
    return cuda_status(bsrp::launch_gselect_init(k_total, state, static_cast<cudaStream_t>(stream)), "bsr_gselect_init");
}

bsr_status_t bsr_gselect_hist(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype, int32_t level,
                              const uint64_t *state, uint32_t *hist, void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_shape(M, K, b, dtype);
    if (st != BSR_OK) return st;
    if (level < 0 || level > 2) return fail(BSR_ERR_INVALID_ARG, "level=%d must be 0, 1 or 2", level);
    if (!state || !hist) return fail(BSR_ERR_INVALID_ARG, "state or hist is NULL");
    if (level == 0 && !X) return fail(BSR_ERR_INVALID_ARG, "X is NULL");
    if (level == 0 && !aligned16(X)) return fail(BSR_ERR_ALIGNMENT, "X is not 16-byte aligned");
    st = check_ws((M / b) * (K / b), ws, ws_bytes);
    if (st != BSR_OK) return st;
    return cuda_status(bsrp::launch_gselect_hist(X, M, K, b, elem_size(dtype), level, state, hist, ws,
                                                 static_cast<cudaStream_t>(stream)),
                       "bsr_gselect_hist launch");
}

bsr_status_t bsr_gselect_update(const uint32_t *hist_total, int32_t level, uint64_t *state, void *stream) {
    if (level < 0 || level > 2) return fail(BSR_ERR_INVALID_ARG, "level=%d must be 0, 1 or 2", level);
    if (!state || !hist_total) return fail(BSR_ERR_INVALID_ARG, "state or hist_total is NULL");
    return cuda_status(bsrp::launch_gselect_update(hist_total, level, state, static_cast<cudaStream_t>(stream)),
                       "bsr_gselect_update launch");
}

bsr_status_t bsr_gselect_counts(int64_t M, int64_t K, int32_t b, const uint64_t *state, uint64_t *counts, void *ws,
                                size_t ws_bytes, void *stream) {
    bsr_status_t st = check_shape(M, K, b, BSR_DT_F32);
    if (st != BSR_OK) return st;
    if (!state || !counts) return fail(BSR_ERR_INVALID_ARG, "state or counts is NULL");
    st = check_ws((M / b) * (K / b), ws, ws_bytes);
    if (st != BSR_OK) return st;
    return cuda_status(bsrp::launch_gselect_counts(M, K, b, state, counts, ws, static_cast<cudaStream_t>(stream)),
                       "bsr_gselect_counts launch");
}

bsr_status_t bsr_gselect_take(const uint64_t *all_counts, int32_t world, int32_t rank, uint64_t *state, void *stream) {
    if (world < 1 || rank < 0 || rank >= world)
        return fail(BSR_ERR_INVALID_ARG, "rank=%d outside [0, world=%d)", rank, world);
    if (!state || !all_counts) return fail(BSR_ERR_INVALID_ARG, "state or all_counts is NULL");
    return cuda_status(bsrp::launch_gselect_take(all_counts, world, rank, state, static_cast<cudaStream_t>(stream)),
                       "bsr_gselect_take launch");
}

bsr_status_t bsr_prune_gselect(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype, const uint64_t *state,
                               int64_t capacity, bsr_t *out, void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_shape(M, K, b, dtype);
    if (st != BSR_OK) return st;
    const int64_t N = (M / b) * (K / b);
    if (capacity < 0 || capacity > N)
        return fail(BSR_ERR_INVALID_ARG, "capacity=%lld outside [0, N=%lld]", (long long)capacity, (long long)N);
    if (!X || !state) return fail(BSR_ERR_INVALID_ARG, "X or state is NULL");
    if (!out || !out->rowptr) return fail(BSR_ERR_INVALID_ARG, "output BSR descriptor / rowptr is NULL");
    if (capacity > 0 && (!out->colidx || !out->values))
        return fail(BSR_ERR_INVALID_ARG, "out->colidx / out->values are NULL with capacity=%lld", (long long)capacity);
    if (!aligned16(X)) return fail(BSR_ERR_ALIGNMENT, "X is not 16-byte aligned");
    if (capacity > 0 && !aligned16(out->values)) return fail(BSR_ERR_ALIGNMENT, "out->values is not 16-byte aligned");
    st = check_ws(N, ws, ws_bytes);
    if (st != BSR_OK) return st;
    cudaError_t e = bsrp::launch_prune_threshold(X, M, K, b, elem_size(dtype), 0u, 0, 0u, capacity, out->rowptr,
                                                 out->colidx, out->values, ws, static_cast<cudaStream_t>(stream), state);
    if (e != cudaSuccess) return cuda_status(e, "bsr_prune_gselect launch");
    out->M = M;
    out->K = K;
    out->b = b;
    out->dtype = dtype;
    out->nnzb = capacity;
    return ok();
}

/* ---- paper-faithful 1 x b per-sample variant (prune_rows.cu) ---- */
size_t bsr_prune_rows_workspace_bytes(int64_t M, int64_t K, int32_t b) {
    if (M <= 0 || K <= 0 || !supported_b(b) || K % b) return 0;
    return ((size_t)M * (K / b) * 4 + 255) & ~(size_t)255;
}

int64_t bsr_rows_keep_per_sample(int64_t sample_rows, int64_t K, int32_t b, double keep) {
    if (sample_rows <= 0 || K <= 0 || b <= 0 || K % b) return -1;
    return bsr_keep_count(sample_rows * (K / b), keep);
}

static bsr_status_t check_rows(int64_t M, int64_t K, int32_t b, int32_t dtype) {
    if (elem_size(dtype) == 0) return fail(BSR_ERR_INVALID_ARG, "dtype %d is not BSR_DT_F32 or BSR_DT_BF16", dtype);
    if (!supported_b(b)) return fail(BSR_ERR_UNSUPPORTED, "block size b=%d not in {4,8,16,32,64}", b);
    if (M <= 0 || K <= 0 || K % b) return fail(BSR_ERR_SHAPE, "b=%d must divide K=%lld (M=%lld)", b, (long long)K, (long long)M);
    if ((K * elem_size(dtype)) % 16) return fail(BSR_ERR_ALIGNMENT, "row pitch of X (K=%lld) is not a multiple of 16 bytes", (long long)K);
    return BSR_OK;
}

bsr_status_t bsr_prune_rows(const void *X, int64_t M, int64_t K, int32_t b, int64_t sample_rows, double keep,
                            int32_t dtype, int32_t *rowptr, int32_t *colidx, void *values, void *ws, size_t ws_bytes,
                            void *stream) {
    bsr_status_t st = check_rows(M, K, b, dtype);
    if (st != BSR_OK) return st;
    if (!(keep >= 0.0 && keep <= 1.0)) return fail(BSR_ERR_INVALID_ARG, "keep=%g must be in [0, 1]", keep);
    if (sample_rows <= 0 || M % sample_rows)
        return fail(BSR_ERR_SHAPE, "sample_rows=%lld must divide M=%lld", (long long)sample_rows, (long long)M);
    const int64_t ks = bsr_rows_keep_per_sample(sample_rows, K, b, keep);
    if (!X || !rowptr) return fail(BSR_ERR_INVALID_ARG, "X or rowptr is NULL");
    if (ks > 0 && (!colidx || !values)) return fail(BSR_ERR_INVALID_ARG, "colidx / values are NULL with k > 0");
    if (!aligned16(X) || (ks > 0 && !aligned16(values))) return fail(BSR_ERR_ALIGNMENT, "X or values is not 16-byte aligned");
    const size_t need = bsr_prune_rows_workspace_bytes(M, K, b);
    if (!ws || ws_bytes < need)
        return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, need);
    return cuda_status(bsrp::launch_prune_rows(X, M, K, b, elem_size(dtype), sample_rows, ks, rowptr, colidx, values,
                                               ws, static_cast<cudaStream_t>(stream)),
                       "bsr_prune_rows launch");
}

bsr_status_t bsr_decompress_rows(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t M,
                                 int64_t K, int32_t b, int32_t dtype, void *X_out, void *stream) {
    bsr_status_t st = check_rows(M, K, b, dtype);
    if (st != BSR_OK) return st;
    if (!rowptr || !X_out) return fail(BSR_ERR_INVALID_ARG, "rowptr or X_out is NULL");
    if (!aligned16(X_out)) return fail(BSR_ERR_ALIGNMENT, "X_out is not 16-byte aligned");
    return cuda_status(bsrp::launch_decompress_rows(rowptr, colidx, values, M, K, b, elem_size(dtype), X_out,
                                                    static_cast<cudaStream_t>(stream)),
                       "bsr_decompress_rows launch");
}

size_t bsr_wgrad_rows_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N) {
    if (M <= 0 || K <= 0 || N <= 0 || !supported_b(b) || K % b) return 0;
    return bsrp::wgrad_rows_ws_bytes(M, K, N);
}

bsr_status_t bsr_wgrad_rows(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnz, int64_t M,
                            int64_t K, int32_t b, int32_t x_dtype, const void *dY, int32_t dy_dtype, int64_t N,
                            float *dW, int32_t accumulate, void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_rows(M, K, b, x_dtype);
    if (st != BSR_OK) return st;
    const int esy = elem_size(dy_dtype);
    if (esy == 0) return fail(BSR_ERR_INVALID_ARG, "dy_dtype %d is not BSR_DT_F32 or BSR_DT_BF16", dy_dtype);
    if (N <= 0 || (N * esy) % 16 || (N * 4) % 16)
        return fail(BSR_ERR_ALIGNMENT, "row pitch of dY/dW (N=%lld) is not a multiple of 16 bytes", (long long)N);
    if (!rowptr || !dY || !dW) return fail(BSR_ERR_INVALID_ARG, "rowptr, dY or dW is NULL");
    if (nnz > 0 && (!colidx || !values)) return fail(BSR_ERR_INVALID_ARG, "colidx / values are NULL with nnz > 0");
    if (accumulate != 0 && accumulate != 1) return fail(BSR_ERR_INVALID_ARG, "accumulate must be 0 or 1");
    const size_t need = bsrp::wgrad_rows_ws_bytes(M, K, N);
    if (need && (!ws || ws_bytes < need))
        return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, need);
    return cuda_status(bsrp::launch_wgrad_rows(rowptr, colidx, nnz > 0 ? values : nullptr, elem_size(x_dtype), M, K, b,
                                               dY, esy, N, dW, accumulate, ws, static_cast<cudaStream_t>(stream)),
                       "bsr_wgrad_rows launch");
}

size_t bsr_wgrad_rows_tc_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N, int32_t x_dtype) {
    if (M <= 0 || K <= 0 || N <= 0 || !supported_b(b) || K % b || elem_size(x_dtype) == 0) return 0;
    if (!dense_tc_shape_ok(M, K, N)) return 0;
    return dense_tc_layout(M, K, N, elem_size(x_dtype), x_dtype == BSR_DT_F32 ? 2 : 1).total;
}

bsr_status_t bsr_wgrad_rows_tc(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnz, int64_t M,
                               int64_t K, int32_t b, int32_t x_dtype, const void *dY, int32_t dy_dtype, int64_t N,
                               float *dW, int32_t accumulate, void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_rows(M, K, b, x_dtype);
    if (st != BSR_OK) return st;
    if (dy_dtype != x_dtype) return fail(BSR_ERR_UNSUPPORTED, "tensor-core 1 x b dW needs dY in the dtype of X");
    if (!dense_tc_shape_ok(M, K, N))
        return fail(BSR_ERR_UNSUPPORTED, "tensor-core 1 x b dW needs 32 | M, 32 | K, N %% 128 == 0 (M=%lld, K=%lld, N=%lld)",
                    (long long)M, (long long)K, (long long)N);
    if (!rowptr || !dY || !dW) return fail(BSR_ERR_INVALID_ARG, "rowptr, dY or dW is NULL");
    if (nnz > 0 && (!colidx || !values)) return fail(BSR_ERR_INVALID_ARG, "colidx / values are NULL with nnz > 0");
    if (accumulate != 0 && accumulate != 1) return fail(BSR_ERR_INVALID_ARG, "accumulate must be 0 or 1");
    if (!aligned16(dY) || !aligned16(dW)) return fail(BSR_ERR_ALIGNMENT, "dY or dW is not 16-byte aligned");
    const int es = elem_size(x_dtype);
    const DenseTcWs w = dense_tc_layout(M, K, N, es, es == 4 ? 2 : 1);
    if (!ws || ws_bytes < w.total)
        return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, w.total);
    if (!aligned16(ws)) return fail(BSR_ERR_ALIGNMENT, "workspace is not 16-byte aligned");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = bsrp::launch_decompress_rows(rowptr, colidx, nnz > 0 ? values : nullptr, M, K, b, es,
                                                 static_cast<char *>(ws) + w.xm, s);
    if (e != cudaSuccess) return cuda_status(e, "bsr_wgrad_rows_tc (masked rows)");
    return cuda_status(dense_tc_finish(M, K, es, es == 4 ? 2 : 1, dY, N, dW, accumulate, ws, w, s),
                       "bsr_wgrad_rows_tc launch");
}

/* ---- producer fusion ---- */
bsr_status_t bsr_act_block_sumsq(const void *Z, void *X_out, int64_t M, int64_t K, int32_t b, int32_t dtype,
                                 int32_t act, void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_shape(M, K, b, dtype);
    if (st != BSR_OK) return st;
    if (act != 0 && act != 1) return fail(BSR_ERR_INVALID_ARG, "act=%d must be 0 (identity) or 1 (GELU, tanh form)", act);
    if (!Z || !X_out) return fail(BSR_ERR_INVALID_ARG, "Z or X_out is NULL");
    if (!aligned16(Z) || !aligned16(X_out)) return fail(BSR_ERR_ALIGNMENT, "Z or X_out is not 16-byte aligned");
    const size_t xb = (size_t)M * K * elem_size(dtype);
    if (Z != X_out && overlap(Z, xb, X_out, xb)) return fail(BSR_ERR_INVALID_ARG, "Z and X_out overlap partially");
    const size_t need = bsrp::prune_ws_layout((M / b) * (K / b)).total;
    if (!ws || ws_bytes < need)
        return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, need);
    return cuda_status(bsrp::launch_act_sumsq(Z, X_out, M, K, b, elem_size(dtype), act, ws,
                                              static_cast<cudaStream_t>(stream)),
                       "bsr_act_block_sumsq launch");
}

bsr_status_t bsr_prune_presummed(const void *X, int64_t M, int64_t K, int32_t b, int64_t k, int32_t dtype, bsr_t *out,
                                 void *ws, size_t ws_bytes, void *stream) {
    return prune_impl(X, M, K, b, k, dtype, out, ws, ws_bytes, stream, 1);
}

bsr_status_t bsr_validate(const bsr_t *A, int32_t *bad_row, void *stream) {
    bsr_status_t st = check_bsr(A);
    if (st != BSR_OK) return st;
    if (!bad_row) return fail(BSR_ERR_INVALID_ARG, "bad_row is NULL");
    if (A->nnzb > 0 && !A->colidx) return fail(BSR_ERR_INVALID_ARG, "colidx is NULL with nnzb > 0");
    return cuda_status(bsrp::launch_validate(A->rowptr, A->colidx, A->M / A->b, A->K / A->b, A->nnzb, bad_row,
                                             static_cast<cudaStream_t>(stream)),
                       "bsr_validate launch");
}

bsr_status_t bsr_decompress(const bsr_t *A, void *X_out, void *stream) {
    bsr_status_t st = check_bsr(A);
    if (st != BSR_OK) return st;
    if (!X_out) return fail(BSR_ERR_INVALID_ARG, "X_out is NULL");
    if (!aligned16(X_out)) return fail(BSR_ERR_ALIGNMENT, "X_out is not 16-byte aligned");
    return cuda_status(bsrp::launch_decompress(A->rowptr, A->colidx, A->values, A->M, A->K, A->b,
                                               elem_size(A->dtype), X_out, static_cast<cudaStream_t>(stream)),
                       "bsr_decompress launch");
}

static bsr_status_t check_wgrad_ws(size_t need, void *ws, size_t ws_bytes, const float *dW, size_t dw_bytes) {
    if (need && (!ws || ws_bytes < need))
        return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, need);
    if (need && !aligned16(ws)) return fail(BSR_ERR_ALIGNMENT, "workspace is not 16-byte aligned");
    if (need && overlap(ws, need, dW, dw_bytes)) return fail(BSR_ERR_INVALID_ARG, "workspace overlaps dW");
    return BSR_OK;
}

bsr_status_t bsr_wgrad_algo(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N, float *dW,
                            int32_t accumulate, int32_t prec, int32_t algo, void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_bsr(A);
    if (st != BSR_OK) return st;
    const int esy = elem_size(dy_dtype);
    if (esy == 0) return fail(BSR_ERR_INVALID_ARG, "dy_dtype %d is not BSR_DT_F32 or BSR_DT_BF16", dy_dtype);
    if (N <= 0 || N > (int64_t(1) << 30)) return fail(BSR_ERR_SHAPE, "N=%lld out of range", (long long)N);
    if (!dY || !dW) return fail(BSR_ERR_INVALID_ARG, "dY or dW is NULL");
    if (accumulate != 0 && accumulate != 1) return fail(BSR_ERR_INVALID_ARG, "accumulate must be 0 or 1");
    if (algo < BSR_ALGO_AUTO || algo > BSR_ALGO_TC_DENSE) return fail(BSR_ERR_INVALID_ARG, "algo %d is not a bsr_algo_t", algo);
    if (!aligned16(dY) || !aligned16(dW)) return fail(BSR_ERR_ALIGNMENT, "dY or dW is not 16-byte aligned");
    if ((N * esy) % 16 != 0 || (N * 4) % 16 != 0)
        return fail(BSR_ERR_ALIGNMENT, "row pitch of dY/dW (N=%lld) is not a multiple of 16 bytes", (long long)N);
    const int esx = elem_size(A->dtype);
    const size_t dw_bytes = (size_t)A->K * N * 4;
    if (overlap(dW, dw_bytes, dY, (size_t)A->M * N * esy)) return fail(BSR_ERR_INVALID_ARG, "dW overlaps dY");
    if (A->K / A->b > 65535)
        return fail(BSR_ERR_UNSUPPORTED, "K/b must stay below 65536 (K/b=%lld)", (long long)(A->K / A->b));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (prec != BSR_PREC_FP32 && prec != BSR_PREC_TF32 && prec != BSR_PREC_BF16)
        return fail(BSR_ERR_INVALID_ARG, "prec %d is not a bsr_prec_t", prec);
    // dense rebuild on the tensor cores: chosen by AUTO below the native block sizes
    const int dkind = prec == BSR_PREC_FP32 ? 2 : prec == BSR_PREC_TF32 ? 0 : 1;
    const int dwant = prec == BSR_PREC_BF16 ? BSR_DT_BF16 : BSR_DT_F32;
    const bool dense_ok = A->dtype == dwant && dy_dtype == dwant && dense_tc_shape_ok(A->M, A->K, N);
    const bool dense_auto = dense_ok && algo == BSR_ALGO_AUTO && (prec == BSR_PREC_FP32 ? A->b < 32 : A->b < 16);
    if (algo == BSR_ALGO_TC_DENSE || dense_auto) {
        if (!dense_ok)
            return fail(BSR_ERR_UNSUPPORTED, "dense-rebuild tensor-core dW needs %s values and dY, 32 | M, 32 | K, "
                                             "N %% 128 == 0", dwant == BSR_DT_BF16 ? "bf16" : "fp32");
        const DenseTcWs w = dense_tc_layout(A->M, A->K, N, elem_size(dwant), dkind);
        st = check_wgrad_ws(w.total, ws, ws_bytes, dW, dw_bytes);
        if (st != BSR_OK) return st;
        cudaError_t e = bsrp::launch_decompress(A->rowptr, A->colidx, A->nnzb ? A->values : nullptr, A->M, A->K, A->b,
                                                esx, static_cast<char *>(ws) + w.xm, s);
        if (e != cudaSuccess) return cuda_status(e, "bsr_wgrad (dense rebuild)");
        return cuda_status(dense_tc_finish(A->M, A->K, esx, dkind, dY, N, dW, accumulate, ws, w, s),
                           "bsr_wgrad (dense rebuild, tensor cores) launch");
    }
    if (prec == BSR_PREC_FP32) {
        // FP32 grade: 3xTF32 tensor cores where implemented, else FFMA
        const bool x3 = A->dtype == BSR_DT_F32 && dy_dtype == BSR_DT_F32 &&
                        bsrp::wgrad_tc_supported(2, algo == BSR_ALGO_AUTO ? 1 : algo, A->b, A->K, N);
        if (algo == BSR_ALGO_TC_SPAN || (algo == BSR_ALGO_TC_RUNS && !x3))
            return fail(BSR_ERR_UNSUPPORTED, "FP32-grade tensor-core dW needs the per-run kernel, f32 values and dY, "
                                             "b in {32, 64} and N %% 128 == 0");
        if (x3 && algo != BSR_ALGO_SIMT) {
            st = check_wgrad_ws(bsrp::wgrad_x3_ws_bytes(A->M, A->K, A->b, N), ws, ws_bytes, dW, dw_bytes);
            if (st != BSR_OK) return st;
            return cuda_status(bsrp::launch_wgrad_tc(A->rowptr, A->colidx, A->values, A->nnzb, 2, BSR_ALGO_TC_RUNS,
                                                     A->M, A->K, A->b, dY, N, dW, accumulate, ws, s),
                               "bsr_wgrad (fp32 grade, 3xTF32) launch");
        }
        st = check_wgrad_ws(bsrp::wgrad_simt_ws_bytes(A->M, A->K, A->b, N), ws, ws_bytes, dW, dw_bytes);
        if (st != BSR_OK) return st;
        return cuda_status(bsrp::launch_wgrad_simt(A->rowptr, A->colidx, A->nnzb ? A->values : nullptr, esx, A->M, A->K,
                                                   A->b, dY, esy, N, dW, accumulate, ws, s),
                           "bsr_wgrad (fp32) launch");
    }
    const int want = prec == BSR_PREC_TF32 ? BSR_DT_F32 : BSR_DT_BF16;
    if (A->dtype != want || dy_dtype != want)
        return fail(BSR_ERR_UNSUPPORTED, "%s tensor-core path needs %s values and dY", prec == BSR_PREC_TF32 ? "TF32" : "BF16",
                    prec == BSR_PREC_TF32 ? "fp32" : "bf16");
    if (algo == BSR_ALGO_SIMT) return fail(BSR_ERR_UNSUPPORTED, "the FFMA kernel implements BSR_PREC_FP32 only");
    if (A->b < 16) return fail(BSR_ERR_UNSUPPORTED, "tensor-core path needs b >= 16 (b=%d)", A->b);
    if (N % 128 != 0) return fail(BSR_ERR_UNSUPPORTED, "tensor-core path needs N %% 128 == 0 (N=%lld)", (long long)N);
    const int kind = prec == BSR_PREC_TF32 ? 0 : 1;
    if (!bsrp::wgrad_tc_supported(kind, algo, A->b, A->K, N))
        return fail(BSR_ERR_UNSUPPORTED, "tensor-core kernel family %d does not implement %s at b=%d, K=%lld", algo,
                    prec == BSR_PREC_TF32 ? "tf32" : "bf16", A->b, (long long)A->K);
    st = check_wgrad_ws(bsrp::wgrad_tc_ws_bytes(A->M, A->K, A->b, N), ws, ws_bytes, dW, dw_bytes);
    if (st != BSR_OK) return st;
    return cuda_status(bsrp::launch_wgrad_tc(A->rowptr, A->colidx, A->values, A->nnzb, kind, algo, A->M, A->K, A->b, dY,
                                             N, dW, accumulate, ws, s),
                       "bsr_wgrad (tensor-core) launch");
}

size_t bsr_wgrad_nk_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N, int32_t prec, int32_t algo) {
    if (bsr_num_blocks(M, K, b) < 0 || N <= 0) return 0;
    return align256(bsr_wgrad_algo_workspace_bytes(M, K, b, N, prec, algo)) + align256((size_t)K * N * sizeof(float));
}

bsr_status_t bsr_wgrad_nk(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N, float *dWt, int32_t accumulate,
                          int32_t prec, int32_t algo, void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_bsr(A);
    if (st != BSR_OK) return st;
    if (N <= 0 || N > (int64_t(1) << 30)) return fail(BSR_ERR_SHAPE, "N=%lld out of range", (long long)N);
    if (!dY || !dWt) return fail(BSR_ERR_INVALID_ARG, "dY or dWt is NULL");
    if (accumulate != 0 && accumulate != 1) return fail(BSR_ERR_INVALID_ARG, "accumulate must be 0 or 1");
    if (!aligned16(dWt)) return fail(BSR_ERR_ALIGNMENT, "dWt is not 16-byte aligned");
    const int esy = elem_size(dy_dtype);
    if (esy == 0) return fail(BSR_ERR_INVALID_ARG, "dy_dtype %d is not BSR_DT_F32 or BSR_DT_BF16", dy_dtype);
    const size_t dw_bytes = (size_t)A->K * N * 4;
    if (overlap(dWt, dw_bytes, dY, (size_t)A->M * N * esy)) return fail(BSR_ERR_INVALID_ARG, "dWt overlaps dY");
    const size_t inner = bsr_wgrad_algo_workspace_bytes(A->M, A->K, A->b, N, prec, algo);
    const size_t need = align256(inner) + align256(dw_bytes);
    st = check_wgrad_ws(need, ws, ws_bytes, dWt, dw_bytes);
    if (st != BSR_OK) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // native: the FP32-grade per-run kernel's chain-capped split-K reduce stores dW^T directly
    const bool dense_auto = algo == BSR_ALGO_AUTO && A->b < 32;
    if (prec == BSR_PREC_FP32 && !dense_auto && (algo == BSR_ALGO_AUTO || algo == BSR_ALGO_TC_RUNS) &&
        A->dtype == BSR_DT_F32 && dy_dtype == BSR_DT_F32 && A->nnzb > 0 && aligned16(dY) && (N * 4) % 16 == 0 &&
        bsrp::wgrad_tc_supported(2, BSR_ALGO_TC_RUNS, A->b, A->K, N) && bsrp::wgrad_x3_native_nk(A->M, A->K, A->b, N)) {
        cudaError_t e = bsrp::launch_wgrad_tc(A->rowptr, A->colidx, A->values, A->nnzb, 2, BSR_ALGO_TC_RUNS, A->M,
                                              A->K, A->b, dY, N, dWt, accumulate, ws, s, nullptr, 1);
        if (e != cudaErrorNotSupported) return cuda_status(e, "bsr_wgrad_nk (fp32 grade, 3xTF32) launch");
        (void)cudaGetLastError();
    }
    // any other path: dW (K x N) into the workspace's tail, then one transposing pass
    float *scratch = reinterpret_cast<float *>(static_cast<char *>(ws) + align256(inner));
    st = bsr_wgrad_algo(A, dY, dy_dtype, N, scratch, 0, prec, algo, inner ? ws : nullptr, inner, stream);
    if (st != BSR_OK) return st;
    return cuda_status(bsrp::launch_transpose_reduce(scratch, dWt, A->K, N, 1, accumulate, s), "bsr_wgrad_nk transpose");
}

bsr_status_t bsr_wgrad(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N, float *dW, int32_t accumulate,
                       int32_t prec, void *ws, size_t ws_bytes, void *stream) {
    return bsr_wgrad_algo(A, dY, dy_dtype, N, dW, accumulate, prec, BSR_ALGO_AUTO, ws, ws_bytes, stream);
}

static bsr_status_t wgrad_multicast_impl(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N, float *mc_dW,
                                         int32_t prec, int32_t algo, void *ws, size_t ws_bytes, void *stream,
                                         int unicast) {
    bsr_status_t st = check_bsr(A);
    if (st != BSR_OK) return st;
    const int esy = elem_size(dy_dtype);
    if (esy == 0) return fail(BSR_ERR_INVALID_ARG, "dy_dtype %d is not BSR_DT_F32 or BSR_DT_BF16", dy_dtype);
    if (N <= 0 || N > (int64_t(1) << 30)) return fail(BSR_ERR_SHAPE, "N=%lld out of range", (long long)N);
    if (!dY || !mc_dW) return fail(BSR_ERR_INVALID_ARG, "dY or mc_dW is NULL");
    if (!aligned16(dY) || !aligned16(mc_dW)) return fail(BSR_ERR_ALIGNMENT, "dY or mc_dW is not 16-byte aligned");
    if (algo != BSR_ALGO_AUTO && algo != BSR_ALGO_TC_RUNS)
        return fail(BSR_ERR_UNSUPPORTED, "the fused multicast dW exists in the per-run tensor-core kernel only");
    int kind = -1;
    if (prec == BSR_PREC_FP32 && A->dtype == BSR_DT_F32 && dy_dtype == BSR_DT_F32) kind = 2;
    if (prec == BSR_PREC_TF32 && A->dtype == BSR_DT_F32 && dy_dtype == BSR_DT_F32) kind = 0;
    if (prec == BSR_PREC_BF16 && A->dtype == BSR_DT_BF16 && dy_dtype == BSR_DT_BF16) kind = 1;
    if (kind < 0 || !bsrp::wgrad_tc_supported(kind, BSR_ALGO_TC_RUNS, A->b, A->K, N) || (kind == 0 && A->b < 32) ||
        A->b < 16 || N % 128 != 0 || A->K / A->b >= 65536)
        return fail(BSR_ERR_UNSUPPORTED, "no per-run tensor-core kernel for prec %d, b=%d, N=%lld with these dtypes", prec,
                    A->b, (long long)N);
    const size_t need = kind == 2 ? bsrp::wgrad_x3_ws_bytes(A->M, A->K, A->b, N) : bsrp::wgrad_tc_ws_bytes(A->M, A->K, A->b, N);
    if (need && (!ws || ws_bytes < need))
        return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, need);
    if (need && !aligned16(ws)) return fail(BSR_ERR_ALIGNMENT, "workspace is not 16-byte aligned");
    return cuda_status(bsrp::launch_wgrad_tc(A->rowptr, A->colidx, A->values, A->nnzb, kind, BSR_ALGO_TC_RUNS, A->M,
                                             A->K, A->b, dY, N, nullptr, 1, ws, static_cast<cudaStream_t>(stream), mc_dW,
                                             0, unicast),
                       "bsr_wgrad_multicast launch");
}

bsr_status_t bsr_wgrad_multicast(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N, float *mc_dW,
                                 int32_t prec, int32_t algo, void *ws, size_t ws_bytes, void *stream) {
    return wgrad_multicast_impl(A, dY, dy_dtype, N, mc_dW, prec, algo, ws, ws_bytes, stream, 0);
}

bsr_status_t bsr_wgrad_multicast_unicast_test(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N,
                                              float *dW_red, int32_t prec, int32_t algo, void *ws, size_t ws_bytes,
                                              void *stream) {
    return wgrad_multicast_impl(A, dY, dy_dtype, N, dW_red, prec, algo, ws, ws_bytes, stream, 1);
}

uint32_t bsr_set_pdl(uint32_t mask) { return bsrp::g_pdl.exchange(mask); }

/* ---- block-sparse affine layer (affine.cu) ---- */
size_t bsr_affine_wgrad_workspace_bytes(int64_t M, int64_t K, int32_t b) {
    if (bsr_num_blocks(M, K, b) < 0 || !supported_b(b)) return 0;
    return bsrp::affine_wgrad_ws_bytes(M, K, b);
}

bsr_status_t bsr_affine_wgrad(const bsr_t *A, const void *dY, int32_t dy_dtype, float *dalpha, int32_t accumulate,
                              void *ws, size_t ws_bytes, void *stream) {
    bsr_status_t st = check_bsr(A);
    if (st != BSR_OK) return st;
    const int esy = elem_size(dy_dtype);
    if (esy == 0) return fail(BSR_ERR_INVALID_ARG, "dy_dtype %d is not BSR_DT_F32 or BSR_DT_BF16", dy_dtype);
    if (!dY || !dalpha) return fail(BSR_ERR_INVALID_ARG, "dY or dalpha is NULL");
    if (accumulate != 0 && accumulate != 1) return fail(BSR_ERR_INVALID_ARG, "accumulate must be 0 or 1");
    if (!aligned16(dY) || !aligned16(dalpha)) return fail(BSR_ERR_ALIGNMENT, "dY or dalpha is not 16-byte aligned");
    if ((A->K * esy) % 16 != 0) return fail(BSR_ERR_ALIGNMENT, "row pitch of dY (K=%lld) is not a multiple of 16 bytes",
                                            (long long)A->K);
    const size_t need = bsrp::affine_wgrad_ws_bytes(A->M, A->K, A->b);
    if (!ws || ws_bytes < need)
        return fail(BSR_ERR_WORKSPACE, "workspace of %zu bytes given, %zu needed", ws ? ws_bytes : (size_t)0, need);
    if (!aligned16(ws)) return fail(BSR_ERR_ALIGNMENT, "workspace is not 16-byte aligned");
    if (overlap(ws, need, dalpha, (size_t)A->K * 4)) return fail(BSR_ERR_INVALID_ARG, "workspace overlaps dalpha");
    return cuda_status(bsrp::launch_affine_wgrad(A->rowptr, A->colidx, A->nnzb ? A->values : nullptr,
                                                 elem_size(A->dtype), A->M, A->K, A->b, dY, esy, dalpha, accumulate,
                                                 ws, static_cast<cudaStream_t>(stream)),
                       "bsr_affine_wgrad launch");
}

const char *bsr_status_string(int32_t status) {
    switch (status) {
        case BSR_OK: return "BSR_OK";
        case BSR_ERR_INVALID_ARG: return "BSR_ERR_INVALID_ARG";
        case BSR_ERR_SHAPE: return "BSR_ERR_SHAPE";
        case BSR_ERR_UNSUPPORTED: return "BSR_ERR_UNSUPPORTED";
        case BSR_ERR_ALIGNMENT: return "BSR_ERR_ALIGNMENT";
        case BSR_ERR_WORKSPACE: return "BSR_ERR_WORKSPACE";
        case BSR_ERR_CUDA: return "BSR_ERR_CUDA";
        default: return "BSR_ERR_UNKNOWN";
    }
}

const char *bsr_last_error(void) { return g_last_error.c_str(); }

uint64_t bsr_kernel_launches(void) { return bsrp::g_launches.load(std::memory_order_relaxed); }

const char *bsr_version(void) { return "bsrprune 0.1.0 sm_100a"; }

}  // extern "C"
