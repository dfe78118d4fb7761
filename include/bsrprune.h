/*
 * bsrprune.h -- C ABI of the B200 (sm_100a) hot path of structured activation
 * pruning, arXiv 2311.16883 (Barley & Froening).
 *
 * What the path computes (/root/reference/PAPER.md, cited as P:L<line>):
 *   forward  : every saved linear-layer activation X (M x K, rows =
 *              batch x tokens, row-major) is tiled into b x b blocks; the l2
 *              norm of every block is computed, the k largest-norm blocks are
 *              kept, the others are zeroed, and the result is stored in Block
 *              Sparse Row form (fig:operator
 *              P:L313-321, BSR P:L159-170).
 *   backward : the weight gradient dW = X_bsr^T . dY is a block-sparse x dense
 *              product over the kept blocks only; dX stays dense
 *              and is not part of this library.
 *
 * Conventions shared by every call
 * --------------------------------
 *  * Pointers are CUDA DEVICE pointers unless marked (host).  The caller owns
 *    every buffer; the library never allocates, frees or synchronises.
 *  * Device work is enqueued on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream) and is asynchronous: results are valid once
 *    the stream reaches that point.  Asynchronous device faults surface at the
 *    caller's next synchronisation.  No call performs a device->host copy, so
 *    every call is CUDA-graph capturable.  bsr_wgrad's kernels and
 *    bsr_decompress are launched with programmatic stream serialization (PDL):
 *    they may become resident while the preceding kernel on `stream` drains,
 *    but read and write nothing before it has completed, so stream-order
 *    semantics are unchanged (bsr_set_pdl(0) turns the attribute off).
 *  * Arguments are validated on the host before anything is enqueued; on any
 *    non-BSR_OK return nothing has been written.  bsr_last_error() then holds a
 *    human-readable reason for the calling thread.
 *  * Block flat index: f = I * (K/b) + J for block row I < M/b and block
 *    column J < K/b.
 *  * Element types: BSR_DT_F32 (IEEE binary32) and BSR_DT_BF16 (bfloat16).
 *  * Supported block edges: b in {4, 8, 16, 32, 64}; b must divide M and K.
 *    Base pointers must be 16-byte aligned and K * sizeof(elem) a multiple of
 *    16 bytes (vectorised rows).
 *  * The library is reentrant; the only global state is the thread-local
 *    error string, per-device kernel attributes set once, the launch counter
 *    and the PDL mask of bsr_set_pdl (an atomic; default = measured best).
 */
#ifndef BSRPRUNE_H
#define BSRPRUNE_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BSR_API __attribute__((visibility("default")))
#else
#define BSR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BSR_OK = 0,
    BSR_ERR_INVALID_ARG = 1, /* null pointer, keep outside [0,1] or NaN, k > N, bad enum */
    BSR_ERR_SHAPE = 2,       /* M, K <= 0, b does not divide M or K, size overflow      */
    BSR_ERR_UNSUPPORTED = 3, /* b not in {4,8,16,32,64}, dtype/precision combination    */
    BSR_ERR_ALIGNMENT = 4,   /* pointer or row pitch not 16-byte aligned                */
    BSR_ERR_WORKSPACE = 5,   /* workspace null or smaller than the size query           */
    BSR_ERR_CUDA = 6         /* a CUDA launch failed; bsr_last_error() has the string   */
} bsr_status_t;

typedef enum { BSR_DT_F32 = 0, BSR_DT_BF16 = 1 } bsr_dtype_t;

/* Arithmetic of bsr_wgrad (reading R9 in DESIGN.md):
 *   BSR_PREC_FP32 : FP32 grade, graded at relative Frobenius error <= 1e-5
 *                   against the fp64 oracle; deterministic.  With f32 values
 *                   and f32 dY, b in {32, 64} and N % 128 == 0 it runs on the
 *                   tcgen05 tensor cores as 3xTF32 (each operand split into a
 *                   tf32 head and an fp32 tail, three MMAs per k step, the two
 *                   correction products in their own TMEM accumulator, at most
 *                   1536 rows per accumulator chain, split partials summed with
 *                   round-to-nearest; reading R17); otherwise fp32 FFMA with
 *                   round-to-nearest in a fixed summation order (f32 or bf16
 *                   operands).
 *   BSR_PREC_TF32 : tcgen05 tensor cores, kind::tf32 on fp32 operands, fp32
 *                   accumulation in TMEM.  Graded at <= 5e-3.
 *   BSR_PREC_BF16 : tcgen05 tensor cores, kind::f16 on bf16 operands (X values
 *                   and dY both bf16), fp32 accumulation in TMEM.  <= 5e-3. */
typedef enum { BSR_PREC_FP32 = 0, BSR_PREC_TF32 = 1, BSR_PREC_BF16 = 2 } bsr_prec_t;

/* dW kernel family for bsr_wgrad_algo (bsr_wgrad = BSR_ALGO_AUTO):
 *   AUTO    : the measured best for the shape: tensor cores when
 *             the precision allows; the per-run tcgen05 kernel for K/b < 64, the
 *             CTA-pair span kernel for K/b >= 64 (tf32/bf16) and for tf32 b = 16;
 *             FP32 FFMA when no tensor-core kernel supports the combination.
 *   TC_RUNS : per-run tcgen05 kernel (tf32/bf16 b >= 32 or bf16 b = 16; FP32
 *             grade b in {32, 64}).
 *   TC_SPAN : CTA-pair span kernel (tf32/bf16, b >= 16; not the FP32 grade).
 *   SIMT    : fp32 FFMA (any b, f32 or bf16 operands; BSR_PREC_FP32 only).
 *   TC_DENSE: dense rebuild -- the masked X rebuilt in the workspace, viewed as a
 *             keep-all 32 x 32 BSR and contracted by the per-run kernel (any b; X and
 *             dY both f32 (FP32 grade / tf32) or both bf16; 32 | M, 32 | K,
 *             N % 128 == 0).  AUTO takes it below the native tensor-core block sizes
 *             (FP32 grade b < 32, tf32 / bf16 b < 16): computing the pruned blocks of a
 *             32 x 32 tile as zeros on the tensor cores beats the FFMA kernel there.
 * A combination the chosen family does not implement is BSR_ERR_UNSUPPORTED. */
typedef enum {
    BSR_ALGO_AUTO = 0, BSR_ALGO_TC_RUNS = 1, BSR_ALGO_TC_SPAN = 2, BSR_ALGO_SIMT = 3, BSR_ALGO_TC_DENSE = 4
} bsr_algo_t;

/* A Block Sparse Row matrix.  The struct itself lives in host
 * memory; the three arrays are device memory owned by the caller.
 *   rowptr [M/b + 1]  int32: rowptr[0] = 0, rowptr[I+1] - rowptr[I] = stored
 *                     blocks in block row I ("crow");
 *                     rowptr[M/b] = nnzb.
 *   colidx [nnzb]     int32: block column of each stored block, strictly
 *                     increasing inside a block row ("col").
 *   values [nnzb][b][b] elements of `dtype`, one block after another in
 *                     (block row, colidx) order, row-major inside a block,
 *                     bit-exact copies of X (reading R7). */
typedef struct {
    int64_t M, K;     /* logical dense shape                        */
    int32_t b;        /* square block edge                          */
    int32_t dtype;    /* bsr_dtype_t of values                      */
    int64_t nnzb;     /* stored blocks (== k after bsr_prune)       */
    int32_t *rowptr;
    int32_t *colidx;
    void *values;
} bsr_t;

/* ---- host-only pure helpers (no CUDA calls) ------------------------------ */

/* N = (M/b) * (K/b); -1 if the shape is invalid or b does not divide M, K. */
BSR_API int64_t bsr_num_blocks(int64_t M, int64_t K, int32_t b);

/* Kept blocks for keep ratio keep = 1 - s: k = floor(keep * N + 0.5), clamped
 * to [0, N] ("k is determined by multiplying the total number of
 * blocks N by the sparsity parameter s"; nearest rounding pinned by Table II,
 * P:L180-197).  -1 if keep is NaN or outside [0, 1] or N < 0. */
BSR_API int64_t bsr_keep_count(int64_t nblocks, double keep);

/* Stored bytes of the BSR: k*b*b*sizeof(dtype) + 4*k + 4*(M/b + 1)
 * (BJ closed form with 4-byte values).  0 on invalid input. */
BSR_API size_t bsr_storage_bytes(int64_t M, int32_t b, int64_t k, int32_t dtype);

/* Device workspace (bytes) bsr_prune / bsr_prune_k need for this shape.
 * 0 on invalid input.  The workspace must be zero-filled (cudaMemset) before
 * its first use and must not be written by anything else between bsr_prune
 * calls: every call leaves it zero-filled again (its grid barrier and radix
 * histograms clean themselves), so no per-call clearing is needed.  A
 * workspace that is not zero-filled makes the kernel trap (BSR launch error)
 * instead of hanging. */
BSR_API size_t bsr_prune_workspace_bytes(int64_t M, int64_t K, int32_t b);

/* Device workspace (bytes) bsr_wgrad needs for this shape and precision.  0
 * means none is needed (a NULL workspace is then accepted).  Every path
 * splits the block rows over several CTAs per output tile when the tiles alone
 * do not fill the GPU (tensor cores: up to 148 CTAs; FP32: up to 2 per SM) and
 * writes one partial dW per split there; bsr_wgrad sums them in split order, so
 * the result is deterministic.  Must be 16-byte aligned and must not overlap dW. */
BSR_API size_t bsr_wgrad_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N, int32_t prec);

/* The same query for an explicit kernel family of bsr_wgrad_algo (bsr_algo_t);
 * bsr_wgrad_workspace_bytes = this with BSR_ALGO_AUTO. */
BSR_API size_t bsr_wgrad_algo_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N, int32_t prec, int32_t algo);

/* ---- device work ------------------------------------------------------------ */

/* Prune X (M x K, row-major, `dtype`) to its top-k blocks by l2 norm and pack
 * them into BSR:
 *   1. sumsq[f] = sum of squares of block f in fp32 (fixed summation tree);
 *      ranking by sumsq equals ranking by the l2 norm sqrt(sumsq).
 *   2. keep the k blocks with the largest sumsq, k = bsr_keep_count(N, keep);
 *      among equal sumsq the lower flat index is kept first (BJ tie rule).
 *   3. write out->rowptr, out->colidx, out->values (layout above).
 * `out` (host struct): rowptr/colidx/values must point to caller-allocated
 * device arrays of sizes M/b+1, k and k*b*b elements; on success the call
 * fills out->M, K, b, dtype and sets out->nnzb = k.  values/colidx may be NULL
 * iff k == 0.  X must not overlap any output.  ws must hold
 * bsr_prune_workspace_bytes(M, K, b) bytes. */
BSR_API bsr_status_t bsr_prune(const void *X, int64_t M, int64_t K, int32_t b, double keep,
                       int32_t dtype, bsr_t *out, void *ws, size_t ws_bytes, void *stream);

/* As bsr_prune with an explicit number of kept blocks k in [0, N]. */
BSR_API bsr_status_t bsr_prune_k(const void *X, int64_t M, int64_t K, int32_t b, int64_t k,
                         int32_t dtype, bsr_t *out, void *ws, size_t ws_bytes, void *stream);

/* Stochastic boundary swapping around the top-k threshold -- the paper's
 * future-work variant: "randomly swapping blocks near the top-k threshold,
 * resulting in some blocks above the threshold being pruned anyway, and
 * vice-versa below threshold".  Reading R19 fixes it:
 * rank the blocks by (sumsq desc, flat index asc) -- the bsr_prune order; let
 * w = min(window, k, N - k).  Pair i < w couples rank k-1-i (kept by bsr_prune)
 * with rank k+i (pruned by it) and swaps the two iff u_i < p, where
 *   z = seed + (i + 1) * 0x9E3779B97F4A7C15 (mod 2^64), then the splitmix64
 *   finaliser z ^= z >> 30, z *= 0xBF58476D1CE4E5B9, z ^= z >> 27,
 *   z *= 0x94D049BB133111EB, z ^= z >> 31, and u_i = (z >> 11) * 2^-53.
 * Exactly k blocks stay kept; p = 0 or w = 0 is bsr_prune_k.  The same seed
 * gives the same selection on every call (the caller varies it per step).
 * window: >= 0 with min(window, k, N - k) <= 4096 (else BSR_ERR_INVALID_ARG);
 * p in [0, 1].  Outputs as bsr_prune_k.  ws: bsr_prune_stochastic_workspace_bytes
 * bytes (a bsr_prune workspace of the same shape extended; zero-filled before
 * first use and left zero-filled).  Stream-ordered, no host sync, CUDA-graph
 * capturable: 2 kernels while every CTA can hold all N keys and the 2w boundary
 * blocks in shared memory (N up to ~43K keys), else 9 (global dual radix select,
 * cooperative marking and packing, one-CTA sort of the boundary). */
BSR_API size_t bsr_prune_stochastic_workspace_bytes(int64_t M, int64_t K, int32_t b);
BSR_API bsr_status_t bsr_prune_stochastic(const void *X, int64_t M, int64_t K, int32_t b, int64_t k,
                                  int64_t window, double p, uint64_t seed, int32_t dtype, bsr_t *out,
                                  void *ws, size_t ws_bytes, void *stream);

/* Test hook for step 1 alone: sumsq[N] (fp32, flat order) of every b x b block
 * of X, computed by the same kernel code as bsr_prune. */
BSR_API bsr_status_t bsr_block_sumsq(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype,
                             float *sumsq, void *stream);

/* Structural check of a BSR on the device (the validation hook of SURVEY §5):
 * rowptr[0] == 0, rowptr non-decreasing, rowptr[M/b] == A->nnzb, and within every
 * block row colidx strictly ascending and in [0, K/b).  Writes to
 * *bad_row (caller-owned DEVICE int32) -1 when every row holds, else the lowest
 * offending block row.  Reads rowptr / colidx only; stream-ordered, no host
 * sync (3 tiny kernels); the values are not inspected. */
BSR_API bsr_status_t bsr_validate(const bsr_t *A, int32_t *bad_row, void *stream);

/* Dense M x K matrix (A->dtype) with every stored block at its position and
 * +0.0 elsewhere: X_out == X masked to the kept blocks, bit for bit
 * (SPEC decode; P:L162-168 read backwards).  X_out must hold M*K elements. */
BSR_API bsr_status_t bsr_decompress(const bsr_t *A, void *X_out, void *stream);

/* Weight gradient (BJ):
 *   dW[J*b + c][n] (+)= sum over stored blocks (I, J), sum over r < b of
 *                       values(I,J)[r][c] * dY[I*b + r][n]
 * i.e. dW = X_bsr^T . dY with dW K x N row-major fp32 and dY M x N row-major of
 * `dy_dtype`.  accumulate = 0 overwrites dW, 1 adds to it.  Block rows and
 * blocks that were pruned contribute nothing and are never read.  `prec`
 * selects the arithmetic (see bsr_prec_t): FP32 accepts f32 or bf16 operands;
 * TF32 needs f32 values and f32 dY and b in {16, 32, 64} (b = 16: two blocks
 * share each 128-byte tf32 swizzle row, span kernel only); BF16 needs bf16
 * values and bf16 dY and b in {16, 32, 64}; both tensor-core paths need N a
 * multiple of 128.  Otherwise BSR_ERR_UNSUPPORTED. */
BSR_API bsr_status_t bsr_wgrad(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N, float *dW,
                       int32_t accumulate, int32_t prec, void *ws, size_t ws_bytes, void *stream);

/* bsr_wgrad with an explicit kernel family (bsr_algo_t): same operation, same
 * grading; used by the parity tests to cover every kernel on every shape.  The
 * workspace query bsr_wgrad_workspace_bytes covers every family. */
BSR_API bsr_status_t bsr_wgrad_algo(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N, float *dW,
                                    int32_t accumulate, int32_t prec, int32_t algo, void *ws, size_t ws_bytes,
                                    void *stream);

/* BSR_DW_NK: the same weight gradient stored transposed, dWt = dW^T (N x K
 * row-major fp32 -- PyTorch's nn.Linear.weight.grad layout, so a layer's backward
 * needs no transpose):  dWt[n][J*b + c] (+)= sum ... (as bsr_wgrad_algo).
 * Same prec / algo / operand rules as bsr_wgrad_algo.  The FP32-grade per-run
 * kernel (b in {32, 64}, N % 128 == 0) writes it natively: its chain-capped
 * split-K reduce sums the partials in split order (bit-identical to bsr_wgrad's
 * dW, transposed) and stores through a 32 x 32 shared-memory transpose; every
 * other path computes dW into the workspace's tail and transposes it in one
 * extra pass (accumulate then adds old + dW, one rounding).  ws: at least
 * bsr_wgrad_nk_workspace_bytes(M, K, b, N, prec, algo) bytes, 16-byte aligned,
 * not overlapping dWt. */
BSR_API size_t bsr_wgrad_nk_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N, int32_t prec, int32_t algo);
BSR_API bsr_status_t bsr_wgrad_nk(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N, float *dWt,
                                  int32_t accumulate, int32_t prec, int32_t algo, void *ws, size_t ws_bytes,
                                  void *stream);

/* dW with the data-parallel sum fused into it (a7 over NVLink
 * SHARP): mc_dW is the MULTIMEM (NVLS multicast) address of a K x N fp32 buffer
 * bound on every rank (e.g. torch symmetric memory's multicast_ptr); this rank's
 * dW = X_bsr^T . dY is ADDED into it with multimem.red.add.f32 -- from the dW
 * epilogue when the rows are not split, else from the split-K reduce -- so the
 * NVSwitch sums the ranks' contributions and every rank's copy holds the total.
 * The caller zeroes the buffer on every rank before and synchronises the ranks
 * after (the adds are asynchronous).  Per-run tensor-core kernel only (prec
 * TF32, BF16 or the FP32 grade, algo AUTO or TC_RUNS, as bsr_wgrad_algo);
 * otherwise BSR_ERR_UNSUPPORTED.  With one rank and a zeroed buffer the result
 * is bit-identical to bsr_wgrad (0 + x = x).  The ranks' sum is not
 * order-deterministic. */
BSR_API bsr_status_t bsr_wgrad_multicast(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N, float *mc_dW,
                                         int32_t prec, int32_t algo, void *ws, size_t ws_bytes, void *stream);

/* Test hook for the fused reduction of bsr_wgrad_multicast on hardware without a
 * multicast object (a single-GPU slice): the same kernels, the same addresses and
 * the same per-element reduction, with red.global.add (device-scope atomics) into
 * the plain device buffer dW_red instead of multimem.red into a multicast address.
 * dW_red (+)= dW; the order of the adds across tiles is not fixed. */
BSR_API bsr_status_t bsr_wgrad_multicast_unicast_test(const bsr_t *A, const void *dY, int32_t dy_dtype, int64_t N,
                                              float *dW_red, int32_t prec, int32_t algo, void *ws,
                                              size_t ws_bytes, void *stream);

/* Programmatic-dependent-launch mask of this process (bit meanings in
 * csrc/launch.h; 0 = plain stream order).  Returns the previous mask.  Results
 * are bit-identical for every mask (tests/test_pdl_gpu.py); only the overlap
 * of a kernel's prologue with its predecessor's tail changes. */
BSR_API uint32_t bsr_set_pdl(uint32_t mask);

/* ---- cross-rank global top-k ----------------------------
 * Under data parallelism each rank holds a shard of X's rows.  bsr_prune keeps
 * keep*N_rank blocks per rank (per-rank scope, R2).  These three calls
 * let the caller keep the k = bsr_keep_count(N_total, keep) largest blocks of the
 * CONCATENATED X instead (rank order = flat order; ties: lower rank, then lower
 * flat index first), so multi-GPU selection equals the single-GPU one
 * (P:L413-418 over the whole batch).  The library does not communicate: the
 * caller all-reduces the digit histograms and all-gathers the counts between
 * the calls (paper_2311_16883_b200.prune_global).  Keys are the fp32 bit
 * patterns of the block sums of squares (bit 31 cleared), exactly as bsr_prune.
 * `ws` is the bsr_prune workspace (same size, zero-filled on first use).
 *
 * bsr_select_hist: level 0 computes every block's sum of squares into ws and
 *   hist[4096] = histogram of key bits 30..19; level 1: hist[1024] of bits 18..9
 *   of the keys whose bits 30..19 == prefix; level 2: hist[512] of bits 8..0 of
 *   the keys whose bits 30..9 == prefix.  hist: device uint32, zeroed by the call.
 * bsr_select_counts: counts[0] = #blocks with (key >> shift) > threshold,
 *   counts[1] = #blocks with (key >> shift) == threshold (device uint64[2]).
 * bsr_prune_threshold: pack the blocks with (key >> shift) > threshold plus the
 *   first tie_take blocks with (key >> shift) == threshold in flat order into
 *   `out` (layout as bsr_prune); k must equal counts[0] + tie_take of the same
 *   (threshold, shift), out sized for k.  Needs the level-0 sums in ws. */
BSR_API bsr_status_t bsr_select_hist(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype, int32_t level,
                                     uint32_t prefix, uint32_t *hist, void *ws, size_t ws_bytes, void *stream);
BSR_API bsr_status_t bsr_select_counts(int64_t M, int64_t K, int32_t b, uint32_t threshold, int32_t shift,
                                       uint64_t *counts, void *ws, size_t ws_bytes, void *stream);
BSR_API bsr_status_t bsr_prune_threshold(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype,
                                         uint32_t threshold, int32_t shift, int64_t tie_take, int64_t k, bsr_t *out,
                                         void *ws, size_t ws_bytes, void *stream);


/* The same protocol with its state in DEVICE memory, so that no step needs a
 * device->host copy: the caller's collectives (NCCL on device buffers) run
 * between stream-ordered calls, and only the final kept count of this rank is
 * read back (to size the result).  The collective sequence is fixed: three
 * histogram all-reduces (a resolved level contributes zeros) and one all-gather.
 *   bsr_gselect_state_bytes   bytes of the opaque state (device, caller-owned).
 *   bsr_gselect_init          state <- k_total (the kept count of the whole batch).
 *   bsr_gselect_hist          level 0..2: this rank's digit histogram of the keys
 *                             matching the state's prefix (level 0 also computes the
 *                             block sums into ws, as bsr_select_hist); hist uint32
 *                             [4096 / 1024 / 512], zeroed by the call.
 *   bsr_gselect_update        after the all-reduce of hist: the boundary bin of the
 *                             summed histogram joins the prefix (1-CTA kernel).
 *   bsr_gselect_counts        this rank's (#keys > T, #keys == T): uint64[2].
 *   bsr_gselect_take          after the all-gather of every rank's counts
 *                             (uint64 [world][2], rank order): this rank's tie quota
 *                             and kept count k_rank (state word 7, uint64).
 *   bsr_prune_gselect         pack with the state's threshold into `out`, whose
 *                             arrays hold `capacity` >= k_rank blocks (e.g.
 *                             min(N_rank, k_total)); rowptr[M/b] = k_rank; out->nnzb
 *                             is set to capacity (the host learns k_rank from state
 *                             word 7).  With one rank: bit-identical to bsr_prune_k. */
BSR_API size_t bsr_gselect_state_bytes(void);
BSR_API bsr_status_t bsr_gselect_init(int64_t k_total, uint64_t *state, void *stream);
BSR_API bsr_status_t bsr_gselect_hist(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype, int32_t level,
                                      const uint64_t *state, uint32_t *hist, void *ws, size_t ws_bytes, void *stream);
BSR_API bsr_status_t bsr_gselect_update(const uint32_t *hist_total, int32_t level, uint64_t *state, void *stream);
BSR_API bsr_status_t bsr_gselect_counts(int64_t M, int64_t K, int32_t b, const uint64_t *state, uint64_t *counts,
                                        void *ws, size_t ws_bytes, void *stream);
BSR_API bsr_status_t bsr_gselect_take(const uint64_t *all_counts, int32_t world, int32_t rank, uint64_t *state,
                                      void *stream);
BSR_API bsr_status_t bsr_prune_gselect(const void *X, int64_t M, int64_t K, int32_t b, int32_t dtype,
                                       const uint64_t *state, int64_t capacity, bsr_t *out, void *ws, size_t ws_bytes,
                                       void *stream);


/* ---- the paper-faithful variant: 1 x b row segments, per-sample scope --------
 * (Table II geometry P:L180-197; "Blocks are only compared
 * locally, not among other activations in the mini-batch".)
 * X is M x K with M = samples x sample_rows.  Blocks are 1 x b row segments;
 * every sample keeps exactly ks = bsr_rows_keep_per_sample(sample_rows, K, b,
 * keep) = nearest(keep * sample_rows * K / b) segments with the largest fp32 sum
 * of squares, ties to the lower flat index within the sample.  Output: one BSR
 * with br = 1, bc = b: rowptr[M + 1], colidx[k] (segment column J, ascending per
 * row), values[k][b] (raw bits), k = (M / sample_rows) * ks.  Requires b | K,
 * sample_rows | M and K * sizeof(dtype) % 16 == 0.  The workspace holds the
 * segment sums (bsr_prune_rows_workspace_bytes).
 * bsr_decompress_rows: the dense M x K matrix with zeros outside kept segments.
 * bsr_wgrad_rows: dW (K x N fp32) = X_bsr^T dY over the kept segments, fp32
 *   FFMA in a fixed order (deterministic); workspace for split partials
 *   (bsr_wgrad_rows_workspace_bytes, may be 0). */
BSR_API int64_t bsr_rows_keep_per_sample(int64_t sample_rows, int64_t K, int32_t b, double keep);
BSR_API size_t bsr_prune_rows_workspace_bytes(int64_t M, int64_t K, int32_t b);
BSR_API bsr_status_t bsr_prune_rows(const void *X, int64_t M, int64_t K, int32_t b, int64_t sample_rows, double keep,
                                    int32_t dtype, int32_t *rowptr, int32_t *colidx, void *values, void *ws,
                                    size_t ws_bytes, void *stream);
BSR_API bsr_status_t bsr_decompress_rows(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t M,
                                         int64_t K, int32_t b, int32_t dtype, void *X_out, void *stream);
BSR_API size_t bsr_wgrad_rows_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N);
/* The same dW on the tensor cores: with per-sample 1 x b segments an 8-row tensor-core
 * K step almost never meets a fully pruned b-wide tile (0.5^8 at keep 0.5), so the
 * kept rows are rebuilt densely (zeros elsewhere), viewed as a keep-all 32 x 32 BSR
 * and contracted by the per-run tcgen05 kernel: FP32 grade (3xTF32, rel-F <= 1e-5)
 * for f32 X and dY, bf16 for bf16 X and dY.  Needs 32 | M, 32 | K, N % 128 == 0,
 * dY in X's dtype (else BSR_ERR_UNSUPPORTED); workspace from the query (0 if the
 * shape is not supported). */
BSR_API size_t bsr_wgrad_rows_tc_workspace_bytes(int64_t M, int64_t K, int32_t b, int64_t N, int32_t x_dtype);
BSR_API bsr_status_t bsr_wgrad_rows_tc(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnz,
                                       int64_t M, int64_t K, int32_t b, int32_t x_dtype, const void *dY,
                                       int32_t dy_dtype, int64_t N, float *dW, int32_t accumulate, void *ws,
                                       size_t ws_bytes, void *stream);
BSR_API bsr_status_t bsr_wgrad_rows(const int32_t *rowptr, const int32_t *colidx, const void *values, int64_t nnz,
                                    int64_t M, int64_t K, int32_t b, int32_t x_dtype, const void *dY,
                                    int32_t dy_dtype, int64_t N, float *dW, int32_t accumulate, void *ws,
                                    size_t ws_bytes, void *stream);


/* ---- producer fusion (the norm pass in the producer of X) -----
 * bsr_act_block_sumsq: X_out = act(Z) (act 0 = identity, 1 = GELU tanh form,
 *   evaluated in fp32, rounded to `dtype`), written once, and the fp32 block sums
 *   of squares of the WRITTEN X (same order and tree as bsr_prune's, so bit-
 *   identical) into the prune workspace.  Z == X_out (in place) is allowed.
 * bsr_prune_presummed: bsr_prune_k that takes the block sums from the workspace
 *   (left there by bsr_act_block_sumsq on the same X, b and workspace) instead of
 *   reading X for them: X is read only for the kept blocks.  Same output. */
BSR_API bsr_status_t bsr_act_block_sumsq(const void *Z, void *X_out, int64_t M, int64_t K, int32_t b, int32_t dtype,
                                         int32_t act, void *ws, size_t ws_bytes, void *stream);
BSR_API bsr_status_t bsr_prune_presummed(const void *X, int64_t M, int64_t K, int32_t b, int64_t k, int32_t dtype,
                                         bsr_t *out, void *ws, size_t ws_bytes, void *stream);


/* ---- block-sparse affine scaling layer -------------------
 * "A block-sparse version of the affine scaling layer found in ResMLP is now also
 * available".  ResMLP's Aff(x) = alpha * x + beta scales each of the
 * K channels of the M x K residual stream; with x saved as the BSR
 * A of its top-k b x b blocks (bsr_prune), the scale gradient is
 *   dalpha[J*b + c] (+)= sum over stored blocks (I, J), sum over r < b of
 *                        values(I,J)[r][c] * dY[I*b + r][J*b + c]
 * dY is M x K row-major (dy_dtype), dalpha K fp32.  (dbeta = column sums of dY
 * and dX = alpha * dY need no activation.)  fp32 FMAs with round-to-nearest in a
 * fixed order, split partials summed in split order: deterministic, graded at
 * rel-F <= 1e-5.  Pruned blocks are never read.  ws: bsr_affine_wgrad_workspace_bytes. */
BSR_API size_t bsr_affine_wgrad_workspace_bytes(int64_t M, int64_t K, int32_t b);
BSR_API bsr_status_t bsr_affine_wgrad(const bsr_t *A, const void *dY, int32_t dy_dtype, float *dalpha,
                                      int32_t accumulate, void *ws, size_t ws_bytes, void *stream);


/* Static description of a status code. */
BSR_API const char *bsr_status_string(int32_t status);

/* Detail of the calling thread's last failing call ("" if none). */
BSR_API const char *bsr_last_error(void);

/* Number of CUDA kernels this library has launched in this process so far
 * (all calls, all threads; memsets are not counted).  Diagnostic: lets a
 * caller prove how many of the library's own kernels ran in a region.  Kernel
 * launches replayed from a CUDA graph captured around a call are not counted
 * again. */
BSR_API uint64_t bsr_kernel_launches(void);

/* Library version string, e.g. "bsrprune 0.1.0 sm_100a". */
BSR_API const char *bsr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BSRPRUNE_H */
