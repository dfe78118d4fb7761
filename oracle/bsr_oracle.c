/*
 * bsr_oracle.c -- CPU oracle for the structured-activation-pruning hot path of
 * arXiv 2311.16883 (Barley & Froening, "Compressing the Backward Pass of
 * Large-Scale Neural Architectures by Structured Activation Pruning").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2311_16883_b200/) never links, imports or calls it,
 * and shares no code, header, table or constant with it.
 *
 * Plain, slow, obviously correct: fp64 arithmetic, single thread, no blocking,
 * no fusion, loops in the order the definitions are written.  Each function
 * cites the passage of /root/reference/PAPER.md ("P:L<line>") or the
 * BASELINE.json north star ("BJ") it follows.  Readings of ambiguous points are
 * listed in DESIGN.md section 3 ("R1".."R14").
 *
 * Blocks are generalised to br x bc (rows x cols).  The north-star path uses
 * square b x b blocks (br = bc = b, BJ); Table II of the paper is
 * stated for 1 x b row segments (br = 1, bc = b), which the same code covers.
 *
 * Element types: dtype 0 = IEEE fp32, dtype 1 = bfloat16 (stored as raw
 * uint16 bit patterns; converted to float exactly by a 16-bit left shift).
 *
 * Every function returns 0 on success and a negative code on a violated
 * precondition (-1 shape, -2 argument).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- element access -------------------------------------------------- */

static double orc_elem(const void *base, int dtype, int64_t i)
{
    if (dtype == 0) {
        return (double)((const float *)base)[i];
    } else {
        uint32_t bits = ((uint32_t)((const uint16_t *)base)[i]) << 16;
        float f;
        memcpy(&f, &bits, sizeof f);
        return (double)f;
    }
}

static int64_t orc_elem_size(int dtype) { return dtype == 0 ? 4 : 2; }

/* ---- O1: shape / block bookkeeping ----------------------------------- */

/* Number of blocks N of an M x K matrix tiled into br x bc blocks.
 * P:L415-417 ("the total number of blocks N").  Returns -1 if br or bc does
 * not divide the matrix (R10: such layers are not prunable, no padding). */
int64_t orc_num_blocks(int64_t M, int64_t K, int64_t br, int64_t bc)
{
    if (M <= 0 || K <= 0 || br <= 0 || bc <= 0) return -1;
    if (M % br != 0 || K % bc != 0) return -1;
    return (M / br) * (K / bc);
}

/* Number of KEPT blocks k for keep ratio keep = 1 - s.
 * "zero out the k smallest blocks, where k is determined by
 * multiplying the total number of blocks N by the sparsity parameter s".
 * Reading R3: the kept count is the nearest integer to keep*N, i.e.
 * floor(keep*N + 0.5), clamped to [0, N].  Table II pins the
 * nearest-integer rounding (tests/golden/table2_bsr_overhead.txt). */
int64_t orc_keep_count(int64_t N, double keep)
{
    if (N < 0 || !(keep >= 0.0 && keep <= 1.0)) return -1;
    double x = floor(keep * (double)N + 0.5);
    int64_t k = (int64_t)x;
    if (k < 0) k = 0;
    if (k > N) k = N;
    return k;
}

/* Stored bytes of a BSR matrix with k stored blocks:
 *   values  k * br * bc * value_bytes
 *   col     k * index_bytes                       ("col")
 *   crow    (M/br + 1) * index_bytes              ("crow")
 * BJ closed form for the north star: k*b^2*4 + k*4 + (M/b+1)*4. */
int64_t orc_storage_bytes(int64_t M, int64_t br, int64_t bc, int64_t k,
                          int64_t value_bytes, int64_t index_bytes)
{
    if (M <= 0 || br <= 0 || bc <= 0 || k < 0 || M % br != 0) return -1;
    return k * br * bc * value_bytes + k * index_bytes + (M / br + 1) * index_bytes;
}

/* ---- O2: block l2 norms ---------------------------------------------- */

/* sumsq[f] = sum over the block's elements of x^2, in fp64, for the block in
 * block-row I and block-column J, flat index f = I*(K/bc) + J; accumulated
 * row-major (r outer, c inner).  The block's l2 (Frobenius) norm is
 * sqrt(sumsq[f]).  P:L101-102 ("The l2-norm is used to compare blocks of
 * activations"), P:L413-418 ("their vector or matrix norms are compared"). */
int orc_block_sumsq(const void *X, int dtype, int64_t M, int64_t K,
                    int64_t br, int64_t bc, double *sumsq)
{
    if (orc_num_blocks(M, K, br, bc) < 0) return -1;
    int64_t nbr = M / br, nbc = K / bc;
    for (int64_t I = 0; I < nbr; ++I)
        for (int64_t J = 0; J < nbc; ++J) {
            double s = 0.0;
            for (int64_t r = 0; r < br; ++r)
                for (int64_t c = 0; c < bc; ++c) {
                    double x = orc_elem(X, dtype, (I * br + r) * K + J * bc + c);
                    s += x * x;
                }
            sumsq[I * nbc + J] = s;
        }
    return 0;
}

/* ---- O4: top-k selection --------------------------------------------- */

static const double *g_norm; /* comparator context (single-threaded oracle) */

/* Order: larger norm first; among equal norms the lower flat index first
 * (BJ: "ties -> lower flat block index"; reading R4). */
static int orc_cmp(const void *a, const void *b)
{
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    double ni = g_norm[i], nj = g_norm[j];
    if (ni > nj) return -1;
    if (ni < nj) return 1;
    return (i < j) ? -1 : (i > j);
}

/* mask[f] = 1 for the k blocks that are KEPT, 0 for the N-k pruned ones.
 * the blocks are ranked by norm and "the k smallest" (here: all
 * but the k largest) are zeroed.  Ranking is by norm = sqrt(sumsq) as the
 * paper states, via a full sort (std-library qsort) of the block indices. */
int orc_select_topk(const double *sumsq, int64_t N, int64_t k, uint8_t *mask)
{
    if (N < 0 || k < 0 || k > N) return -2;
    double *norm = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    int64_t *idx = (int64_t *)malloc((size_t)(N > 0 ? N : 1) * sizeof(int64_t));
    if (!norm || !idx) { free(norm); free(idx); return -2; }
    for (int64_t f = 0; f < N; ++f) { norm[f] = sqrt(sumsq[f]); idx[f] = f; }
    g_norm = norm;
    qsort(idx, (size_t)N, sizeof(int64_t), orc_cmp);
    for (int64_t f = 0; f < N; ++f) mask[f] = 0;
    for (int64_t t = 0; t < k; ++t) mask[idx[t]] = 1;
    free(norm);
    free(idx);
    return 0;
}

/* ---- O5: BSR construction -------------------------------------------- */

/* Convert the masked matrix to Block Sparse Row form.  P:L159-170:
 *   crow[0] = 0, crow[I+1] = crow[I] + (number of stored blocks in block row I)
 *   "The last element in crow is then the total number of non-zero blocks";
 *   col lists each stored block's block-column, in order along the row;
 *   values holds the stored blocks one after another, row-major inside a block
 *   (reading R7), copied byte for byte from X.
 * Every kept block is stored, including an all-zero one (reading R6), so
 * rowptr[M/br] == number of set mask bits. */
int orc_build_bsr(const void *X, int dtype, int64_t M, int64_t K,
                  int64_t br, int64_t bc, const uint8_t *mask,
                  int32_t *rowptr, int32_t *colidx, void *values)
{
    if (orc_num_blocks(M, K, br, bc) < 0) return -1;
    int64_t nbr = M / br, nbc = K / bc, es = orc_elem_size(dtype);
    const uint8_t *src = (const uint8_t *)X;
    uint8_t *dst = (uint8_t *)values;
    int64_t p = 0;
    rowptr[0] = 0;
    for (int64_t I = 0; I < nbr; ++I) {
        for (int64_t J = 0; J < nbc; ++J) {
            if (!mask[I * nbc + J]) continue;
            colidx[p] = (int32_t)J;
            for (int64_t r = 0; r < br; ++r)
                memcpy(dst + (p * br * bc + r * bc) * es,
                       src + ((I * br + r) * K + J * bc) * es, (size_t)(bc * es));
            ++p;
        }
        rowptr[I + 1] = (int32_t)p;
    }
    return 0;
}

/* The whole forward-side step: norms -> top-k -> BSR (P:L305-311,
 * fig:operator P:L313-321).  k is the explicit number of kept blocks. */
int orc_prune(const void *X, int dtype, int64_t M, int64_t K, int64_t b, int64_t k,
              int32_t *rowptr, int32_t *colidx, void *values, double *sumsq_out,
              uint8_t *mask_out)
{
    int64_t N = orc_num_blocks(M, K, b, b);
    if (N < 0) return -1;
    if (k < 0 || k > N) return -2;
    int rc = orc_block_sumsq(X, dtype, M, K, b, b, sumsq_out);
    if (rc) return rc;
    rc = orc_select_topk(sumsq_out, N, k, mask_out);
    if (rc) return rc;
    return orc_build_bsr(X, dtype, M, K, b, b, mask_out, rowptr, colidx, values);
}

/* ---- O6: decompress -------------------------------------------------- */

/* Dense M x K matrix from BSR: zeros everywhere, each stored block copied to
 * block position (I, col[p]) (P:L162-168 read in reverse; SPEC decode). */
int orc_decompress(const int32_t *rowptr, const int32_t *colidx, const void *values,
                   int dtype, int64_t M, int64_t K, int64_t br, int64_t bc, void *Xout)
{
    if (orc_num_blocks(M, K, br, bc) < 0) return -1;
    int64_t nbr = M / br, es = orc_elem_size(dtype);
    memset(Xout, 0, (size_t)(M * K * es));
    const uint8_t *src = (const uint8_t *)values;
    uint8_t *dst = (uint8_t *)Xout;
    for (int64_t I = 0; I < nbr; ++I)
        for (int64_t p = rowptr[I]; p < rowptr[I + 1]; ++p) {
            int64_t J = colidx[p];
            for (int64_t r = 0; r < br; ++r)
                memcpy(dst + ((I * br + r) * K + J * bc) * es,
                       src + (p * br * bc + r * bc) * es, (size_t)(bc * es));
        }
    return 0;
}

/* ---- O7: block-sparse weight gradient -------------------------------- */

/* dW = X_bsr^T . dY, dW is K x Nout (row-major, fp64), dY is M x Nout.
 * P:L323-326 (weight gradient from the BSR activation via BSpMM), BJ
 * ("dW = X_bsr^T . dY ... over the kept blocks only"), reading R8.
 *   dW[J*bc + c][n] = sum over stored blocks p=(I,J), sum over r <
 *                     values[p][r][c] * dY[I*br + r][n]
 * Plain quadruple loop in stored-block order, fp64 accumulation. */
int orc_wgrad(const int32_t *rowptr, const int32_t *colidx, const void *values, int dtype,
              int64_t M, int64_t K, int64_t br, int64_t bc,
              const void *dY, int dy_dtype, int64_t Nout, double *dW)
{
    if (orc_num_blocks(M, K, br, bc) < 0 || Nout <= 0) return -1;
    int64_t nbr = M / br;
    for (int64_t i = 0; i < K * Nout; ++i) dW[i] = 0.0;
    for (int64_t I = 0; I < nbr; ++I)
        for (int64_t p = rowptr[I]; p < rowptr[I + 1]; ++p) {
            int64_t J = colidx[p];
            for (int64_t r = 0; r < br; ++r)
                for (int64_t c = 0; c < bc; ++c) {
                    double v = orc_elem(values, dtype, p * br * bc + r * bc + c);
                    double *out = dW + (J * bc + c) * Nout;
                    int64_t yrow = (I * br + r) * Nout;
                    for (int64_t n = 0; n < Nout; ++n)
                        out[n] += v * orc_elem(dY, dy_dtype, yrow + n);
                }
        }
    return 0;
}

/* Selected entries of dW, each computed on its own from the same definition
 * (used for parity at full size, where the whole product is too slow):
 *   out[t] = dW[rows[t]][cols[t]]. */
int orc_wgrad_entries(const int32_t *rowptr, const int32_t *colidx, const void *values,
                      int dtype, int64_t M, int64_t K, int64_t br, int64_t bc,
                      const void *dY, int dy_dtype, int64_t Nout,
                      const int64_t *rows, const int64_t *cols, int64_t count, double *out)
{
    if (orc_num_blocks(M, K, br, bc) < 0 || Nout <= 0) return -1;
    int64_t nbr = M / br;
    for (int64_t t = 0; t < count; ++t) {
        int64_t row = rows[t], n = cols[t];
        if (row < 0 || row >= K || n < 0 || n >= Nout) return -2;
        int64_t J = row / bc, c = row % bc;
        double s = 0.0;
        for (int64_t I = 0; I < nbr; ++I)
            for (int64_t p = rowptr[I]; p < rowptr[I + 1]; ++p) {
                if (colidx[p] != J) continue;
                for (int64_t r = 0; r < br; ++r)
                    s += orc_elem(values, dtype, p * br * bc + r * bc + c) *
                         orc_elem(dY, dy_dtype, (I * br + r) * Nout + n);
            }
        out[t] = s;
    }
    return 0;
}

/* ---- block-sparse affine scaling layer ----------------------
 * "A block-sparse version of the affine scaling layer found in ResMLP":
 * Aff(x) = alpha * x + beta per channel; its scale gradient from the BSR of x,
 *   dalpha[J*bc + c] = sum over stored blocks p=(I,J), sum over r < br of
 *                      values[p][r][c] * dY[(I*br + r)][J*bc + c]
 * dY is M x K (the shape of x), dalpha K entries (fp64). */
int orc_affine_wgrad(const int32_t *rowptr, const int32_t *colidx, const void *values, int dtype,
                     int64_t M, int64_t K, int64_t br, int64_t bc,
                     const void *dY, int dy_dtype, double *dalpha)
{
    if (orc_num_blocks(M, K, br, bc) < 0) return -1;
    int64_t nbr = M / br;
    for (int64_t i = 0; i < K; ++i) dalpha[i] = 0.0;
    for (int64_t I = 0; I < nbr; ++I)
        for (int64_t p = rowptr[I]; p < rowptr[I + 1]; ++p) {
            int64_t J = colidx[p];
            for (int64_t r = 0; r < br; ++r)
                for (int64_t c = 0; c < bc; ++c)
                    dalpha[J * bc + c] += orc_elem(values, dtype, p * br * bc + r * bc + c) *
                                          orc_elem(dY, dy_dtype, (I * br + r) * K + J * bc + c);
        }
    return 0;
}

/* ---- stochastic boundary swapping ---------------------------
 * "One could imagine randomly swapping blocks near the top-k threshold, resulting
 * in some blocks above the threshold being pruned anyway, and vice-versa below
 * threshold" (future work in the paper).  Reading R19:
 * rank the blocks by (norm desc, flat index asc) (O4); the deterministic top-k
 * keeps ranks [0, k).  With w' = min(window, k, N - k), pair i < w' couples rank
 * k-1-i (kept) with rank k+i (pruned); the pair swaps -- the first pruned, the
 * second kept -- iff u_i < p, where u_i is the counter-based uniform
 *   z = seed + (i + 1) * 0x9E3779B97F4A7C15 (mod 2^64), splitmix64 finaliser,
 *   u_i = (z >> 11) * 2^-53.
 * Exactly k blocks stay kept.  mask[f] = 1 for kept blocks. */
static uint64_t orc_splitmix(uint64_t seed, uint64_t i)
{
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double orc_swap_uniform(uint64_t seed, int64_t i)
{
    return (double)(orc_splitmix(seed, (uint64_t)i) >> 11) * (1.0 / 9007199254740992.0);
}

int orc_select_topk_stochastic(const double *sumsq, int64_t N, int64_t k, int64_t window, double p,
                               uint64_t seed, uint8_t *mask)
{
    if (N < 0 || k < 0 || k > N || window < 0 || !(p >= 0.0 && p <= 1.0)) return -2;
    double *norm = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    int64_t *order = (int64_t *)malloc((size_t)(N > 0 ? N : 1) * sizeof(int64_t));
    if (!norm || !order) { free(norm); free(order); return -2; }
    for (int64_t i = 0; i < N; ++i) { norm[i] = sqrt(sumsq[i]); order[i] = i; }
    g_norm = norm;  /* the same ranking as orc_select_topk (O4) */
    qsort(order, (size_t)N, sizeof(int64_t), orc_cmp);
    for (int64_t i = 0; i < N; ++i) mask[i] = 0;
    for (int64_t r = 0; r < k; ++r) mask[order[r]] = 1;
    int64_t w = window;
    if (w > k) w = k;
    if (w > N - k) w = N - k;
    for (int64_t i = 0; i < w; ++i)
        if (orc_swap_uniform(seed, i) < p) {
            mask[order[k - 1 - i]] = 0;
            mask[order[k + i]] = 1;
        }
    free(norm);
    free(order);
    return 0;
}
