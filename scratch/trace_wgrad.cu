// Per-role cycle accounting of the wgrad TC kernel on a C2-like problem (b=32, keep 0.5).
//   ./trace_wgrad [kind]   kind 0 = tf32 (fp32 data), 1 = bf16
#ifndef NO_TRACE
#define WGRAD_TRACE 1
#endif
#include "../paper_2311_16883_b200/csrc/wgrad_tc.cu"
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
namespace bsrp { void count_launch(uint64_t) {} }
int main(int argc, char **argv) {
    const int M = 25088, K = 384, N = 1536, b = 32;
    const int nbr = M / b, nbc = K / b;
    std::mt19937 rng(1);
    std::vector<int> rowptr(nbr + 1), colidx;
    rowptr[0] = 0;
    for (int I = 0; I < nbr; ++I) {
        for (int J = 0; J < nbc; ++J) if (rng() & 1) colidx.push_back(J);
        rowptr[I + 1] = colidx.size();
    }
    int nnzb = colidx.size();
    float *dY, *vals, *dW, *ws; int *drp, *dci;
    cudaMalloc(&dY, (size_t)M * N * 4); cudaMalloc(&vals, (size_t)nnzb * b * b * 4);
    cudaMalloc(&dW, (size_t)K * N * 4); cudaMalloc(&ws, (size_t)148 * K * N * 4);
    cudaMemset(dY, 0, (size_t)M * N * 4); cudaMemset(vals, 0, (size_t)nnzb * b * b * 4);
    cudaMalloc(&drp, 4 * (nbr + 1)); cudaMalloc(&dci, 4 * nnzb);
    cudaMemcpy(drp, rowptr.data(), 4 * (nbr + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(dci, colidx.data(), 4 * nnzb, cudaMemcpyHostToDevice);
    int kind = argc > 1 ? atoi(argv[1]) : 0;
    auto pl = bsrp::tc::plan_for<0, 32>(M, K, N, 148);
    printf("plan tf32: kr_blocks %d nkr %d nbslots %d na %d sa %d nsplit %d smem %d chunk %d a_col0 %u\n", pl.kr_blocks, pl.nkr,
           pl.nbslots, pl.na, pl.sa, pl.nsplit, pl.smem, pl.chunk_steps, pl.a_col0);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t e = bsrp::launch_wgrad_tc(drp, dci, vals, nnzb, kind, M, K, b, dY, N, dW, 0, ws, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("rep %d: %s %.1f us (kernel + reduce)\n", rep, cudaGetErrorString(cudaGetLastError()), ms * 1e3);
    }
    {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        const int64_t n4 = (int64_t)K * N / 4;
        cudaEventRecord(e0);
        bsrp::tc::splitk_reduce_kernel<<<576, 256>>>((const float4 *)ws, (float4 *)dW, n4, pl.nsplit, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("reduce alone: %.1f us\n", ms * 1e3);
    }
#ifdef NO_TRACE
    return 0;
#else
    static unsigned long long tr[160][256];
    cudaMemcpyFromSymbol(tr, bsrp::tc::g_trace, sizeof tr);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < 144; ++c) if (tr[c][0]) t0 = std::min(t0, tr[c][0]);
    unsigned long long emax = 0, smax = 0, mmax = 0; double loopsum = 0, startsum = 0; int nC = 0;
    double v[16] = {0};
    for (int c = 0; c < 160; ++c) if (tr[c][0]) {
        emax = std::max(emax, tr[c][204]); smax = std::max(smax, tr[c][0]); mmax = std::max(mmax, tr[c][205]);
        loopsum += (double)(tr[c][203] - tr[c][205]); startsum += (double)(tr[c][205] - tr[c][0]); ++nC;
        for (int k = 0; k < 16; ++k) v[k] += (double)tr[c][210 + k];
    }
    const double rows = v[2];
    printf("CTAs %d: last start %.2f  last loop start %.2f  last end %.2f us; mean prologue %.2f, main loop %.2f us\n", nC,
           (smax - t0) / 1e3, (mmax - t0) / 1e3, (emax - t0) / 1e3, startsum / nC / 1e3, loopsum / nC / 1e3);
    printf("steps/CTA %.1f (B producer %.1f); per-row figures below are per STEP\n", rows / nC, v[7] / nC);
    double ai = 0, aw = 0;
    for (int c = 0; c < 160; ++c) if (tr[c][0]) { ai += tr[c][206]; aw += tr[c][207]; }
    printf("A producer: wait sempty %.0f / row;  A mover slab wait %.0f\n", ai / rows, aw / rows);
    printf("A mover  per row (cyc): wait aempty %.0f  store %.0f  slab wait+lds %.0f  total %.0f\n", v[0] / rows, v[3] / rows, v[12] / rows, v[1] / rows);
    double bm = 0, bt = 0;
    for (int c = 0; c < 160; ++c) if (tr[c][0]) { bm += tr[c][208]; bt += tr[c][209]; }
    printf("Bprod    per row (cyc): wait empty %.0f  wait plan %.0f  meta %.0f  tma %.0f  total %.0f\n", v[4] / rows, v[6] / rows, bm / rows, bt / rows, v[5] / rows);
    printf("MMA      per row (cyc): wait full %.0f  wait afull %.0f  issue %.0f (run loop %.0f, %.2f runs/row)  total %.0f\n", v[8] / rows, v[9] / rows, v[11] / rows, v[13] / rows, v[14] / rows, v[10] / rows);
    {
        static long long lat[160][4][64];
        cudaMemcpyFromSymbol(lat, bsrp::tc::g_lat, sizeof lat);
        double bl = 0, al = 0; int nb = 0, na_ = 0;
        for (int c = 0; c < nC; ++c) for (int j = 4; j < 30; ++j) {
            if (lat[c][1][j] > lat[c][0][j] && lat[c][0][j]) { bl += lat[c][1][j] - lat[c][0][j]; ++nb; }
            if (lat[c][3][j] > lat[c][2][j] && lat[c][2][j]) { al += lat[c][3][j] - lat[c][2][j]; ++na_; }
        }
        printf("latency issue->consumer ready (cyc): B %.0f (n=%d)  A %.0f (n=%d)\n", bl / nb, nb, al / na_, na_);
    }
    return 0;
#endif
}
