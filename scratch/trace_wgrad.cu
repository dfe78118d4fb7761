// Timeline of the wgrad TC kernel on a C2-like problem (b=32, keep 0.5, f32/tf32).
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
    {
        auto pl = bsrp::tc::plan_for<0, 32>(M, K, N, 148, 6.0);
        printf("plan tf32: kr_blocks %d nkr %d stages %d nbslots %d nsplit %d smem %d chunk %d tmem %u\n", pl.kr_blocks, pl.nkr, pl.stages, pl.nbslots, pl.nsplit, pl.smem, pl.chunk_rows, pl.tmem_cols);
        cudaError_t e = cudaFuncSetAttribute(bsrp::tc::wgrad_tc_kernel<0, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem);
        printf("setattr: %s\n", cudaGetErrorString(e));
        int v; cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0); printf("optin max %d\n", v);
        cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, bsrp::tc::wgrad_tc_kernel<0, 32>); printf("static smem %zu regs %d\n", fa.sharedSizeBytes, fa.numRegs);
    }

    for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t e = bsrp::launch_wgrad_tc(drp, dci, vals, nnzb, kind, M, K, b, dY, N, dW, 0, ws, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("rep %d: %s %.1f us\n", rep, cudaGetErrorString(e), ms * 1e3);
    }
#ifdef NO_TRACE
    return 0;
#endif
    {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        const int64_t n4 = (int64_t)K * N / 4;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            bsrp::tc::splitk_reduce_kernel<<<576, 256>>>((const float4 *)ws, (float4 *)dW, n4, 12, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("reduce alone: %.1f us\n", ms * 1e3);
        }
    }
    static unsigned long long tr[160][256];
#ifndef NO_TRACE
    cudaMemcpyFromSymbol(tr, bsrp::tc::g_trace, sizeof tr);
#endif
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < 144; ++c) t0 = std::min(t0, tr[c][0]);
    {
        unsigned long long emax = 0, smax = 0, plmax = 0; double loopsum = 0;
        int nC = 0;
        for (int c = 0; c < 160; ++c) if (tr[c][0]) {
            emax = std::max(emax, tr[c][204]); smax = std::max(smax, tr[c][0]); plmax = std::max(plmax, tr[c][205]);
            loopsum += (double)(tr[c][203] - tr[c][205]); ++nC;
        }
        printf("CTAs %d: last start %.2f  last plan %.2f  last end %.2f  mean main loop %.2f us\n", nC, (smax - t0) / 1e3, (plmax - t0) / 1e3, (emax - t0) / 1e3, loopsum / nC / 1e3);
    }
    {
        double v[16] = {0}; double rows = 0; int n = 0;
        for (int c = 0; c < 160; ++c) if (tr[c][0]) { for (int k = 0; k < 16; ++k) v[k] += tr[c][210 + k]; rows += tr[c][213]; ++n; }
        printf("A producer per row (cyc): wait %.0f issue %.0f total %.0f (rows/CTA %.1f)\n", v[0] / rows, v[1] / rows, v[2] / rows, rows / n);
        printf("B producer per row (cyc): wait %.0f issue %.0f total %.0f\n", v[4] / rows, v[5] / rows, v[6] / rows);
        printf("mma warp1 per row: wait %.0f issue %.0f total %.0f | warp2 wait %.0f issue %.0f\n", v[8] / rows, v[9] / rows, v[10] / rows, v[11] / rows, v[12] / rows);
    }
    for (int c : {0, 1, 12, 77, 143}) {
        printf("CTA %d: start %.2f  prod %.2f plan %.2f  epi %.2f..%.2f\n", c, (tr[c][0] - t0) / 1e3, (tr[c][1] - t0) / 1e3, (tr[c][205] - t0) / 1e3, (tr[c][203] - t0) / 1e3, (tr[c][204] - t0) / 1e3);
        printf("  TMA issue :"); for (int r = 0; r < 20; r += 1) printf(" %.2f", (tr[c][2 + r] - t0) / 1e3); printf("\n");
        printf("  MMA start :"); for (int r = 0; r < 20; r += 1) printf(" %.2f", (tr[c][102 + r] - t0) / 1e3); printf("\n");
    }
    return 0;
}
