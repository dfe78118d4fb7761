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
    static unsigned long long tr[160][256];
#ifndef NO_TRACE
    cudaMemcpyFromSymbol(tr, bsrp::tc::g_trace, sizeof tr);
#endif
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < 144; ++c) t0 = std::min(t0, tr[c][0]);
    for (int c : {0, 1, 12, 77, 143}) {
        printf("CTA %d: start %.2f  prod %.2f plan %.2f  epi %.2f..%.2f\n", c, (tr[c][0] - t0) / 1e3, (tr[c][1] - t0) / 1e3, (tr[c][205] - t0) / 1e3, (tr[c][203] - t0) / 1e3, (tr[c][204] - t0) / 1e3);
        printf("  TMA issue :"); for (int r = 0; r < 20; r += 1) printf(" %.2f", (tr[c][2 + r] - t0) / 1e3); printf("\n");
        printf("  MMA start :"); for (int r = 0; r < 20; r += 1) printf(" %.2f", (tr[c][102 + r] - t0) / 1e3); printf("\n");
    }
    return 0;
}
