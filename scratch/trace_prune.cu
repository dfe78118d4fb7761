#define PRUNE_TRACE 1
#include "../paper_2311_16883_b200/csrc/prune.cu"
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
namespace bsrp { void count_launch(uint64_t) {} }
int main(int argc, char **argv) {
    const int M = 25088, K = argc > 1 ? atoi(argv[1]) : 384, b = argc > 2 ? atoi(argv[2]) : 32;
    const int64_t N = (int64_t)(M / b) * (K / b);
    const int64_t k = N / 2;
    std::vector<float> hX((size_t)M * K);
    std::mt19937 rng(1); std::normal_distribution<float> nd;
    for (auto &x : hX) x = nd(rng);
    float *X, *vals; int *rp, *ci; void *ws;
    cudaMalloc(&X, hX.size() * 4); cudaMemcpy(X, hX.data(), hX.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&vals, (size_t)k * b * b * 4); cudaMalloc(&rp, 4 * (M / b + 1)); cudaMalloc(&ci, 4 * k);
    auto w = bsrp::prune_ws_layout(N); cudaMalloc(&ws, w.total); cudaMemset(ws, 0, w.total);
    for (int rep = 0; rep < 4; ++rep) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t e = bsrp::launch_prune(X, M, K, b, 4, k, rp, ci, vals, ws, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("rep %d: %s %.1f us\n", rep, cudaGetErrorString(e), ms * 1e3);
    }
    static unsigned long long tr[2048][8];
    cudaMemcpyFromSymbol(tr, bsrp::g_ptrace, sizeof tr);
    unsigned long long t0 = ~0ull; int nC = 0;
    for (int c = 0; c < 2048; ++c) if (tr[c][0]) { t0 = std::min(t0, tr[c][0]); ++nC; }
    double mx[6] = {0};
    for (int c = 0; c < nC; ++c) for (int i = 0; i < 6; ++i) mx[i] = std::max(mx[i], (tr[c][i] - t0) / 1e3);
    { double a6=0,a7=0; for (int c = 0; c < nC; ++c) { a6 = std::max(a6, (tr[c][6]-t0)/1e3); a7 = std::max(a7, (tr[c][7]-t0)/1e3);} printf("barrier2/keys %.2f cands-refined %.2f\n", a6, a7); }
    printf("CTAs %d; max over CTAs: start %.2f  p1 done %.2f  barrier1 %.2f  select done %.2f  scan done %.2f  pack done %.2f\n", nC, mx[0], mx[1], mx[2], mx[3], mx[4], mx[5]);
    for (int c : {0, nC - 1}) printf("CTA %d: %.2f %.2f %.2f %.2f %.2f %.2f\n", c, (tr[c][0]-t0)/1e3, (tr[c][1]-t0)/1e3, (tr[c][2]-t0)/1e3, (tr[c][3]-t0)/1e3, (tr[c][4]-t0)/1e3, (tr[c][5]-t0)/1e3);
    return 0;
}
