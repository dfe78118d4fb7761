#include "../paper_2311_16883_b200/csrc/wgrad_tc.cu"
#include <cstdio>
namespace bsrp { void count_launch(uint64_t) {} }
int main() {
    const int64_t M = 64 * 64, K = 20 * 64, N = 384; const int nnzb = 128;
    auto pl = bsrp::tc::plan_for<0, 64>(M, K, N, 148);
    double avg = (double)nnzb / (double)(M / 64) * pl.kr_blocks / (double)(K / 64);
    auto p2 = bsrp::tc::plan_for<0, 64>(M, K, N, 148, avg);
    for (auto q : {pl, p2})
        printf("kr_blocks %d nkr %d stages %d nbslots %d nsplit %d smem %d chunk %d tmem %u\n", q.kr_blocks, q.nkr, q.stages, q.nbslots, q.nsplit, q.smem, q.chunk_rows, q.tmem_cols);
    printf("kFixedSmem %d kStageExtra %d\n", bsrp::tc::kFixedSmem, bsrp::tc::kStageExtra);
}
