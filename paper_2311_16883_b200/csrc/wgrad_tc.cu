// wgrad_tc.cu -- tcgen05/TMEM tensor-core path of the BSR weight gradient.
// (placeholder until the tcgen05 kernel lands)
#include "launch.h"

namespace bsrp {

size_t wgrad_tc_ws_bytes(int64_t, int64_t, int, int64_t) { return 0; }

cudaError_t launch_wgrad_tc(const int32_t *, const int32_t *, const void *, int, int64_t, int64_t, int,
                            const void *, int64_t, float *, int, void *, cudaStream_t) {
    return cudaErrorNotSupported;
}

}  // namespace bsrp
