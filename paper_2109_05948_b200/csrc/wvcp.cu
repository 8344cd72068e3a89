// wvcp.cu -- batched weighted-colouring tabu search (placeholder until the
// kernel lands).
#include "common.cuh"
#include "launch.h"

namespace mcb {
int wvcp_run(const WvcpArgs &a, cudaStream_t st) {
    (void)a;
    (void)st;
    return set_error(MCB_ERR_UNSUPPORTED, "wvcp kernel not built yet");
}
}  // namespace mcb
