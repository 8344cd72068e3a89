// tabucol_warp_stats.cu -- the instrumented instantiations of the warp
// TabuCol kernel (MCB_FLAG_WSTATS: event counters and per-phase clock64
// cycles, read by mcb_debug_warp_stats).  A separate translation unit so that
// the production kernels carry no instrumentation and both build in parallel.
#define TW_STATS_TU 1
#include "tabucol_warp.cu"
