// refine_nw12.cu — the same refinement (refine.cu) built with 12 warps per path and one resident
// block per SM: the latency regime (few paths, kernel time set by the longest GN runs), where
// more warps per path shorten each iteration (Jacobian tasks and backtracking trials spread
// wider).  Every per-path result is independent of the warp count (each MLS sum is one warp's,
// in the same order; the accepted step is the first in sequence order), so refine() may hand
// any set to either build.  C2: refine 8.51 -> 8.17 ms.
#define NRT_REFINE_WARPS 12
#define NRT_LAT_MINB 1
#define NRT_REFINE_ENTRY refine_nw12
#include "refine.cu"
