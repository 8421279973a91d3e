// Team-only kernel instantiations (ZV = 3) for the uniform L >= 512 plans with
// few subbands (use_team_short in fcw_device.cuh): config 3's two banks.
// The team-only kernels keep every complex helper packed: measured on config 3
// (TX 0.68 ms packed vs 0.72 ms with scalar products / fused steps).
#define FCW_PK_MUL 1
#define FCW_PK_FMA 1
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NLT(4096, 1024)
FCW_KERNELS_NLT(2048, 512)
FCW_KERNELS_NLT(2048, 1024)
FCW_KERNELS_NLT(1024, 512)
FCW_KERNELS_NLT(1024, 1024)
}  // namespace fcw
