// Kernel instantiations for N = 16 .. 512 (generic path only).
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(16, 0)
FCW_KERNELS_NL(32, 0)
FCW_KERNELS_NL(64, 0)
FCW_KERNELS_NL(128, 0)
FCW_KERNELS_NL(256, 0)
FCW_KERNELS_NL(512, 0)
}  // namespace fcw
