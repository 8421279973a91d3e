// Kernel instantiations for N = 16 .. 512 (generic path only).
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_GENERIC(16)
FCW_KERNELS_GENERIC(32)
FCW_KERNELS_GENERIC(64)
FCW_KERNELS_GENERIC(128)
FCW_KERNELS_GENERIC(256)
FCW_KERNELS_GENERIC(512)
}  // namespace fcw
