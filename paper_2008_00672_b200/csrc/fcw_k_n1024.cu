// Kernel instantiations for N = 1024 (generic + uniform-L specialisations).
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_FULL(1024)
}  // namespace fcw
