// Kernel instantiations for N = 2048 (generic + uniform-L specialisations).
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_FULL(2048)
}  // namespace fcw
