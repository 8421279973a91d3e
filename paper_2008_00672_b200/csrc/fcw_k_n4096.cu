// Kernel instantiations for N = 4096 (generic + uniform-L specialisations).
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_FULL(4096)
}  // namespace fcw
