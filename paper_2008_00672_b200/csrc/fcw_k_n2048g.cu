// Kernel instantiations for N = 2048: generic mixed-L kernels.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(2048, 0)
}  // namespace fcw
