// Kernel instantiations for N = 4096: generic mixed-L kernels.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(4096, 0)
}  // namespace fcw
