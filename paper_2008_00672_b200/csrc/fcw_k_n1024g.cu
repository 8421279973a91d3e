// Kernel instantiations for N = 1024: generic mixed-L kernels.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(1024, 0)
}  // namespace fcw
