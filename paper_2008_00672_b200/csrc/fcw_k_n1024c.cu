// Kernel instantiations for N = 1024: uniform-L specialisations L = 512, 1024.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(1024, 512)
FCW_KERNELS_NL(1024, 1024)
}  // namespace fcw
