// Kernel instantiations for N = 4096: uniform-L specialisations L = 512, 1024.
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NL(4096, 512)
FCW_KERNELS_NL(4096, 1024)
}  // namespace fcw
