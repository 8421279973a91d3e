// Kernel instantiations for N = 1024, L = 16 with the narrowband long transforms (ZV = 2).
#include "fcw_k_inst.cuh"

namespace fcw {
FCW_KERNELS_NLN(1024, 16)
}  // namespace fcw
