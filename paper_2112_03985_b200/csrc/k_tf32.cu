// k_tf32.cu — instantiations of the FP32-path (3xTF32 tcgen05) MTTKRP, mttkrp_tf32.cuh:
// one-CTA (cta_group::1) and CTA-pair (cta_group::2) variants per ring depth.
#include "kernels.h"

namespace jk {
TfFn tf32_kernel(int stages, bool pair) {
  if (pair) {
    switch (stages) {
      case 8: return mttkrp_tf32_kernel<8, true>;
      case 6: return mttkrp_tf32_kernel<6, true>;
      case 4: return mttkrp_tf32_kernel<4, true>;
      default: return mttkrp_tf32_kernel<3, true>;
    }
  }
  switch (stages) {
    case 8: return mttkrp_tf32_kernel<8>;
    case 6: return mttkrp_tf32_kernel<6>;
    case 4: return mttkrp_tf32_kernel<4>;
    default: return mttkrp_tf32_kernel<3>;
  }
}
}  // namespace jk
