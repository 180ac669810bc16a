// k_i8.cu — instantiations of the FP64-accurate INT8-sliced MTTKRP variants, mttkrp_i8.cuh.
#include "kernels.h"

namespace jk {
I8Fn i8_kernel(int variant) {
  if (variant == 1) return mttkrp_i8_kernel<kI8ResStages, true>;
  if (variant == 0) return mttkrp_i8_kernel<kI8Stages, false>;
  return mttkrp_i8_kernel<kI8Stages, false, true>;
}
}  // namespace jk
