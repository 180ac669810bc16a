// k_resident.cu — instantiations of the cluster-resident whole-iterate kernel (resident.cuh).
#include "kernels.h"

namespace jk {
ResFn resident_kernel(int rclass) {
  if (rclass <= 2) return resident_sweep_kernel<2>;
  if (rclass <= 4) return resident_sweep_kernel<4>;
  return resident_sweep_kernel<8>;
}
}  // namespace jk
