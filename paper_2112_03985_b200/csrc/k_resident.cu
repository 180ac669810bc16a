// k_resident.cu — instantiations of the whole-iterate kernels for small tensors: cluster-resident
// (resident.cuh) and warp-per-submodel (warp_resident.cuh).
#include "kernels.h"

namespace jk {
ResFn resident_kernel(int rclass) {
  if (rclass <= 2) return resident_sweep_kernel<2>;
  if (rclass <= 4) return resident_sweep_kernel<4>;
  return resident_sweep_kernel<8>;
}
template <int NM>
static WrFn wr_pick(int rclass) {
  if (rclass <= 2) return warp_sweep_kernel<2, NM>;
  if (rclass <= 4) return warp_sweep_kernel<4, NM>;
  return warp_sweep_kernel<8, NM>;
}
WrFn warp_resident_kernel(int rclass, int N) {
  if (N == 3) return wr_pick<3>(rclass);
  if (N == 4) return wr_pick<4>(rclass);
  if (N == 5) return wr_pick<5>(rclass);
  return nullptr;  // N > 5: the other paths
}
}  // namespace jk
