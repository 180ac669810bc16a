// k_tf32.cu — instantiations of the FP32-path (3xTF32 tcgen05) MTTKRP, mttkrp_tf32.cuh:
// one-CTA (cta_group::1) and CTA-pair (cta_group::2) variants per ring depth (2, 3, 4) and per
// j'-values-per-k-tile (1, 2, 4).
#include "kernels.h"

namespace jk {
template <bool PAIR, int JM>
static TfFn tf32_pick(int stages) {
  switch (stages) {
    case 4: return mttkrp_tf32_kernel<4, PAIR, JM>;
    case 3: return mttkrp_tf32_kernel<3, PAIR, JM>;
    default: return mttkrp_tf32_kernel<2, PAIR, JM>;
  }
}
TfFn tf32_kernel(int stages, bool pair, int jm) {
  if (pair) return jm >= 4 ? tf32_pick<true, 4>(stages) : jm == 2 ? tf32_pick<true, 2>(stages) : tf32_pick<true, 1>(stages);
  return jm >= 4 ? tf32_pick<false, 4>(stages) : jm == 2 ? tf32_pick<false, 2>(stages) : tf32_pick<false, 1>(stages);
}
}  // namespace jk
