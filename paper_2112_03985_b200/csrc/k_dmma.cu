// k_dmma.cu — instantiations of the FP64 DMMA MTTKRP (mttkrp.cuh) for one B-operand layout and
// one k-tile depth. Compiled four times: -DJK_KMAJOR=0|1 (mode 0: i_n contiguous in T; modes >= 1)
// x -DJK_KB=16|20 (i_q0 values per k-tile). Two tile widths each: 8 consumer warps (128 fused
// columns) and 5 (80 columns, e.g. C = 400).
#include "kernels.h"

#if !defined(JK_KMAJOR) || !defined(JK_KB)
#error "compile with -DJK_KMAJOR=0|1 -DJK_KB=16|20"
#endif
#define JK_CAT4(a, b, c, d) a##b##c##d
#define JK_NAME(km, kb) JK_CAT4(dmma_kernels_km, km, _kb, kb)

namespace jk {
namespace {
template <int NT, int ST, int WM>
size_t smem_of(int nslow) { return MttkrpCfg<NT, (JK_KMAJOR != 0), ST, WM, JK_KB>::smem_bytes(nslow); }

template <int ST, int WM, int... NTs>
void fill(MttkrpFn* fns, SmemFn* sm) {
  int i = 0;
  ((fns[i] = mttkrp_dmma_kernel<NTs, (JK_KMAJOR != 0), ST, WM, JK_KB>, sm[i] = smem_of<NTs, ST, WM>, ++i), ...);
}
}  // namespace

void JK_NAME(JK_KMAJOR, JK_KB)(MttkrpFn fn[kNumWM][2][kMaxNT], SmemFn smem[kNumWM][2][kMaxNT]) {
  fill<2, kWMs[0], 1, 2, 3, 4, 5, 6, 7, 8>(fn[0][0], smem[0][0]);
  fill<4, kWMs[0], 1, 2, 3, 4, 5, 6, 7, 8>(fn[0][1], smem[0][1]);
  fill<2, kWMs[1], 1, 2, 3, 4, 5, 6, 7, 8>(fn[1][0], smem[1][0]);
  fill<4, kWMs[1], 1, 2, 3, 4, 5, 6, 7, 8>(fn[1][1], smem[1][1]);
}
}  // namespace jk
