// k_dmma.cu — instantiations of the FP64 DMMA MTTKRP (mttkrp.cuh) for one B-operand layout.
// Compiled twice: -DJK_KMAJOR=0 (mode 0: i_n contiguous in T) and -DJK_KMAJOR=1 (modes >= 1).
// Two tile widths: 8 consumer warps (128 fused columns) and 5 (80 columns, e.g. C = 400).
#include "kernels.h"

#ifndef JK_KMAJOR
#error "compile with -DJK_KMAJOR=0 or 1"
#endif

namespace jk {
namespace {
template <int NT, int ST, int WM>
size_t smem_of(int nslow) { return MttkrpCfg<NT, (JK_KMAJOR != 0), ST, WM>::smem_bytes(nslow); }

template <int ST, int WM, int... NTs>
void fill(MttkrpFn* fns, SmemFn* sm) {
  int i = 0;
  ((fns[i] = mttkrp_dmma_kernel<NTs, (JK_KMAJOR != 0), ST, WM>, sm[i] = smem_of<NTs, ST, WM>, ++i), ...);
}
}  // namespace

#if JK_KMAJOR
void dmma_kernels_km1(MttkrpFn fn[kNumWM][2][kMaxNT], SmemFn smem[kNumWM][2][kMaxNT]) {
#else
void dmma_kernels_km0(MttkrpFn fn[kNumWM][2][kMaxNT], SmemFn smem[kNumWM][2][kMaxNT]) {
#endif
  fill<2, kWMs[0], 1, 2, 3, 4, 5, 6, 7, 8>(fn[0][0], smem[0][0]);
  fill<4, kWMs[0], 1, 2, 3, 4, 5, 6, 7, 8>(fn[0][1], smem[0][1]);
  fill<2, kWMs[1], 1, 2, 3, 4, 5, 6, 7, 8>(fn[1][0], smem[1][0]);
  fill<4, kWMs[1], 1, 2, 3, 4, 5, 6, 7, 8>(fn[1][1], smem[1][1]);
}
}  // namespace jk
