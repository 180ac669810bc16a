// k_epi.cu — the per-submodel ALS epilogue kernels (epilogue.cuh) of one rank class.
// Compiled once per class: -DJK_RMAX={2,4,6,8,10,12,16}.
#include "kernels.h"

#ifndef JK_RMAX
#error "compile with -DJK_RMAX=<rank class>"
#endif
#define JK_CAT2(a, b) a##b
#define JK_CAT(a, b) JK_CAT2(a, b)

namespace jk {
EpiFns JK_CAT(epi_kernels_, JK_RMAX)() {
  EpiFns f;
  f.smem = als_epilogue_kernel<JK_RMAX>;
  f.mixed = als_epilogue_mixed_kernel<JK_RMAX>;
  f.rows = als_epilogue_rows_kernel<JK_RMAX>;
  return f;
}
}  // namespace jk
