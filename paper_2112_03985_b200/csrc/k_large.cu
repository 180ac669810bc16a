// k_large.cu — the streaming epilogue and Gramian for ranks 17..32 (epilogue_large.cuh).
#define JK_TU_LARGE
#include "kernels.h"
#include "epilogue_large.cuh"

namespace jk {
EpiFn epi_large_kernel() { return als_epilogue_large_kernel; }
GramLargeFn gram_large_kernel_fn() { return gram_large_kernel; }
}  // namespace jk
