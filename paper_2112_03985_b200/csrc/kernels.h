// kernels.h — host-side handles of the kernels compiled in their own translation units.
//
// The heavy templated kernels (the FP64 DMMA MTTKRP variants, the FP32 and INT8 tcgen05 MTTKRPs,
// the per-rank-class epilogues) are instantiated in separate .cu files (k_*.cu) so that the
// library builds in parallel; each file exports plain getters returning the kernels' host stubs,
// which jkcals.cu launches with cudaLaunchKernelEx / <<<>>> on a function pointer.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "epilogue.cuh"
#include "mttkrp.cuh"
#include "mttkrp_i8.cuh"
#include "mttkrp_tf32.cuh"
#include "resident.cuh"
#include "warp_resident.cuh"

namespace jk {

typedef void (*MttkrpFn)(const CUtensorMap, const CUtensorMap, MttkrpView, MttkrpGeom, const TileInfo*, double*);
typedef size_t (*SmemFn)(int);
// k_dmma.cu (compiled once per KMAJOR): fn[wv][st][nt - 1]: wv indexes the consumer-warp count
// kWMs[wv] (tile width 16 x WM columns), st = 0 -> 2 stages, 1 -> 4 stages
constexpr int kNumWM = 2;
constexpr int kWMs[kNumWM] = {8, 5};
// and k-tile depth kKBs[kv] (i_q0 values per k-tile: 16, or 20 when it divides I_q0 better)
constexpr int kNumKB = 2;
constexpr int kKBs[kNumKB] = {16, 20};
void dmma_kernels_km0_kb16(MttkrpFn fn[kNumWM][2][kMaxNT], SmemFn smem[kNumWM][2][kMaxNT]);
void dmma_kernels_km1_kb16(MttkrpFn fn[kNumWM][2][kMaxNT], SmemFn smem[kNumWM][2][kMaxNT]);
void dmma_kernels_km0_kb20(MttkrpFn fn[kNumWM][2][kMaxNT], SmemFn smem[kNumWM][2][kMaxNT]);
void dmma_kernels_km1_kb20(MttkrpFn fn[kNumWM][2][kMaxNT], SmemFn smem[kNumWM][2][kMaxNT]);

typedef void (*TfFn)(const CUtensorMap, const CUtensorMap, const CUtensorMap, MttkrpView, TfGeom, const TileInfo*,
                     double*);
TfFn tf32_kernel(int stages, bool pair = false, int jm = 1);  // k_tf32.cu: stages {2,3,4}, pair: cta_group::2, jm {1,2,4}

typedef void (*I8Fn)(const CUtensorMap, const CUtensorMap, I8Geom, const TileInfo*, double*);
I8Fn i8_kernel(int variant);  // k_i8.cu: 0 streaming, 1 resident A, 2 2-CTA cluster

typedef void (*EpiFn)(EpiArgs);
struct EpiFns {
  EpiFn smem, mixed, rows;
};
// k_epi.cu, compiled once per rank class RMAX in {2, 4, 6, 8, 10, 12, 16}
EpiFns epi_kernels_2();
EpiFns epi_kernels_4();
EpiFns epi_kernels_6();
EpiFns epi_kernels_8();
EpiFns epi_kernels_10();
EpiFns epi_kernels_12();
EpiFns epi_kernels_16();

// k_large.cu: ranks 17..32
typedef void (*GramLargeFn)(const double*, int, int64_t, int, const int*, const int*, const int*, int, int, double*);
EpiFn epi_large_kernel();
GramLargeFn gram_large_kernel_fn();

// k_resident.cu: the cluster-resident whole-iterate kernel for small tensors (resident.cuh)
typedef void (*ResFn)(ResArgs);
ResFn resident_kernel(int rclass);  // rank class: 2, 4 or 8
typedef void (*WrFn)(WrArgs);
WrFn warp_resident_kernel(int rclass, int N);  // tiny tensors, N <= 5 (nullptr otherwise): one warp per submodel

}  // namespace jk
