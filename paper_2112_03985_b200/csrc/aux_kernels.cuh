// aux_kernels.cuh — the one-time and bookkeeping kernels around the hot loop:
// slice norms (a0), warm-start broadcast (a0, Alg. 3 alg:start-jk-1..alg:stop-jk-1),
// initial Gramians (a0/a3), factor extraction (a9), jackknife moments (a9, Alg. 2
// alg:jk:std) and masked compaction of converged submodels (a8).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "epilogue.cuh"

namespace jk {

// (a0) mode-0 slice norms, pass 1: CTA b sums T(i0, j)^2 over its chunk of columns j of
// T_(0) (column-major, so consecutive threads read consecutive i0: coalesced).
__global__ void slice_norms_partial_kernel(const double* __restrict__ T, int64_t I0, int64_t ld, int64_t J0,
                                           int64_t chunk, double* __restrict__ part) {
  const int64_t j0 = (int64_t)blockIdx.x * chunk, j1 = min(J0, j0 + chunk);
  for (int64_t i = threadIdx.x; i < I0; i += blockDim.x) {
    double s = 0.0;
    // unrolled so that 8 loads are in flight per thread; the adds stay in column order
#pragma unroll 8
    for (int64_t j = j0; j < j1; ++j) {
      double x = __ldcs(T + i + ld * j);
      s += x * x;
    }
    part[(int64_t)blockIdx.x * I0 + i] = s;
  }
}

// pass 2 (single CTA): s_p = sum_b part[b][p] in order; ||T||^2 = sum_p s_p in order;
// ||T_-p||^2 = ||T||^2 - s_p for every submodel; delete-d:
// ||T_-g||^2 = ||T||^2 - sum_{i in group} s_i.
__global__ void slice_norms_final_kernel(const double* __restrict__ part, int nb, int64_t I0,
                                         double* __restrict__ s, double* __restrict__ normT2,
                                         const int64_t* __restrict__ pglob, int d, int nsub,
                                         double* __restrict__ normT2p) {
  for (int64_t i = threadIdx.x; i < I0; i += blockDim.x) {
    double acc = 0.0;
#pragma unroll 8
    for (int b = 0; b < nb; ++b) acc += part[(int64_t)b * I0 + i];  // (8 loads in flight, adds in order)
    s[i] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int64_t i = 0; i < I0; ++i) tot += s[i];
    *normT2 = tot;
    for (int q = 0; q < nsub; ++q) {
      const int64_t p0 = pglob[q], p1 = (p0 + d < I0) ? p0 + d : I0;
      double rm = 0.0;
      for (int64_t i = p0; i < p1; ++i) rm += s[i];
      normT2p[q] = tot - rm;
    }
  }
}

// (a0) warm start: block k of the mode-n multi-factor = P_n of its submodel's model. `P` is the
// column concatenation [P_n(model 0) | P_n(model 1) | ...] (host col-major I x sum_m R_m staged on
// the device); block k (columns [blkcol[k], blkcol[k] + R_k)) takes columns [subRc, subRc + R_k)
// of it. The mode-0 block k gets its group's rows [p_k, p_k + d) zeroed (Alg. 3
// alg:cals_jk:multifactor0; delete-d PAPER.md:416-417). The caller zeroes U first (padding).
__global__ void init_blocks_kernel(const double* __restrict__ P, int I, int Rs, int K, int64_t ldu,
                                   double* __restrict__ U, int zero_rows, const int* __restrict__ blk2sub,
                                   const int* __restrict__ blkcol, const int* __restrict__ subR,
                                   const int* __restrict__ subRc, const int64_t* __restrict__ pglob, int d) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)I * K * Rs) return;
  const int r = (int)(e % Rs);
  const int k = (int)((e / Rs) % K);
  const int i = (int)(e / ((int64_t)Rs * K));
  const int sub = blk2sub[k];
  if (r >= subR[sub]) return;
  double v = P[i + (int64_t)I * (subRc[sub] + r)];
  if (zero_rows && i >= pglob[sub] && i < pglob[sub] + d) v = 0.0;
  U[(int64_t)i * ldu + blkcol[k] + r] = v;
}

// one submodel's block from a host-provided col-major matrix (set_init_submodel): mode 0
// arrives without its group's rows [pdrop, pdrop + cnt), which are re-inserted as zeros.
__global__ void set_block_kernel(const double* __restrict__ src, int I, int R, int64_t ldu, int col,
                                 int64_t pdrop, int cnt, double* __restrict__ U) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= I * R) return;
  const int i = e / R, r = e % R;
  double v;
  if (pdrop >= 0) {
    const int rows = I - cnt;
    v = (i >= pdrop && i < pdrop + cnt) ? 0.0 : src[(i < pdrop ? i : i - cnt) + (int64_t)rows * r];
  } else {
    v = src[i + (int64_t)I * r];
  }
  U[(int64_t)i * ldu + col + r] = v;
}

// Gramian of one block (one CTA per live block): Gram_n^(sub) = U_blk^T U_blk.
// Block k spans columns [blkcol[k], blkcol[k] + R_k); gram is [N][nsub][Rs*Rs] (R_k x R_k used).
template <int RMAX>
__global__ void __launch_bounds__(kEpiThreads) gram_kernel(const double* __restrict__ U, int I, int64_t ldu,
                                                           int Rs, const int* __restrict__ blk2sub,
                                                           const int* __restrict__ blkcol,
                                                           const int* __restrict__ subR, int nsub, int n,
                                                           double* __restrict__ gram) {
  const int k = blockIdx.x, sub = blk2sub[k], R = subR[sub];
  __shared__ double red[(kEpiThreads / 32 + 1) * (RMAX * RMAX + RMAX + 1)];
  double g[RMAX * RMAX];
#pragma unroll
  for (int e = 0; e < RMAX * RMAX; ++e) g[e] = 0.0;
  for (int i = threadIdx.x; i < I; i += kEpiThreads) {
    const double* row = U + (int64_t)i * ldu + blkcol[k];
    double u[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) u[r] = r < R ? row[r] : 0.0;
#pragma unroll
    for (int r = 0; r < RMAX; ++r)
#pragma unroll
      for (int q = 0; q < RMAX; ++q) g[r * RMAX + q] += u[r] * u[q];
  }
  block_sum<RMAX>(g, RMAX * RMAX, red);
  const double* gt = red + (kEpiThreads / 32) * RMAX * RMAX;
  for (int e = threadIdx.x; e < R * R; e += kEpiThreads)
    gram[((int64_t)n * nsub + sub) * Rs * Rs + e] = gt[(e / R) * RMAX + (e % R)];
}

// reset per-submodel state at set_init
__global__ void reset_state_kernel(int nsub, double* fit, double* fit_prev, double* err, int* iters, int* flags,
                                   int* active) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nsub) return;
  fit[q] = 0.0;
  fit_prev[q] = 0.0;
  err[q] = 0.0;
  iters[q] = 0;
  flags[q] = 0;
  active[q] = 1;
}

// (a9) extract a row-major (stride ld) I x R block into a column-major output, dropping
// rows [drop, drop + cnt) (the left-out group's zero rows in mode 0) when drop >= 0.
__global__ void extract_kernel(const double* __restrict__ src, int64_t ld, int I, int R, int64_t drop,
                               int cnt, double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int rows = drop >= 0 ? I - cnt : I;
  if (e >= rows * R) return;
  const int r = e / rows, io = e % rows;
  const int i = (drop >= 0 && io >= drop) ? io + cnt : io;
  out[e] = src[(int64_t)i * ld + r];
}

// (a9) every submodel's mode block at once: submodel q's column-major rows_q x R_q block goes to
// out + dstoff[q] (mode 0: its group's rows [p_q, p_q + |group|) dropped, |group| = min(d, I - p_q)).
// grid.y strides over submodels.
__global__ void extract_all_kernel(const double* __restrict__ base, const int64_t* __restrict__ src_off,
                                   const int64_t* __restrict__ src_ld, const int* __restrict__ subR,
                                   const int64_t* __restrict__ dstoff, int nsub, int I, int drop,
                                   const int64_t* __restrict__ pglob, int d, double* __restrict__ out) {
  for (int q = blockIdx.y; q < nsub; q += gridDim.y) {
    const int R = subR[q];
    const int64_t p = drop ? pglob[q] : -1;
    const int cnt = drop ? (int)((p + d < I) ? d : I - p) : 0;
    const int rows = I - cnt;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * R; e += gridDim.x * blockDim.x) {
      const int r = e / rows, io = e % rows;
      const int i = (drop && io >= p) ? io + cnt : io;
      out[dstoff[q] + e] = base[src_off[q] + (int64_t)i * src_ld[q] + r];
    }
  }
}

// (a9) per-element moments over the handle's submodels (two-pass: mean = sum/g, M2 = sum
// (x - mean)^2). One warp per element: lanes stride over the submodels, then a shuffle tree --
// a fixed order, so the result is deterministic. src_off[q] / src_ld[q] locate submodel q's
// block (row-major) relative to `base`. Output column-major I x R.
__global__ void moments_kernel(const double* __restrict__ base, const int64_t* __restrict__ src_off,
                               const int64_t* __restrict__ src_ld, int nsub, int I, int R,
                               double* __restrict__ mean, double* __restrict__ m2) {
  const int lane = threadIdx.x & 31;
  const int e = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (e >= I * R) return;  // (warp-uniform)
  const int r = e / I, i = e % I;
  double s = 0.0;
  for (int q = lane; q < nsub; q += 32) s += base[src_off[q] + (int64_t)i * src_ld[q] + r];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const double mu = s / (double)nsub;
  double ss = 0.0;
  for (int q = lane; q < nsub; q += 32) {
    const double d = base[src_off[q] + (int64_t)i * src_ld[q] + r] - mu;
    ss += d * d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) {
    mean[e] = mu;
    m2[e] = ss;
  }
}

// (a8) store a converged block (columns [col, col + R)) into the result store (row-major I x R).
__global__ void store_block_kernel(const double* __restrict__ U, int I, int64_t ldu, int R, int col,
                                   double* __restrict__ dst) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= I * R) return;
  const int i = e / R, r = e % R;
  dst[e] = U[(int64_t)i * ldu + col + r];
}

// (a8) the same for every block converged since the last compaction in one launch per mode:
// tab[3 y .. 3 y + 2] = (first column, rank R, slot) of block y; its mode-n block lands at
// Ures + slot * slot_doubles + sum_{m<n} I_m * R (the per-slot result store layout)
__global__ void store_blocks_kernel(const double* __restrict__ U, int I, int64_t ldu, const int* __restrict__ tab,
                                    int64_t slot_doubles, int64_t sumIprev, double* __restrict__ Ures) {
  const int y = blockIdx.y;
  const int col = tab[3 * y], R = tab[3 * y + 1], slot = tab[3 * y + 2];
  double* dst = Ures + (int64_t)slot * slot_doubles + sumIprev * R;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < I * R; e += gridDim.x * blockDim.x) {
    const int i = e / R, r = e % R;
    dst[e] = U[(int64_t)i * ldu + col + r];
  }
}

// (a8) masked compaction: gather the surviving blocks' columns (new column c <- old column
// colmap[c]) to the front of the other multi-factor buffer; columns >= C_new become zero padding.
__global__ void gather_blocks_kernel(const double* __restrict__ Uold, double* __restrict__ Unew, int I,
                                     int64_t ldu, const int* __restrict__ colmap, int Cnew) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)I * ldu) return;
  const int i = (int)(e / ldu), c = (int)(e % ldu);
  Unew[e] = (c < Cnew) ? Uold[(int64_t)i * ldu + colmap[c]] : 0.0;
}

// Tolerance-mode loop condition (body tail of the WHILE graph node, jkcals.cu ensure_tol_graph):
// misc ints [4] active submodels after this sweep (the N-1 epilogue's count), [6] sweeps run by
// this launch, [8] sweep budget, [9] compaction threshold. Continue while the budget lasts, some
// submodel is active and fewer than 64 fused columns have converged (Alg. 3 stop / a8 compaction).
__global__ void tol_decide_kernel(int* __restrict__ misc_i, cudaGraphConditionalHandle hnd) {
  const int nact = misc_i[4];
  const int sw = misc_i[6] + 1;
  misc_i[6] = sw;
  cudaGraphSetConditional(hnd, (sw < misc_i[8] && nact > misc_i[9]) ? 1u : 0u);
}

}  // namespace jk
