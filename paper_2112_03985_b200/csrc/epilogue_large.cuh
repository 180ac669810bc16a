// epilogue_large.cuh — the per-submodel ALS step for ranks 17..32.
//
// Same arithmetic as als_epilogue_kernel (Hadamard of cached Gramians, Cholesky with a Jacobi
// pseudoinverse fallback, the zero rows of the left-out group, 2-norm normalisation, the new
// Gramian, error / fit / convergence), restructured so that nothing scales as R^2 per thread:
//   * the Cholesky factor is built column by column by one warp in shared memory;
//   * rows stream through shared memory in chunks of kLgRows; each thread solves one row in place
//     (forward / back substitution against L in shared memory);
//   * each of the R(R+1)/2 entries of V^T V (and each column of V.M) is owned by ONE thread, which
//     accumulates it over all rows in a fixed order -- no cross-thread reduction, deterministic;
//   * V is written to U, then a second pass scales U by 1/lambda.
// It serves any I_n (rows are streamed), so it is also the large-I_n path for these ranks. The
// paper's second application (44 x 2700 x 200 with R in {19, 20, 21}) needs it.
#pragma once
#include "epilogue.cuh"

namespace jk {

constexpr int kLgThreads = 256;

// The Jacobi pseudoinverse of epilogue.cuh's jacobi_pinv (same rotations, same order, same
// rcond rule) on caller-provided work arrays, so that R up to 32 does not need 16 KB of stack
// per thread: A and Q are R x R scratch in shared memory, Hp is written with row stride ldp.
static __device__ __noinline__ void jacobi_pinv_ptr(const double* H, int R, double* A, double* Q, double* Hp, int ldp,
                                             double rcond) {
  for (int e = 0; e < R * R; ++e) { A[e] = H[e]; Q[e] = 0.0; }
  for (int i = 0; i < R; ++i) Q[i * R + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j) {
        double x = A[i * R + j];
        tot += x * x;
        if (i != j) off += x * x;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < R - 1; ++p)
      for (int q = p + 1; q < R; ++q) {
        double apq = A[p * R + q];
        if (apq == 0.0) continue;
        double theta = (A[q * R + q] - A[p * R + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < R; ++k) {
          double akp = A[k * R + p], akq = A[k * R + q];
          A[k * R + p] = c * akp - sn * akq;
          A[k * R + q] = sn * akp + c * akq;
        }
        for (int k = 0; k < R; ++k) {
          double apk = A[p * R + k], aqk = A[q * R + k];
          A[p * R + k] = c * apk - sn * aqk;
          A[q * R + k] = sn * apk + c * aqk;
        }
        for (int k = 0; k < R; ++k) {
          double qkp = Q[k * R + p], qkq = Q[k * R + q];
          Q[k * R + p] = c * qkp - sn * qkq;
          Q[k * R + q] = sn * qkp + c * qkq;
        }
      }
  }
  double wmax = 0.0;
  for (int i = 0; i < R; ++i) wmax = fmax(wmax, A[i * R + i]);
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R; ++b) Hp[a * ldp + b] = 0.0;
  for (int i = 0; i < R; ++i) {
    double w = A[i * R + i];
    if (!(w > rcond * wmax) || w <= 0.0) continue;
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b) Hp[a * ldp + b] += Q[a * R + i] * Q[b * R + i] / w;
  }
}
constexpr int kLgRMax = 32;
constexpr int kLgRows = 256;           // rows per chunk: one row per thread
constexpr int kLgLd = kLgRMax + 1;     // odd row stride: thread-per-row accesses hit distinct banks
// Ms + Vs = 2 x 256 x 33 x 8 = 132 KB of dynamic shared memory (opt-in; one CTA per SM)
inline size_t epi_large_smem_bytes() { return (size_t)2 * kLgRows * kLgLd * sizeof(double); }
#ifdef JK_TU_LARGE

__global__ void __launch_bounds__(kLgThreads) als_epilogue_large_kernel(EpiArgs a) {
  const int k = blockIdx.x;
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the MTTKRP grid has completed
  asm volatile("griddepcontrol.launch_dependents;\n" :::);
  if (a.n == 0 && k == 0 && threadIdx.x == 0) *a.active_count = 0;  // per-sweep counter reset
  const int sub = a.blk2sub[k];
  if (!a.active[sub]) return;  // frozen (converged or failed)
  const int R = a.subR ? a.subR[sub] : a.R, Rs = a.R, n = a.n, N = a.N, tid = threadIdx.x, In = a.In;
  const int lane = tid & 31, warp = tid >> 5;
  const bool last = (n == N - 1);
  const int64_t pz0 = (n == 0) ? a.pglob[sub] : -1;  // padded rows [pz0, pz1)
  const int64_t pz1 = (n == 0) ? pz0 + a.d : -1;
  const int cb = a.blkcol ? a.blkcol[k] : k * R;
  const int NQ = R * (R + 1) / 2;

  __shared__ double H[kLgRMax * kLgRMax];
  __shared__ double L[kLgRMax * kLgRMax];  // lower Cholesky factor (row-major) or H^+ (pinv)
  __shared__ double tot[kLgRMax * (kLgRMax + 1) / 2 + kLgRMax];  // V^T V upper triangle, then V.M per column
  __shared__ double ilam_s[kLgRMax];
  __shared__ int use_pinv;
  extern __shared__ double dyn[];
  double* Ms = dyn;                    // [kLgRows][kLgLd]
  double* Vs = dyn + kLgRows * kLgLd;  // [kLgRows][kLgLd]

  // (a3) Hadamard of the cached Gramians of every other mode
  for (int e = tid; e < R * R; e += kLgThreads) {
    double h = 1.0;
    for (int m = 0; m < N; ++m)
      if (m != n) h *= a.gram[((int64_t)m * a.nsub + sub) * Rs * Rs + e];
    H[e] = h;
  }
  __syncthreads();
  // (a4) Cholesky H = L L^T (textbook, no pivoting), column by column by warp 0
  if (warp == 0) {
    bool ok = true;
    for (int j = 0; j < R; ++j) {
      double s = 0.0;
      if (lane == 0) {
        s = H[j * R + j];
        for (int q = 0; q < j; ++q) s -= L[j * kLgRMax + q] * L[j * kLgRMax + q];
      }
      s = __shfl_sync(0xffffffffu, s, 0);
      if (!(s > 0.0) || !isfinite(s)) {
        ok = false;
        break;
      }
      const double d = sqrt(s);
      if (lane == 0) L[j * kLgRMax + j] = d;
      for (int i = j + 1 + lane; i < R; i += 32) {
        double t = H[i * R + j];
        for (int q = 0; q < j; ++q) t -= L[i * kLgRMax + q] * L[j * kLgRMax + q];
        L[i * kLgRMax + j] = t / d;
      }
      __syncwarp();
    }
    if (lane == 0) use_pinv = ok ? 0 : 1;
  }
  __syncthreads();
  if (use_pinv) {  // (the chunk buffers are free until the row loop: Jacobi scratch)
    if (tid == 0) {
      jacobi_pinv_ptr(H, R, Ms, Vs, L, kLgRMax, 1e-12);
      a.flags[sub] |= F_PINV;
    }
    __syncthreads();
  }
  const bool pinv = use_pinv != 0;

  // each thread owns up to kOwn (r, c) entries of V^T V (upper triangle) and thread r < R owns
  // column r of V.M; sums run over rows in order
  constexpr int kOwn = (kLgRMax * (kLgRMax + 1) / 2 + kLgThreads - 1) / kLgThreads;  // 3
  int own_r[kOwn], own_c[kOwn];
  double own_acc[kOwn];
#pragma unroll
  for (int o = 0; o < kOwn; ++o) {
    own_r[o] = -1;
    own_c[o] = -1;
    own_acc[o] = 0.0;
    const int q = tid + o * kLgThreads;
    if (q < NQ) {  // q -> (r, c), r <= c, packed upper triangle by rows
      int r = 0, base = 0;
      while (base + (R - r) <= q) {
        base += R - r;
        ++r;
      }
      own_r[o] = r;
      own_c[o] = r + (q - base);
    }
  }
  double cross = 0.0;

  const int64_t piece = (int64_t)a.BN * a.BM;
  for (int i0 = 0; i0 < In; i0 += kLgRows) {
    const int rows = min(kLgRows, In - i0);
    // (a2) fixed-order sum of this chunk's partial pieces
    for (int e = tid; e < rows * R; e += kLgThreads) {
      const int il = e / R, r = e % R;
      const int i = i0 + il, c = cb + r, tn = i / a.BN, tm = c / a.BM;
      const TileInfo ti = a.tinfo[tn * a.nMt + tm];
      const double* p = a.parts + (int64_t)ti.piece_base * piece + (int64_t)(i - tn * a.BN) * a.BM + (c - tm * a.BM);
      double s = 0.0;
      for (int pc = 0; pc < ti.npieces; ++pc) s += __ldcg(p + (int64_t)pc * piece);
      Ms[il * kLgLd + r] = s;
    }
    __syncthreads();
    // (a4/a5) row solves V(i,:) = M(i,:) H^{-1}, one row per thread, in shared memory
    for (int il = tid; il < rows; il += kLgThreads) {
      const int64_t i = i0 + il;
      const double* m = Ms + il * kLgLd;
      double* v = Vs + il * kLgLd;
      if (i >= pz0 && i < pz1) {
        for (int r = 0; r < R; ++r) v[r] = 0.0;
      } else if (!pinv) {
        for (int r = 0; r < R; ++r) {  // L y = m
          double t = m[r];
          for (int q = 0; q < r; ++q) t -= L[r * kLgRMax + q] * v[q];
          v[r] = t / L[r * kLgRMax + r];
        }
        for (int r = R - 1; r >= 0; --r) {  // L^T v = y
          double t = v[r];
          for (int q = r + 1; q < R; ++q) t -= L[q * kLgRMax + r] * v[q];
          v[r] = t / L[r * kLgRMax + r];
        }
      } else {
        for (int r = 0; r < R; ++r) {
          double s = 0.0;
          for (int q = 0; q < R; ++q) s += m[q] * L[q * kLgRMax + r];
          v[r] = s;
        }
      }
    }
    __syncthreads();
    // owned sums over this chunk's rows, and V (un-normalised) to U
#pragma unroll
    for (int o = 0; o < kOwn; ++o)
      if (own_r[o] >= 0)
        for (int il = 0; il < rows; ++il) own_acc[o] += Vs[il * kLgLd + own_r[o]] * Vs[il * kLgLd + own_c[o]];
    if (tid < R)
      for (int il = 0; il < rows; ++il) cross += Vs[il * kLgLd + tid] * Ms[il * kLgLd + tid];
    for (int e = tid; e < rows * R; e += kLgThreads) {
      const int il = e / R, r = e % R;
      a.U[(int64_t)(i0 + il) * a.ldu + cb + r] = Vs[il * kLgLd + r];
    }
    __syncthreads();
  }
#pragma unroll
  for (int o = 0; o < kOwn; ++o)
    if (own_r[o] >= 0) {
      const int r = own_r[o], c = own_c[o];
      tot[r * R - r * (r - 1) / 2 + (c - r)] = own_acc[o];
    }
  if (tid < R) tot[NQ + tid] = cross;
  __syncthreads();
  auto vtv = [&](int r, int c) -> double {
    const int lo = r < c ? r : c, hi = r < c ? c : r;
    return tot[lo * R - lo * (lo - 1) / 2 + (hi - lo)];
  };
  // (a6) lambda_r = ||V(:,r)||, U = V / lambda; Gram of U = (V^T V) / (lambda lambda^T)
  if (tid < R) {
    const double lm = sqrt(vtv(tid, tid));
    ilam_s[tid] = lm > 0.0 ? 1.0 / lm : 1.0;
    a.lambda[(int64_t)sub * Rs + tid] = lm;
  }
  __syncthreads();
  for (int64_t e = tid; e < (int64_t)In * R; e += kLgThreads) {
    const int64_t i = e / R;
    const int r = (int)(e % R);
    double* u = a.U + i * a.ldu + cb + r;
    *u = *u * ilam_s[r];
  }
  for (int e = tid; e < R * R; e += kLgThreads) {
    const int r = e / R, c = e % R;
    a.gram[((int64_t)n * a.nsub + sub) * Rs * Rs + e] = vtv(r, c) * ilam_s[r] * ilam_s[c];
  }
  if (last && tid == 0) {  // (a7) error, fit, history, convergence mask
    double quad = 0.0, crs = 0.0;
    for (int r = 0; r < R; ++r) {
      crs += tot[NQ + r];
      for (int c = 0; c < R; ++c) quad += H[r * R + c] * vtv(r, c);
    }
    const double nt2 = a.normT2p[sub];
    const double e = nt2 + quad - 2.0 * crs;
    int it = a.iters[sub] + 1;
    a.iters[sub] = it;
    a.err[sub] = e;
    a.hist[(int64_t)sub * a.hist_cap + (it - 1) % a.hist_cap] = e;
    int f = a.flags[sub];
    bool act = true;
    if (!isfinite(e)) {
      f |= F_NONFINITE;
      act = false;
    } else {
      if (e < -1e-9 * nt2) f |= F_BREAKDOWN;
      const double fit = nt2 > 0.0 ? 1.0 - sqrt(fmax(e, 0.0)) / sqrt(nt2) : 0.0;
      const double tol = *a.tol;
      if (tol > 0.0 && it >= 2 && fabs(fit - a.fit_prev[sub]) < tol) {
        f |= F_CONVERGED;
        act = false;
      }
      a.fit[sub] = fit;
      a.fit_prev[sub] = fit;
    }
    a.flags[sub] = f;
    if (!act) a.active[sub] = 0;
    else atomicAdd(a.active_count, 1);
  }
}
#endif
#ifdef JK_TU_LARGE

// Gramian of one block for ranks 17..32 (set_init / set_init_submodel / import): each thread owns
// entries of U^T U and sums them over all rows in order.
__global__ void __launch_bounds__(kLgThreads) gram_large_kernel(const double* __restrict__ U, int I, int64_t ldu,
                                                                int Rs, const int* __restrict__ blk2sub,
                                                                const int* __restrict__ blkcol,
                                                                const int* __restrict__ subR, int nsub, int n,
                                                                double* __restrict__ gram) {
  const int k = blockIdx.x, sub = blk2sub[k], R = subR[sub];
  const double* base = U + blkcol[k];
  for (int e = threadIdx.x; e < R * R; e += kLgThreads) {
    const int r = e / R, c = e % R;
    double s = 0.0;
    for (int i = 0; i < I; ++i) s += base[(int64_t)i * ldu + r] * base[(int64_t)i * ldu + c];
    gram[((int64_t)n * nsub + sub) * Rs * Rs + e] = s;
  }
}
#endif

}  // namespace jk
