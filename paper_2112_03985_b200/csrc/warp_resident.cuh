// warp_resident.cuh — the whole JK-CALS iterate of a TINY tensor in one launch, one warp per
// submodel, no barrier on the sweep path.
//
// For tensors of a few thousand entries (the tiny config, 10x8x6) every step of a sweep is a few
// hundred cycles of work, and both the streamed path (6 kernel launches per sweep) and the
// cluster-resident kernel (CTA and cluster barriers per mode, resident.cuh) are bound by
// synchronisation latency. Here each CTA keeps the whole of T in shared memory and each of its
// warps owns ONE submodel (the instances are independent) with its factor
// blocks, Gramians and scratch in shared memory; the warp runs every sweep alone:
//   mode n: M(i, c) = sum_j T_(n)(i, j) prod_{m != n} U_m(i_m(j), c) with lanes over rows i and the
//   KRP row formed on the fly (Eq. 1, Alg. 3 alg:cals_jk:mttkrp); then the update of
//   Alg. 3 (alg:cals_jk:hadamard .. alg:cals_jk:error) with lane 0 factoring H,
//   lanes over rows for the solve and shuffle reductions for V^T V, V.M, lambda.
// Only __syncwarp on the sweep path; a converged warp stops on its own (tol > 0). Sums run in a
// fixed order: deterministic. State is written back as in resident.cuh.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "resident.cuh"

namespace jk {

constexpr int kWrWarps = 4;  // submodels (warps) per CTA

struct WrArgs {
  int N, R, d, hist_cap, max_iters, nsub, K;
  int dims[kMaxModes];
  int64_t gst[kMaxModes];  // workspace strides of T (mode-0 pitch I0p)
  int64_t ldu;
  int Pel;                 // prod(dims): T entries, compact in shared memory
  int warp_doubles;        // shared doubles per warp (factor blocks, M, V, Gramians, H, L)
  const double* T;
  double* U[kMaxModes];
  const int* blk2sub;
  const int64_t* pglob;
  double* gram;
  double* lambda;
  const double* normT2p;
  double *fit, *fit_prev, *err;
  int *iters, *flags, *active;
  double* hist;
  const double* tol;
  int* sweeps_out;
};

// per-warp shared doubles for rank R: factor blocks (sum I_m x R), M and V (maxI x R each),
// Gramians (N R^2), H, L (R^2 each), 1/L_jj (R)
__host__ __device__ inline int wr_warp_doubles(int N, const int* dims, int R) {
  int sumI = 0, maxI = 0;
  for (int m = 0; m < N; ++m) {
    sumI += dims[m];
    maxI = dims[m] > maxI ? dims[m] : maxI;
  }
  return sumI * R + 2 * maxI * R + N * R * R + 2 * R * R + R + 2 + 32 * R;  // (+ MTTKRP partials)
}

template <int RMAX, int NM>  // NM: the number of modes, compile-time (index arithmetic in registers)
__global__ void __launch_bounds__(kWrWarps * 32) warp_sweep_kernel(WrArgs a) {
  extern __shared__ __align__(16) double wr_smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int N = NM, last = NM - 1;
  const int R = a.R;
  double* Ts = wr_smem;  // T, column-major, compact strides
  // ---- T into shared memory (the only CTA-wide step)
  for (int e = tid; e < a.Pel; e += kWrWarps * 32) {
    int rem = e;
    int64_t go = 0;
    for (int m = 0; m < N; ++m) {
      const int im = rem % a.dims[m];
      rem /= a.dims[m];
      go += (int64_t)im * a.gst[m];
    }
    Ts[e] = a.T[go];
  }
  __syncthreads();
  const int k = blockIdx.x * kWrWarps + warp;  // this warp's block (submodel)
  if (k >= a.K) return;
  const int sub = a.blk2sub[k];
  int st[NM], uo[NM], dm[NM], maxI = 0;  // compact T strides, factor-block offsets, dims
  {
    int s = 1, o = 0;
#pragma unroll
    for (int m = 0; m < N; ++m) {
      dm[m] = a.dims[m];
      st[m] = s;
      s *= a.dims[m];
      uo[m] = o;
      o += a.dims[m] * R;
      maxI = max(maxI, a.dims[m]);
    }
  }
  double* W = wr_smem + ((a.Pel + 1) & ~1) + (size_t)warp * a.warp_doubles;
  double* Ub = W;                                  // [m][I_m][R]
  int sumIR = 0;
#pragma unroll
  for (int m = 0; m < N; ++m) sumIR += dm[m] * R;
  double* Ms = W + sumIR;                          // [maxI][R]
  double* Vs = Ms + maxI * R;                      // [maxI][R]
  double* Gs = Vs + maxI * R;                      // [N][R][R]
  double* H = Gs + N * R * R;
  double* Lf = H + R * R;
  double* Linv = Lf + R * R;
  double* Mp = Linv + R + 2;                       // [G][I_n][R] MTTKRP partials (I_n < 32)
  for (int m = 0; m < N; ++m)
    for (int e = lane; e < a.dims[m] * R; e += 32) {
      const int i = e / R, r = e % R;
      Ub[uo[m] + e] = a.U[m][(int64_t)i * a.ldu + (int64_t)k * R + r];
    }
  for (int e = lane; e < N * R * R; e += 32) {
    const int m = e / (R * R), rr = e % (R * R);
    Gs[e] = a.gram[((int64_t)m * a.nsub + sub) * R * R + rr];
  }
  const int64_t pz0 = a.pglob[sub];
  const double nt2 = a.normT2p[sub], tol = *a.tol;
  int it = a.iters[sub], fl = a.flags[sub];
  double fp = a.fit_prev[sub];
  bool act = a.active[sub] != 0;
  __syncwarp();

  int sweeps = 0;
  for (int s = 0; s < a.max_iters && act; ++s) {
    ++sweeps;
    // the mode loop is unrolled (NM is compile-time) so that q0, the slow modes and every array
    // index below are static: with a runtime n the slow-mode tables went to local memory (r02)
#pragma unroll
    for (int n = 0; n < NM; ++n) {
      int In = 0;
#pragma unroll
      for (int y = 0; y < NM; ++y)
        if (y == n) In = dm[y];
      // (a2) MTTKRP, lanes over rows: M(i, c) = sum_j' S_j'(c) sum_k T(i, k, j') U_q0(k, c), k = i_q0
      // the fastest other mode, j' the slower ones (Eq. 3 order); the KRP is never formed
      const int q0 = (n == 0) ? 1 : 0;
      int sdim[NM], sst[NM], suo[NM], sidx[NM];  // slow modes (ascending), entries [0, NM - 2)
#pragma unroll
      for (int z = 0; z < NM; ++z) sdim[z] = 1, sst[z] = 0, suo[z] = 0, sidx[z] = 0;
      int Jp = 1;
      {
        int zc = 0;  // (unrolled loops with compile-time bounds: every index below is static)
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          const bool sl = (m != n && m != q0);
#pragma unroll
          for (int z = 0; z < NM - 2; ++z)
            if (sl && z == zc) {
              sdim[z] = dm[m];
              sst[z] = st[m];
              suo[z] = uo[m];
            }
          if (sl) {
            Jp *= dm[m];
            ++zc;
          }
        }
      }
      int stn = 0, stq = 0, uoq = 0, Iq0 = 0;
#pragma unroll
      for (int y = 0; y < NM; ++y) {
        if (y == n) stn = st[y];
        if (y == q0) {
          stq = st[y];
          uoq = uo[y];
          Iq0 = dm[y];
        }
      }
      if (In < 32) {
        // short modes: lanes over (row i, j'-group g), G = 32 / I_n groups taking every G-th j',
        // the k chain split in two accumulators; the G partials of a row are then summed in g
        // order by lane i (fixed order: deterministic). r02: tiny 10.9 -> see DESIGN.md §9c
        const int G = 32 / In, i = lane % In, g = lane / In;
        if (g < G) {
          double acc[RMAX];
#pragma unroll
          for (int r = 0; r < RMAX; ++r) acc[r] = 0.0;
          const double* uq = Ub + uoq;
          for (int jp = g; jp < Jp; jp += G) {
            int rem = jp, toff = 0;
            double sv[RMAX];
#pragma unroll
            for (int r = 0; r < RMAX; ++r) sv[r] = 1.0;
#pragma unroll
            for (int z = 0; z < NM - 2; ++z) {
              const int iz = rem % sdim[z];
              rem /= sdim[z];
              toff += iz * sst[z];
              const double* ur = Ub + suo[z] + iz * R;
#pragma unroll
              for (int r = 0; r < RMAX; ++r)
                if (r < R) sv[r] *= ur[r];
            }
            double pe[RMAX], po[RMAX];
#pragma unroll
            for (int r = 0; r < RMAX; ++r) pe[r] = po[r] = 0.0;
            const double* t = Ts + i * stn + toff;
            int kk = 0;
            for (; kk + 2 <= Iq0; kk += 2) {
              const double a0 = t[kk * stq], a1 = t[(kk + 1) * stq];
#pragma unroll
              for (int r = 0; r < RMAX; ++r)
                if (r < R) {
                  pe[r] = fma(a0, uq[kk * R + r], pe[r]);
                  po[r] = fma(a1, uq[(kk + 1) * R + r], po[r]);
                }
            }
            if (kk < Iq0) {
              const double a0 = t[kk * stq];
#pragma unroll
              for (int r = 0; r < RMAX; ++r)
                if (r < R) pe[r] = fma(a0, uq[kk * R + r], pe[r]);
            }
#pragma unroll
            for (int r = 0; r < RMAX; ++r) acc[r] = fma(sv[r], pe[r] + po[r], acc[r]);
          }
#pragma unroll
          for (int r = 0; r < RMAX; ++r)
            if (r < R) Mp[(g * In + i) * R + r] = acc[r];
        }
        __syncwarp();
        if (lane < In) {
#pragma unroll
          for (int r = 0; r < RMAX; ++r)
            if (r < R) {
              double sm = Mp[lane * R + r];
              for (int q = 1; q < G; ++q) sm += Mp[(q * In + lane) * R + r];
              Ms[lane * R + r] = sm;
            }
        }
      } else {
        double acc[RMAX][2];  // [c][row slot] two rows per lane (In <= 64 typical)
        for (int i0 = lane; i0 < In; i0 += 64) {
          const int i1 = i0 + 32;
          const bool two = i1 < In;
  #pragma unroll
          for (int r = 0; r < RMAX; ++r) acc[r][0] = acc[r][1] = 0.0;
          int toff = 0;
  #pragma unroll
          for (int z = 0; z < NM - 2; ++z) sidx[z] = 0;
          for (int jp = 0; jp < Jp; ++jp) {
            double sv[RMAX];  // S_j'(c): the same on every lane (broadcast loads)
  #pragma unroll
            for (int r = 0; r < RMAX; ++r) sv[r] = 1.0;
  #pragma unroll
            for (int z = 0; z < NM - 2; ++z) {
              const double* ur = Ub + suo[z] + sidx[z] * R;
  #pragma unroll
              for (int r = 0; r < RMAX; ++r)
                if (r < R) sv[r] *= ur[r];
            }
            double p0[RMAX], p1[RMAX];
  #pragma unroll
            for (int r = 0; r < RMAX; ++r) p0[r] = p1[r] = 0.0;
            const double* t0 = Ts + i0 * stn + toff;
            const double* t1 = Ts + (two ? i1 : i0) * stn + toff;
            const double* uq = Ub + uoq;
  #pragma unroll 4
            for (int k = 0; k < Iq0; ++k) {
              const double a0 = t0[k * stq], a1 = t1[k * stq];
  #pragma unroll
              for (int r = 0; r < RMAX; ++r)
                if (r < R) {
                  const double u = uq[k * R + r];
                  p0[r] = fma(a0, u, p0[r]);
                  p1[r] = fma(a1, u, p1[r]);
                }
            }
  #pragma unroll
            for (int r = 0; r < RMAX; ++r) {
              acc[r][0] = fma(sv[r], p0[r], acc[r][0]);
              acc[r][1] = fma(sv[r], p1[r], acc[r][1]);
            }
  #pragma unroll
            for (int z = 0; z < NM - 2; ++z) {  // next j' (mixed radix, fastest slow mode first)
              toff += sst[z];
              if (++sidx[z] < sdim[z]) break;
              toff -= sst[z] * sdim[z];
              sidx[z] = 0;
            }
          }
  #pragma unroll
          for (int r = 0; r < RMAX; ++r)
            if (r < R) {
              Ms[i0 * R + r] = acc[r][0];
              if (two) Ms[i1 * R + r] = acc[r][1];
            }
        }
      }
      __syncwarp();
      // (a3) Hadamard of the cached Gramians of the other modes; (a4) Cholesky on lane 0
      for (int e = lane; e < R * R; e += 32) {
        double hh = 1.0;
        for (int m = 0; m < N; ++m)
          if (m != n) hh *= Gs[m * R * R + e];  // (N compile-time: unrolled)
        H[e] = hh;
      }
      __syncwarp();
      int pinv = 0;
      if (lane == 0) {
        double L[RMAX][RMAX];
        bool ok = true;
#pragma unroll
        for (int jj = 0; jj < RMAX; ++jj) {
          if (jj < R && ok) {
            double sacc = H[jj * R + jj];
#pragma unroll
            for (int qq = 0; qq < jj; ++qq) sacc -= L[jj][qq] * L[jj][qq];
            if (!(sacc > 0.0) || !isfinite(sacc)) {
              ok = false;
            } else {
              const double dd = sqrt(sacc), id = 1.0 / dd;
              L[jj][jj] = dd;
              Linv[jj] = id;
#pragma unroll
              for (int i = jj + 1; i < RMAX; ++i)
                if (i < R) {
                  double tt = H[i * R + jj];
#pragma unroll
                  for (int qq = 0; qq < jj; ++qq) tt -= L[i][qq] * L[jj][qq];
                  L[i][jj] = tt * id;
                }
            }
          }
        }
        if (ok) {
#pragma unroll
          for (int i = 0; i < RMAX; ++i)
#pragma unroll
            for (int jj = 0; jj <= i; ++jj)
              if (i < R) Lf[i * R + jj] = L[i][jj];
        } else {
          jacobi_pinv<RMAX>(H, R, Lf, 1e-12);
          fl |= F_PINV;
          a.flags[sub] = fl;
        }
        pinv = ok ? 0 : 1;
      }
      pinv = __shfl_sync(0xffffffffu, pinv, 0);
      fl = __shfl_sync(0xffffffffu, fl, 0);
      __syncwarp();
      // (a4/a5) V(i,:) = M(i,:) H^-1 over rows (mode 0: the group's rows [p0, p0 + d) are zero)
      const int64_t z0 = (n == 0) ? pz0 : -1, z1 = (n == 0) ? pz0 + a.d : -1;
      constexpr int NQ = RMAX * (RMAX + 1) / 2;
      double accq[NQ + 1];
#pragma unroll
      for (int z = 0; z <= NQ; ++z) accq[z] = 0.0;
      for (int i = lane; i < In; i += 32) {
        double mv[RMAX], v[RMAX];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) mv[r] = (r < R) ? Ms[i * R + r] : 0.0;
        if (i >= z0 && i < z1) {
#pragma unroll
          for (int r = 0; r < RMAX; ++r) v[r] = 0.0;
        } else if (!pinv) {
          double y[RMAX];
#pragma unroll
          for (int r = 0; r < RMAX; ++r) {
            y[r] = 0.0;
            if (r < R) {
              double tt = mv[r];
#pragma unroll
              for (int qq = 0; qq < r; ++qq) tt -= Lf[r * R + qq] * y[qq];
              y[r] = tt * Linv[r];
            }
          }
#pragma unroll
          for (int r = RMAX - 1; r >= 0; --r) {
            v[r] = 0.0;
            if (r < R) {
              double tt = y[r];
#pragma unroll
              for (int qq = r + 1; qq < RMAX; ++qq)
                if (qq < R) tt -= Lf[qq * R + r] * v[qq];
              v[r] = tt * Linv[r];
            }
          }
        } else {
#pragma unroll
          for (int r = 0; r < RMAX; ++r) {
            double sacc = 0.0;
#pragma unroll
            for (int qq = 0; qq < RMAX; ++qq)
              if (qq < R && r < R) sacc += mv[qq] * Lf[qq * R + r];
            v[r] = sacc;
          }
        }
        int z = 0;
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          if (r < R) Vs[i * R + r] = v[r];
#pragma unroll
          for (int c = r; c < RMAX; ++c, ++z) accq[z] += v[r] * v[c];
        }
#pragma unroll
        for (int r = 0; r < RMAX; ++r) accq[NQ] += v[r] * mv[r];
      }
#pragma unroll
      for (int z = 0; z <= NQ; ++z) accq[z] = res_warp_sum(accq[z]);
      auto vtv = [&](int r, int c) -> double {
        const int lo = r < c ? r : c, hi = r < c ? c : r;
        const int ix = lo * RMAX - lo * (lo - 1) / 2 + (hi - lo);
        double x = 0.0;
#pragma unroll
        for (int z = 0; z < NQ; ++z)
          if (z == ix) x = accq[z];
        return x;
      };
      // (a6) lambda_r = ||V(:,r)||, U = V / lambda (lambda = 0: unchanged); Gram_n = V^T V / (lambda lambda^T)
      double lam[RMAX], il[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        lam[r] = r < R ? sqrt(vtv(r, r)) : 0.0;
        il[r] = lam[r] > 0.0 ? 1.0 / lam[r] : 1.0;
      }
      __syncwarp();
      for (int i = lane; i < In; i += 32) {
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          if (r < R) Ub[uo[n] + i * R + r] = Vs[i * R + r] * il[r];
      }
      if (lane == 0) {
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
#pragma unroll
          for (int c = 0; c < RMAX; ++c)
            if (r < R && c < R) Gs[n * R * R + r * R + c] = vtv(r, c) * il[r] * il[c];
      }
      if (n == last) {  // (a7) error, fit, history, convergence
        if (lane < R) {
#pragma unroll
          for (int r = 0; r < RMAX; ++r)
            if (r == lane) a.lambda[(int64_t)sub * R + r] = lam[r];
        }
        double quad = 0.0;
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
#pragma unroll
          for (int c = 0; c < RMAX; ++c)
            if (r < R && c < R) quad += H[r * R + c] * vtv(r, c);
        const double e = nt2 + quad - 2.0 * accq[NQ];
        ++it;
        bool stay = true;
        if (!isfinite(e)) {
          fl |= F_NONFINITE;
          stay = false;
        } else {
          if (e < -1e-9 * nt2) fl |= F_BREAKDOWN;
          const double fitv = nt2 > 0.0 ? 1.0 - sqrt(fmax(e, 0.0)) / sqrt(nt2) : 0.0;
          if (tol > 0.0 && it >= 2 && fabs(fitv - fp) < tol) {
            fl |= F_CONVERGED;
            stay = false;
          }
          if (lane == 0) {
            a.fit[sub] = fitv;
            a.fit_prev[sub] = fitv;
          }
          fp = fitv;
        }
        if (lane == 0) {
          a.iters[sub] = it;
          a.err[sub] = e;
          a.hist[(int64_t)sub * a.hist_cap + (it - 1) % a.hist_cap] = e;
          a.flags[sub] = fl;
          if (!stay) a.active[sub] = 0;
        }
        act = stay;
      }
      __syncwarp();
    }
  }
  // ---- write back the factor blocks (every mode) and Gramians
  for (int m = 0; m < N; ++m)
    for (int e = lane; e < a.dims[m] * R; e += 32) {
      const int i = e / R, r = e % R;
      a.U[m][(int64_t)i * a.ldu + (int64_t)k * R + r] = Ub[uo[m] + e];
    }
  for (int e = lane; e < N * R * R; e += 32) {
    const int m = e / (R * R), rr = e % (R * R);
    a.gram[((int64_t)m * a.nsub + sub) * R * R + rr] = Gs[e];
  }
  if (lane == 0) atomicMax(a.sweeps_out, sweeps);
}

}  // namespace jk
