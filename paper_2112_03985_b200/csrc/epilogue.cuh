// epilogue.cuh — per-submodel ALS update after the fused MTTKRP of mode n.
//
// One CTA per live submodel block k (sub = blk2sub[k]) does, in this order
// (Alg. 3 lines alg:cals_jk:hadamard .. alg:cals_jk:error):
//   H    = Hadamard over m != n of the cached Gramians Gram_m^(sub)          (a3)
//   M    = fixed-order sum of the split-K / stream-K partial pieces         (a2 reduce)
//   V    = M H^{-1}: Cholesky (thread 0), pinv fallback via Jacobi         (a4)
//   n==0: V(p,:) = 0  (zero row of the left-out sample, alg:cals_jk:multifactor) (a5)
//   lambda_r = ||V(:,r)||_2 ; U = V / lambda (lambda = 0 -> unchanged)       (a6)
//   Gram_n^(sub) = U^T U (cached for the next modes)
//   n==N-1: e = ||T_-p||^2 + sum(H .* V^T V) - 2 sum(V .* M); fit; history;
//           convergence mask (|fit - fit_prev| < tol from sweep 2)          (a7)
// Everything is summed in a fixed order, so results are run-to-run deterministic.
#pragma once
#ifdef JK_EPI_PROF
#include <cstdio>
#endif
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "mttkrp.cuh"

namespace jk {

enum { F_CONVERGED = 1, F_PINV = 2, F_NONFINITE = 4, F_BREAKDOWN = 8 };

struct EpiArgs {
  int N, n, R;                   // R: the handle's largest rank Rs (strides of gram / lambda)
  const int* subR;               // mixed-rank pool: submodel -> rank R_k (nullptr: every block has R)
  const int* blkcol;             // mixed-rank pool: live block -> first column (nullptr: k R)
  int In;
  int64_t ldu;
  int nsub;                      // submodels of the handle (state arrays are indexed by sub)
  double* U;                     // multi-factor of mode n (row-major In x ldu)
  const int* blk2sub;            // live block -> submodel
  const int64_t* pglob;          // submodel -> first global left-out row p0 (group g: p0 = g d)
  int d;                         // delete-d group size: rows [p0, min(p0 + d, I_0)) are padded
  const double* parts;           // partial pieces of the fused MTTKRP
  const TileInfo* tinfo;
  int BM, BN, nMt;
  double* gram;                  // [N][nsub][R][R]
  double* lambda;                // [nsub][R]
  const double* normT2p;         // [nsub]  ||T_-p||^2
  double* fit;                   // [nsub]
  double* fit_prev;              // [nsub]
  double* err;                   // [nsub]
  int* iters;                    // [nsub]
  int* flags;                    // [nsub]
  int* active;                   // [nsub]
  double* hist;                  // [nsub][hist_cap]
  int hist_cap;
  const double* tol;             // device scalar (graph-stable)
  int* active_count;             // incremented at n == N-1 by still-active submodels
};

constexpr int kEpiThreads = 128;
#ifdef JK_TU_HOST

// Pre-reduction of the stream-K partial pieces for tiles split over many CTAs (a small-C shard
// fills the GPU with up to 64 CTAs per tile; one epilogue CTA per submodel would otherwise sum
// them alone). One CTA per 32 consecutive elements of a tile (tile_elems = BN x BM is a multiple
// of 128): warp w sums the w-th contiguous eighth of the piece range with all of its loads in
// flight (coalesced 256 B rows), then warp 0 adds the eight partials in warp order. The order is
// fixed, so results are deterministic; a one-thread-per-element loop was latency-bound (r02: a
// syn200 shard at G = 8, 59 pieces per tile: 13.5 us per mode). The epilogue then reads one piece
// per tile.
constexpr int kRedWarps = 8;
__global__ void __launch_bounds__(32 * kRedWarps) reduce_pieces_kernel(const double* __restrict__ parts,
                                                                       const TileInfo* __restrict__ tinfo, int ntiles,
                                                                       int tile_elems, double* __restrict__ red) {
  __shared__ double part[kRedWarps][32];
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the MTTKRP grid has completed
  asm volatile("griddepcontrol.launch_dependents;\n" :::);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  const int t = (int)((int64_t)blockIdx.x * 32 / tile_elems);
  const TileInfo ti = tinfo[t];
  const int64_t o = e - (int64_t)t * tile_elems;
  const double* p = parts + (int64_t)ti.piece_base * tile_elems + o;
  const int lo = (int)((int64_t)ti.npieces * w / kRedWarps), hi = (int)((int64_t)ti.npieces * (w + 1) / kRedWarps);
  double s = 0.0;
  int pc = lo;
  for (; pc + 8 <= hi; pc += 8) {
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = __ldcg(p + (int64_t)(pc + q) * tile_elems);
#pragma unroll
    for (int q = 0; q < 8; ++q) s += x[q];
  }
  {
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = (pc + q < hi) ? __ldcg(p + (int64_t)(pc + q) * tile_elems) : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (pc + q < hi) s += x[q];
  }
  part[w][lane] = s;
  __syncthreads();
  if (w == 0) {
    double r = part[0][lane];
#pragma unroll
    for (int q = 1; q < kRedWarps; ++q) r += part[q][lane];
    red[e] = r;
  }
  (void)ntiles;
}
#endif

template <int RMAX>
__device__ __forceinline__ void block_sum(double* vals, int cnt, double* red) {
  // vals: per-thread array of cnt (<= RMAX*RMAX + RMAX + 1) values -> summed into red[0..cnt)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = kEpiThreads / 32;
  for (int q = 0; q < cnt; ++q) {
    double x = vals[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp * cnt + q] = x;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w * cnt + q];
    red[NW * cnt + q] = s;
  }
  __syncthreads();
}

// Symmetric pseudoinverse by cyclic Jacobi (single thread, R <= RMAX).
template <int RMAX>
__device__ __noinline__ void jacobi_pinv(const double* H, int R, double* Hp, double rcond) {
  double A[RMAX * RMAX], Q[RMAX * RMAX];
  for (int e = 0; e < R * R; ++e) { A[e] = H[e]; Q[e] = 0.0; }
  for (int i = 0; i < R; ++i) Q[i * R + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < R; ++j) {
        double a = A[i * R + j];
        tot += a * a;
        if (i != j) off += a * a;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < R - 1; ++p)
      for (int q = p + 1; q < R; ++q) {
        double apq = A[p * R + q];
        if (apq == 0.0) continue;
        double theta = (A[q * R + q] - A[p * R + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < R; ++k) {
          double akp = A[k * R + p], akq = A[k * R + q];
          A[k * R + p] = c * akp - s * akq;
          A[k * R + q] = s * akp + c * akq;
        }
        for (int k = 0; k < R; ++k) {
          double apk = A[p * R + k], aqk = A[q * R + k];
          A[p * R + k] = c * apk - s * aqk;
          A[q * R + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < R; ++k) {
          double qkp = Q[k * R + p], qkq = Q[k * R + q];
          Q[k * R + p] = c * qkp - s * qkq;
          Q[k * R + q] = s * qkp + c * qkq;
        }
      }
  }
  double wmax = 0.0;
  for (int i = 0; i < R; ++i) wmax = fmax(wmax, A[i * R + i]);
  for (int e = 0; e < R * R; ++e) Hp[e] = 0.0;
  for (int i = 0; i < R; ++i) {
    double w = A[i * R + i];
    if (!(w > rcond * wmax) || w <= 0.0) continue;
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b) Hp[a * R + b] += Q[a * R + i] * Q[b * R + i] / w;
  }
}

template <int RMAX>
__global__ void __launch_bounds__(kEpiThreads) als_epilogue_rows_kernel(EpiArgs a) {
  const int k = blockIdx.x;
  asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the MTTKRP grid has completed
  asm volatile("griddepcontrol.launch_dependents;\n" :::);
  if (a.n == 0 && k == 0 && threadIdx.x == 0) *a.active_count = 0;  // per-sweep counter reset
  const int sub = a.blk2sub[k];
  if (!a.active[sub]) return;  // frozen (converged or failed)
  const int R = a.subR ? a.subR[sub] : a.R, Rs = a.R, n = a.n, N = a.N, tid = threadIdx.x;
  const bool last = (n == N - 1);
  const int64_t pz0 = (n == 0) ? a.pglob[sub] : -1;   // padded rows [pz0, pz1)
  const int64_t pz1 = (n == 0) ? pz0 + a.d : -1;
  const int cb = a.blkcol ? a.blkcol[k] : k * R;

  __shared__ double H[RMAX * RMAX];
  __shared__ double Lf[RMAX * RMAX];       // Cholesky factor (row-major lower) or H^+
  __shared__ int use_pinv;
  __shared__ double red[(kEpiThreads / 32 + 1) * (RMAX * RMAX + RMAX + 1)];

  // (a3) Hadamard of the cached Gramians of every other mode
  for (int e = tid; e < R * R; e += kEpiThreads) {
    double h = 1.0;
    for (int m = 0; m < N; ++m)
      if (m != n) h *= a.gram[((int64_t)m * a.nsub + sub) * Rs * Rs + e];
    H[e] = h;
  }
  __syncthreads();
  // (a4) Cholesky H = L L^T (textbook, no pivoting); pinv fallback
  if (tid == 0) {
    bool ok = true;
    for (int j = 0; j < R && ok; ++j) {
      double s = H[j * R + j];
      for (int q = 0; q < j; ++q) s -= Lf[j * R + q] * Lf[j * R + q];
      if (!(s > 0.0) || !isfinite(s)) { ok = false; break; }
      Lf[j * R + j] = sqrt(s);
      for (int i = j + 1; i < R; ++i) {
        double t = H[i * R + j];
        for (int q = 0; q < j; ++q) t -= Lf[i * R + q] * Lf[j * R + q];
        Lf[i * R + j] = t / Lf[j * R + j];
      }
    }
    use_pinv = ok ? 0 : 1;
    if (!ok) {
      jacobi_pinv<RMAX>(H, R, Lf, 1e-12);
      a.flags[sub] |= F_PINV;
    }
  }
  __syncthreads();
  const bool pinv = use_pinv != 0;

  // pass 1: reduce partials, solve, write V; accumulate column norms (and V^T V, V.M)
  double cn[RMAX], vtv[RMAX * RMAX], cross = 0.0;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) cn[r] = 0.0;
#pragma unroll
  for (int e = 0; e < RMAX * RMAX; ++e) vtv[e] = 0.0;

  for (int i = tid; i < a.In; i += kEpiThreads) {
    double m[RMAX], v[RMAX];
    const int tn = i / a.BN;
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      m[r] = 0.0;
      if (r < R) {
        const int c = cb + r, tm = c / a.BM;
        const TileInfo ti = a.tinfo[tn * a.nMt + tm];
        const double* p = a.parts + (int64_t)ti.piece_base * a.BN * a.BM + (int64_t)(i - tn * a.BN) * a.BM + (c - tm * a.BM);
        double s = 0.0;
        for (int pc = 0; pc < ti.npieces; ++pc) s += p[(int64_t)pc * a.BN * a.BM];
        m[r] = s;
      }
    }
    if (i >= pz0 && i < pz1) {
#pragma unroll
      for (int r = 0; r < RMAX; ++r) v[r] = 0.0;
    } else if (!pinv) {
      double y[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        if (r < R) {
          double t = m[r];
#pragma unroll
          for (int q = 0; q < r; ++q) t -= Lf[r * R + q] * y[q];
          y[r] = t / Lf[r * R + r];
        }
      }
#pragma unroll
      for (int r = RMAX - 1; r >= 0; --r) {
        if (r < R) {
          double t = y[r];
#pragma unroll
          for (int q = r + 1; q < RMAX; ++q)
            if (q < R) t -= Lf[q * R + r] * v[q];
          v[r] = t / Lf[r * R + r];
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        if (r < R) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < RMAX; ++q)
            if (q < R) s += m[q] * Lf[q * R + r];
          v[r] = s;
        }
      }
    }
    double* urow = a.U + (int64_t)i * a.ldu + cb;
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (r < R) {
        urow[r] = v[r];
        cn[r] += v[r] * v[r];
        if (last) {
          cross += v[r] * m[r];
#pragma unroll
          for (int q = 0; q < RMAX; ++q)
            if (q < R) vtv[r * RMAX + q] += v[r] * v[q];
        }
      }
    }
  }
  // block reductions (fixed order)
  double vals[RMAX * RMAX + RMAX + 1];
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) vals[cnt++] = cn[r];
  vals[cnt++] = cross;
  if (last) {
#pragma unroll
    for (int e = 0; e < RMAX * RMAX; ++e) vals[cnt++] = vtv[e];
  }
  block_sum<RMAX>(vals, cnt, red);
  constexpr int NW = kEpiThreads / 32;
  const double* tot = red + NW * cnt;
  double lam[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) lam[r] = (r < R) ? sqrt(tot[r]) : 0.0;
  double quad = 0.0, crs = tot[RMAX];
  if (last) {
    for (int r = 0; r < R; ++r)
      for (int q = 0; q < R; ++q) quad += H[r * R + q] * tot[RMAX + 1 + r * RMAX + q];
  }
  __syncthreads();  // everyone has read `red` before it is reused

  // pass 2: normalise (a6) and accumulate the Gramian of the normalised block
  double gr[RMAX * RMAX];
#pragma unroll
  for (int e = 0; e < RMAX * RMAX; ++e) gr[e] = 0.0;
  for (int i = tid; i < a.In; i += kEpiThreads) {
    double* urow = a.U + (int64_t)i * a.ldu + cb;
    double uu[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      uu[r] = 0.0;
      if (r < R) {
        double x = urow[r];
        uu[r] = lam[r] > 0.0 ? x / lam[r] : x;
        urow[r] = uu[r];
      }
    }
#pragma unroll
    for (int r = 0; r < RMAX; ++r)
#pragma unroll
      for (int q = 0; q < RMAX; ++q)
        if (r < R && q < R) gr[r * RMAX + q] += uu[r] * uu[q];
  }
  block_sum<RMAX>(gr, RMAX * RMAX, red);
  const double* gt = red + NW * RMAX * RMAX;
  for (int e = tid; e < R * R; e += kEpiThreads) {
    int r = e / R, q = e % R;
    a.gram[((int64_t)n * a.nsub + sub) * Rs * Rs + e] = gt[r * RMAX + q];
  }
  if (tid < R) a.lambda[(int64_t)sub * Rs + tid] = lam[tid];

  if (last && tid == 0) {  // (a7) error, fit, history, convergence mask
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

// Fast path (I_n * R small enough for shared memory): the same arithmetic as the row kernel
// above -- identical per-row solve and fixed-order sums -- but with M and V staged in shared
// memory so that the partial reduction, the solves and every reduction run with all threads.
constexpr int kEpi2Threads = 256;

#ifdef JK_EPI_PROF
#define EPI_PROBE(i)                                                                              \
  do {                                                                                            \
    if (threadIdx.x == 0) {                                                                       \
      unsigned long long t_;                                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                      \
      epi_ts_[(i)] = t_;                                                                          \
    }                                                                                             \
  } while (0)
#define EPI_PROBE_DUMP()                                                                          \
  do {                                                                                            \
    if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))                     \
      printf("EPI blk %d n %d: %llu %llu %llu %llu %llu %llu %llu chol %llu\n", blockIdx.x,       \
             a.n, epi_ts_[1] - epi_ts_[0], epi_ts_[2] - epi_ts_[0], epi_ts_[3] - epi_ts_[0],       \
             epi_ts_[4] - epi_ts_[0], epi_ts_[5] - epi_ts_[0], epi_ts_[6] - epi_ts_[0],            \
             epi_ts_[7] - epi_ts_[0], epi_ts_[8] - epi_ts_[0]);                                    \
  } while (0)
#else
#define EPI_PROBE(i) do {} while (0)
#define EPI_PROBE_DUMP() do {} while (0)
#endif


__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  return x;
}


template <int J, int Q>
__device__ __forceinline__ void sum_pieces(const EpiArgs& a, int cb, int R, int In, double* Ms, int ldm) {
  const int64_t piece = (int64_t)a.BN * a.BM;
  const int T = blockDim.x;
  for (int e0 = threadIdx.x; e0 < In * R; e0 += J * T) {
    const double* p[J];
    int np[J];
    double s[J];
    int npmax = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int e = e0 + j * T;
      s[j] = 0.0;
      np[j] = 0;
      p[j] = a.parts;
      if (e < In * R) {
        const int i = e / R, r = e % R;
        const int c = cb + r, tn = i / a.BN, tm = c / a.BM;
        const TileInfo ti = a.tinfo[tn * a.nMt + tm];
        p[j] = a.parts + (int64_t)ti.piece_base * piece + (int64_t)(i - tn * a.BN) * a.BM + (c - tm * a.BM);
        np[j] = ti.npieces;
        npmax = max(npmax, ti.npieces);
      }
    }
    for (int pc = 0; pc < npmax; pc += Q) {
      double x[J][Q];
#pragma unroll
      for (int j = 0; j < J; ++j)
#pragma unroll
        for (int q = 0; q < Q; ++q) x[j][q] = (pc + q < np[j]) ? __ldcg(p[j] + (int64_t)(pc + q) * piece) : 0.0;
#pragma unroll
      for (int j = 0; j < J; ++j)
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (pc + q < np[j]) s[j] += x[j][q];
    }
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (e0 + j * T < In * R) Ms[((e0 + j * T) / R) * ldm + (e0 + j * T) % R] = s[j];
  }
}

// q-th quantity over rows: Q_q = sum_i f_q(i), one warp per quantity, fixed order
// (lane-strided partial sums, then the shuffle tree).
template <class F>
__device__ __forceinline__ void warp_reduce_all(int nq, int In, double* out, F f) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int q = warp; q < nq; q += nw) {
    double s = 0.0;
    for (int i = lane; i < In; i += 32) s += f(q, i);
    s = warp_sum(s);
    if (lane == 0) out[q] = s;
  }
}

// Body of the fast epilogue for one live block k (submodel `sub`, rank R <= RMAX).
template <int RMAX>
__device__ __forceinline__ void epi_smem_body(const EpiArgs& a, const int k, const int sub, const int R) {
  constexpr int NQ = RMAX * (RMAX + 1) / 2;  // upper triangle of V^T V
#ifdef JK_EPI_PROF
  __shared__ unsigned long long epi_ts_[16];
#endif
  EPI_PROBE(0);  // (stamps are relative to the body's start, after griddepcontrol.wait)
  EPI_PROBE(1);
  const int Rs = a.R, n = a.n, N = a.N, tid = threadIdx.x, In = a.In;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kEpi2Threads / 32;
  const bool last = (n == N - 1);
  const int64_t pz0 = (n == 0) ? a.pglob[sub] : -1;   // padded rows [pz0, pz1)
  const int64_t pz1 = (n == 0) ? pz0 + a.d : -1;
  const int cb = a.blkcol ? a.blkcol[k] : k * R;

  __shared__ double H[RMAX * RMAX];
  __shared__ double Lf[RMAX * RMAX];   // Cholesky factor (row-major lower) or H^+
  __shared__ double Linv[RMAX];        // 1 / L(j,j)
  __shared__ double red[NW][NQ + 1];
  __shared__ double tot[NQ + 1];
  __shared__ double ilam_s[RMAX];
  __shared__ int use_pinv;
  extern __shared__ double dyn[];
  double* Ms = dyn;             // [In][ldm]
  // rows padded to an odd stride: the thread-per-row solve then reads / writes distinct banks
  // (an even R such as the 4-way config's 4 would otherwise conflict R-ways)
  const int ldm = R | 1;
  double* Vs = dyn + In * ldm;  // [In][ldm]

  // (a3) Hadamard of the cached Gramians of every other mode. H depends only on the other modes'
  // Gramians, written by earlier epilogues that completed before this grid was launched, so it
  // and its Cholesky factor are formed BEFORE waiting for the MTTKRP grid (programmatic
  // dependent launch: this prologue overlaps the MTTKRP's tail; L2 loads, not L1)
  if (tid < R * R) {
    double h = 1.0;
    for (int m = 0; m < N; ++m)
      if (m != n) h *= __ldcg(a.gram + ((int64_t)m * a.nsub + sub) * Rs * Rs + tid);
    H[tid] = h;
  }
  __syncthreads();
  EPI_PROBE(2);
  // (a4) Cholesky H = L L^T (textbook, no pivoting) in registers of thread 0; pinv fallback
  if (tid == 0) {
    double L[RMAX][RMAX];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < RMAX; ++j) {
      if (j < R && ok) {
        double s = H[j * R + j];
#pragma unroll
        for (int q = 0; q < j; ++q) s -= L[j][q] * L[j][q];
        if (!(s > 0.0) || !isfinite(s)) {
          ok = false;
        } else {
          const double d = sqrt(s), id = 1.0 / d;
          L[j][j] = d;
          Linv[j] = id;
#pragma unroll
          for (int i = j + 1; i < RMAX; ++i) {
            if (i < R) {
              double t = H[i * R + j];
#pragma unroll
              for (int q = 0; q < j; ++q) t -= L[i][q] * L[j][q];
              L[i][j] = t * id;
            }
          }
        }
      }
    }
    use_pinv = ok ? 0 : 1;
    if (ok) {
#pragma unroll
      for (int i = 0; i < RMAX; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j)
          if (i < R) Lf[i * R + j] = L[i][j];
    } else {
      jacobi_pinv<RMAX>(H, R, Lf, 1e-12);
      a.flags[sub] |= F_PINV;
    }
  }
  EPI_PROBE(8);  // (after thread 0's Cholesky: barrier-free, so other threads pass earlier)
  // (a7) the stop test's per-submodel scalars, requested before the wait (their last writers are
  // >= 2 grids back, like the Gramians above) so thread 0's final step is not a chain of L2 loads
  double pf_nt2 = 0.0, pf_fitp = 0.0, pf_tol = 0.0;
  int pf_it = 0, pf_fl = 0;
  if (last && tid == 0) {
    pf_nt2 = a.normT2p[sub];
    pf_fitp = a.fit_prev[sub];
    pf_tol = *a.tol;
    pf_it = a.iters[sub];
    pf_fl = a.flags[sub];  // (after this thread's own F_PINV update above)
  }
  // the MTTKRP of this mode has completed: its reduced tiles are visible from here on
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" :::);
  if (n == 0 && k == 0 && tid == 0) *a.active_count = 0;  // per-sweep counter reset
  // (a2) fixed-order sum of the partial pieces of this submodel's R columns (one reduced piece per
  // tile on the FP64 path): J elements per thread x Q pieces = 16 independent loads in flight
  if (In * R <= kEpi2Threads) sum_pieces<1, 16>(a, cb, R, In, Ms, ldm);
  else sum_pieces<4, 4>(a, cb, R, In, Ms, ldm);
  __syncthreads();
  EPI_PROBE(3);
  const bool pinv = use_pinv != 0;
  // (a4/a5) per-row solve V(i,:) = M(i,:) H^{-1} (the left-out row p of mode 0 is zero) and,
  // in the same pass, this thread's share of V^T V (upper triangle) and of V.M
  double acc[NQ + 1];
#pragma unroll
  for (int q = 0; q <= NQ; ++q) acc[q] = 0.0;
  for (int i = tid; i < In; i += blockDim.x) {
    double m[RMAX], v[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) m[r] = (r < R) ? Ms[i * ldm + r] : 0.0;
    if (i >= pz0 && i < pz1) {
#pragma unroll
      for (int r = 0; r < RMAX; ++r) v[r] = 0.0;
    } else if (!pinv) {
      double y[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        y[r] = 0.0;
        if (r < R) {
          double t = m[r];
#pragma unroll
          for (int q = 0; q < r; ++q) t -= Lf[r * R + q] * y[q];
          y[r] = t * Linv[r];
        }
      }
#pragma unroll
      for (int r = RMAX - 1; r >= 0; --r) {
        v[r] = 0.0;
        if (r < R) {
          double t = y[r];
#pragma unroll
          for (int q = r + 1; q < RMAX; ++q)
            if (q < R) t -= Lf[q * R + r] * v[q];
          v[r] = t * Linv[r];
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < RMAX; ++q)
          if (q < R && r < R) s += m[q] * Lf[q * R + r];
        v[r] = s;
      }
    }
    int q = 0;
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (r < R) Vs[i * ldm + r] = v[r];
#pragma unroll
      for (int c = r; c < RMAX; ++c, ++q) acc[q] += v[r] * v[c];
    }
#pragma unroll
    for (int r = 0; r < RMAX; ++r) acc[NQ] += v[r] * m[r];
  }
  // block reduction of the NQ+1 quantities in a fixed order (shuffle tree, then warps in order)
#pragma unroll
  for (int q = 0; q <= NQ; ++q) {
    const double x = warp_sum(acc[q]);
    if (lane == 0) red[warp][q] = x;
  }
  __syncthreads();
  EPI_PROBE(4);
  for (int q = tid; q <= NQ; q += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w][q];
    tot[q] = s;
  }
  __syncthreads();
  EPI_PROBE(5);
  // (a6) lambda_r = ||V(:,r)||, U = V / lambda; Gram of U = (V^T V) / (lambda lambda^T)
  auto vtv = [&](int r, int c) -> double {  // index into the packed upper triangle
    const int lo = r < c ? r : c, hi = r < c ? c : r;
    return tot[lo * RMAX - lo * (lo - 1) / 2 + (hi - lo)];
  };
  if (tid < R) {
    const double lm = sqrt(vtv(tid, tid));
    ilam_s[tid] = lm > 0.0 ? 1.0 / lm : 1.0;
    a.lambda[(int64_t)sub * Rs + tid] = lm;
  }
  __syncthreads();
  for (int e = tid; e < In * R; e += blockDim.x) {
    const int i = e / R, r = e % R;
    a.U[(int64_t)i * a.ldu + cb + r] = Vs[i * ldm + r] * ilam_s[r];
  }
  if (tid < R * R) {
    const int r = tid / R, c = tid % R;
    a.gram[((int64_t)n * a.nsub + sub) * Rs * Rs + tid] = vtv(r, c) * ilam_s[r] * ilam_s[c];
  }
  EPI_PROBE(6);
  if (last && tid == 0) {  // (a7) error, fit, history, convergence mask
    double quad = 0.0;
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < R; ++c) quad += H[r * R + c] * vtv(r, c);
    const double crs = tot[NQ];
    const double nt2 = pf_nt2;
    const double e = nt2 + quad - 2.0 * crs;
    int it = pf_it + 1;
    a.iters[sub] = it;
    a.err[sub] = e;
    a.hist[(int64_t)sub * a.hist_cap + (it - 1) % a.hist_cap] = e;
    int f = pf_fl;
    bool act = true;
    if (!isfinite(e)) {
      f |= F_NONFINITE;
      act = false;
    } else {
      if (e < -1e-9 * nt2) f |= F_BREAKDOWN;
      const double fit = nt2 > 0.0 ? 1.0 - sqrt(fmax(e, 0.0)) / sqrt(nt2) : 0.0;
      const double tol = pf_tol;
      if (tol > 0.0 && it >= 2 && fabs(fit - pf_fitp) < tol) {
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
  EPI_PROBE(7);
  EPI_PROBE_DUMP();
}

// frozen block (converged or failed): nothing to update, but block 0 still resets the per-sweep
// active counter at mode 0 (after the previous grid, which may still read it, has completed)
__device__ __forceinline__ void epi_frozen(const EpiArgs& a, int k) {
  if (a.n == 0 && k == 0 && threadIdx.x == 0) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    *a.active_count = 0;
  }
}

template <int RMAX>
__global__ void __launch_bounds__(kEpi2Threads) als_epilogue_kernel(EpiArgs a) {
  const int k = blockIdx.x;
  // (block table and masks are only changed by the host between sweeps: safe before the wait)
  const int sub = a.blk2sub[k];
  if (!a.active[sub]) return epi_frozen(a, k);
  epi_smem_body<RMAX>(a, k, sub, a.subR ? a.subR[sub] : a.R);  // waits for the MTTKRP inside
}

// Mixed-rank pool: one launch for every block; each block runs the body instantiated for the
// smallest rank class that holds its own rank (so an R = 3 block does not pay for R = 9).
// RMAXC, the class of the pool's largest rank, bounds the branches compiled in (and so the
// kernel's register count: classes <= 8 keep two 256-thread CTAs per SM).
template <int RMAXC>
__global__ void __launch_bounds__(kEpi2Threads) als_epilogue_mixed_kernel(EpiArgs a) {
  const int k = blockIdx.x;
  const int sub = a.blk2sub[k];
  if (!a.active[sub]) return epi_frozen(a, k);
  const int R = a.subR[sub];
  if (R <= 2) epi_smem_body<2>(a, k, sub, R);
  else if (RMAXC >= 4 && R <= 4) epi_smem_body<(RMAXC >= 4 ? 4 : 2)>(a, k, sub, R);
  else if (RMAXC >= 6 && R <= 6) epi_smem_body<(RMAXC >= 6 ? 6 : 2)>(a, k, sub, R);
  else if (RMAXC >= 8 && R <= 8) epi_smem_body<(RMAXC >= 8 ? 8 : 2)>(a, k, sub, R);
  else if (RMAXC >= 10 && R <= 10) epi_smem_body<(RMAXC >= 10 ? 10 : 2)>(a, k, sub, R);
  else if (RMAXC >= 12 && R <= 12) epi_smem_body<(RMAXC >= 12 ? 12 : 2)>(a, k, sub, R);
  else if (RMAXC >= 16) epi_smem_body<(RMAXC >= 16 ? 16 : 2)>(a, k, sub, R);
}

}  // namespace jk
