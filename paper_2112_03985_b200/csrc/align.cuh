// Submodel alignment and aligned jackknife statistics.
//
// Alg. 2 line alg:jk:perm_scale adjusts every fitted submodel P_hat_{-p} for the
// CP permutation / sign / scale indeterminacy before the standard deviations of alg:jk:std
// (PAPER.md:339). The paper defers the scheme to its citation; reading A12 fixes it:
//   cos_n(r,s) = <U_n(:,r), P_n(:,s)> / (||U_n(:,r)|| ||P_n(:,s)||)  (0 if a norm is 0), n >= 1
//   C(r,s) = prod_{n>=1} |cos_n(r,s)|;  sigma = argmax_perm sum_r C(r, sigma(r)), the lowest
//   lexicographic rank among equal maxima;  sign_n(r) = sign of cos_n(r, sigma(r)) (n >= 1),
//   sign_0(r) = prod_{n>=1} sign_n(r);  aligned column sigma(r): unit-norm signed U_n(:,r)
//   (n >= 1), and sign_0 lambda_r prod_{n>=1} ||U_n(:,r)|| U_0(:,r) in mode 0.
// One CTA per submodel: warp-per-quantity dot products (fixed order), the exhaustive
// assignment split over the CTA's threads by lexicographic rank ranges (R <= 10), then the
// aligned factors are written to the aligned store (row-major I_n x R per mode).
#pragma once
#include <cstdint>

namespace jk {

constexpr int kAlignThreads = 256;
constexpr int kAlignRMax = 10;

struct AlignArgs {
  const double* base;        // workspace base (source offsets are relative to it)
  const int64_t* asrc;       // [nsub][N] offset (doubles) of submodel q's mode-n block
  const int64_t* asld;       // [nsub][N] its row stride
  const double* lambda;      // [nsub][Rs]
  const int* subR;           // [nsub]
  const int* subRc;          // [nsub] first column of its model in the reference store
  const double* pref[8];     // reference (warm start) of mode n: col-major I_n x sumRm
  int64_t dims[8];
  int N, Rs;
  int64_t sumI;              // aligned-store slot stride / Rs
  double* aln;               // aligned store: slot q at q * sumI * Rs
  int* perm;                 // [nsub][Rs]
  int* sign;                 // [nsub][N][Rs]
  double* cong;              // [nsub][Rs]
};

__device__ __forceinline__ double align_warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ void unrank_perm(int64_t rank, int R, int* a) {
  // lexicographic permutation of 0..R-1 with the given rank (factorial number system)
  int64_t fact[kAlignRMax + 1];
  fact[0] = 1;
  for (int i = 1; i <= R; ++i) fact[i] = fact[i - 1] * i;
  int pool[kAlignRMax];
  for (int i = 0; i < R; ++i) pool[i] = i;
  for (int i = 0; i < R; ++i) {
    const int64_t f = fact[R - 1 - i];
    const int d = (int)(rank / f);
    rank %= f;
    a[i] = pool[d];
    for (int j = d; j < R - 1 - i; ++j) pool[j] = pool[j + 1];
  }
}

__device__ __forceinline__ bool next_perm_dev(int* a, int n) {
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) return false;
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  int t = a[i]; a[i] = a[j]; a[j] = t;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) { t = a[l]; a[l] = a[r]; a[r] = t; }
  return true;
}

__global__ void __launch_bounds__(kAlignThreads) align_kernel(AlignArgs a) {
  const int q = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kAlignThreads / 32;
  const int R = a.subR[q], N = a.N;
  __shared__ double cosv[8][kAlignRMax * kAlignRMax];
  __shared__ double nu[8][kAlignRMax], np_[8][kAlignRMax];
  __shared__ double C[kAlignRMax * kAlignRMax];
  __shared__ double bestv[kAlignThreads];
  __shared__ long long bestr[kAlignThreads];
  __shared__ int inv[kAlignRMax], sgn[8][kAlignRMax];
  __shared__ double scale0[kAlignRMax];

  // cosines of every (submodel component r, reference component s) pair, modes n >= 1:
  // quantities 0..R*R-1 are dots, then R norms of U, then R norms of P; one warp per quantity
  for (int n = 1; n < N; ++n) {
    const int64_t I = a.dims[n];
    const double* U = a.base + a.asrc[(int64_t)q * N + n];
    const int64_t ld = a.asld[(int64_t)q * N + n];
    const double* P = a.pref[n] + I * a.subRc[q];
    for (int t = warp; t < R * R + 2 * R; t += NW) {
      double s = 0.0;
      if (t < R * R) {
        const int r = t / R, c = t % R;
        for (int64_t i = lane; i < I; i += 32) s += U[i * ld + r] * P[i + I * c];
      } else if (t < R * R + R) {
        const int r = t - R * R;
        for (int64_t i = lane; i < I; i += 32) s += U[i * ld + r] * U[i * ld + r];
      } else {
        const int c = t - R * R - R;
        for (int64_t i = lane; i < I; i += 32) s += P[i + I * c] * P[i + I * c];
      }
      s = align_warp_sum(s);
      if (lane == 0) {
        if (t < R * R) cosv[n][t] = s;
        else if (t < R * R + R) nu[n][t - R * R] = sqrt(s);
        else np_[n][t - R * R - R] = sqrt(s);
      }
    }
  }
  __syncthreads();
  for (int t = tid; t < R * R; t += kAlignThreads) {
    const int r = t / R, c = t % R;
    double cc = 1.0;
    for (int n = 1; n < N; ++n) {
      const double den = nu[n][r] * np_[n][c];
      const double cs = den > 0.0 ? cosv[n][t] / den : 0.0;
      cosv[n][t] = cs;
      cc *= fabs(cs);
    }
    C[t] = cc;
  }
  __syncthreads();
  // exhaustive assignment: thread t scans lexicographic ranks [t*chunk, (t+1)*chunk)
  int64_t total = 1;
  for (int i = 2; i <= R; ++i) total *= i;
  const int64_t chunk = (total + kAlignThreads - 1) / kAlignThreads;
  int64_t r0 = (int64_t)tid * chunk;
  double bv = -1.0;
  long long br = -1;
  if (r0 < total) {
    int p[kAlignRMax];
    unrank_perm(r0, R, p);
    const int64_t r1 = (r0 + chunk < total) ? r0 + chunk : total;
    for (int64_t rk = r0; rk < r1; ++rk) {
      double v = 0.0;
      for (int r = 0; r < R; ++r) v += C[r * R + p[r]];
      if (v > bv) { bv = v; br = rk; }
      next_perm_dev(p, R);
    }
  }
  bestv[tid] = bv;
  bestr[tid] = br;
  __syncthreads();
  if (tid == 0) {
    double v = -1.0;
    long long rk = 0;
    for (int t = 0; t < kAlignThreads; ++t)   // ranges are in rank order: first strict max wins
      if (bestr[t] >= 0 && bestv[t] > v) { v = bestv[t]; rk = bestr[t]; }
    int p[kAlignRMax];
    unrank_perm(rk, R, p);
    for (int r = 0; r < R; ++r) {
      inv[p[r]] = r;
      int s0 = 1;
      double sc = a.lambda[(int64_t)q * a.Rs + r];
      for (int n = 1; n < N; ++n) {
        const int sg = cosv[n][r * R + p[r]] < 0.0 ? -1 : 1;
        sgn[n][r] = sg;
        s0 *= sg;
        sc *= nu[n][r];
      }
      sgn[0][r] = s0;
      scale0[r] = s0 * sc;
      a.perm[(int64_t)q * a.Rs + r] = p[r];
      a.cong[(int64_t)q * a.Rs + p[r]] = C[r * R + p[r]];
      for (int n = 0; n < N; ++n) a.sign[((int64_t)q * N + n) * a.Rs + r] = sgn[n][r];
    }
  }
  __syncthreads();
  // aligned factors: slot q, mode n at offset sum_{m<n} I_m R (row-major I_n x R)
  double* out = a.aln + (int64_t)q * a.sumI * a.Rs;
  for (int n = 0; n < N; ++n) {
    const int64_t I = a.dims[n];
    const double* U = a.base + a.asrc[(int64_t)q * N + n];
    const int64_t ld = a.asld[(int64_t)q * N + n];
    for (int64_t e = tid; e < I * R; e += kAlignThreads) {
      const int64_t i = e / R;
      const int s = (int)(e % R), r = inv[s];
      const double x = U[i * ld + r];
      double y;
      if (n == 0) y = scale0[r] * x;
      else y = nu[n][r] > 0.0 ? sgn[n][r] * x / nu[n][r] : x;
      out[e] = y;
    }
    out += I * R;
  }
}

// Per-element moments of the listed submodels' aligned blocks; for the sampled mode (present
// != 0) an element (i, r) only counts the submodels whose left-out group does not contain row i
// (reading A20). Outputs column-major I x R: count, mean, M2 = sum (x - mean)^2.
__global__ void moments_present_kernel(const double* __restrict__ base, const int64_t* __restrict__ src_off,
                                       const int64_t* __restrict__ src_ld, const int64_t* __restrict__ pg,
                                       int present, int d, int nsub, int I, int R, double* __restrict__ cnt,
                                       double* __restrict__ mean, double* __restrict__ m2) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= I * R) return;
  const int r = e / I, i = e % I;
  double s = 0.0;
  int c = 0;
  for (int q = 0; q < nsub; ++q) {
    if (present && i >= pg[q] && i < pg[q] + d) continue;
    s += base[src_off[q] + (int64_t)i * src_ld[q] + r];
    ++c;
  }
  const double mu = c > 0 ? s / (double)c : 0.0;
  double ss = 0.0;
  for (int q = 0; q < nsub; ++q) {
    if (present && i >= pg[q] && i < pg[q] + d) continue;
    const double t = base[src_off[q] + (int64_t)i * src_ld[q] + r] - mu;
    ss += t * t;
  }
  cnt[e] = (double)c;
  mean[e] = mu;
  m2[e] = ss;
}

}  // namespace jk
