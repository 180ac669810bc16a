// resident.cuh — the whole JK-CALS iterate in ONE launch for small tensors, T resident in the
// distributed shared memory of a thread-block cluster.
//
// The standard path launches an MTTKRP and an epilogue per mode; for the small configs (tiny
// 10x8x6, syn50 50^3) a sweep is a few microseconds of arithmetic but ~20-50 us of launch and
// grid-dependency latency (r01: 23 us / 43-55 us per sweep; the paper sees the same overhead
// dominate its small tensor). Submodels are independent ALS instances
// (PAPER.md:286-289), so a cluster of `cs` CTAs can own a group of submodels and run every sweep
// of them with no global synchronisation at all:
//   * T is split along its last mode into cs slabs; CTA r keeps slab r in shared memory for the
//     whole launch (row pitches = 4 mod 16 doubles: conflict-free fragment loads).
//   * every CTA keeps a replica of all N factor blocks of the group's fused columns.
//   * mode n: each CTA forms its slab's share of M(i, c) = sum_j T_(n)(i, j) KRP(j, c) for the
//     group's columns (Eq. 1 / Alg. 3 alg:cals_jk:mttkrp) on the FP64 tensor
//     pipe (DMMA m8n8k4: columns on the m side, rows on the n side, k = consecutive i_q0 of one
//     j'), the KRP formed in registers as U_q0(i_q0, c) S_j'(c) and never stored; cluster
//     barrier; the owner CTA of each submodel sums the cs partial blocks in rank order through
//     DSMEM (mode N-1: each CTA owns its slab's rows outright) and runs the ALS update of Alg. 3
//     (alg:cals_jk:hadamard .. alg:cals_jk:error: Hadamard of cached Gramians,
//     Cholesky / pinv solve, zero the left-out rows at mode 0, 2-norm normalisation, Gramian,
//     error / fit / convergence at mode N-1) and stores the new block into every CTA's replica
//     (DSMEM); cluster barrier.
//   * converged submodels are frozen; a cluster whose submodels are all frozen stops (tol > 0:
//     a device-side stop, no host round trip per sweep).
// At exit the owners write factors and Gramians back to the workspace (lambda, fits, flags,
// histories are written as they change), so every other entry point sees the same state as
// after the standard path. Sums run in a fixed order: results are deterministic (not bitwise
// equal to the standard path's, which splits K differently; both are held to the oracle).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "epilogue.cuh"

namespace jk {

namespace cgr = cooperative_groups;

constexpr int kResThreads = 256;
constexpr int kResWarps = kResThreads / 32;
constexpr int kResMaxM = 4;      // m8 column tiles per group (fused columns <= 32)
constexpr int kResMaxNw = 4;     // n8 row tiles per warp and pass
constexpr int kResMaxOwn = 8;    // submodels owned by one CTA
constexpr int kResMaxCp = kResMaxM * 8;

// warps split a mode's n8 row tiles into TG groups and its k-steps into KG = 8 / TG ranges
__host__ __device__ inline int res_tgroups(int rows) {
  const int nN = (rows + 7) / 8;
  int tg = 1;
  while (tg * 2 <= kResWarps && tg * 2 <= nN) tg *= 2;
  return tg;
}
// row pitch of the factor replicas / partial blocks: >= Cp, = 4 mod 8 doubles (k x c fragment loads
// tig * Cpi + gid hit 16 distinct bank pairs)
__host__ __device__ inline int res_cpitch(int Cp) { return ((Cp + 3) / 8) * 8 + 4; }

struct ResArgs {
  int N, R, cs, kpc, Cp, Cpi, slab, d, hist_cap, max_iters, nsub, K;
  int dims[kMaxModes];
  int pitch[kMaxModes];    // shared-memory strides of T (doubles); mode N-1 slab-local
  int64_t gst[kMaxModes];  // workspace strides of T (mode-0 pitch I0p)
  int64_t ldu;
  // dynamic shared memory layout (byte offsets)
  int o_T, o_U[kMaxModes], o_M, o_E, o_G, o_X, o_S;
  const double* T;
  double* U[kMaxModes];
  const int* blk2sub;
  const int64_t* pglob;
  double* gram;            // [N][nsub][R][R]
  double* lambda;          // [nsub][R]
  const double* normT2p;
  double *fit, *fit_prev, *err;
  int *iters, *flags, *active;
  double* hist;
  const double* tol;
  int* sweeps_out;         // max sweeps run by any cluster (atomicMax)
#ifdef JK_RES_PROF
  long long* prof;         // dev builds: clock64 per phase, block 0 thread 0
#endif
};
#ifdef JK_RES_PROF
#define RES_T(i) do { if (blockIdx.x == 0 && threadIdx.x == 0) { long long t_ = clock64(); pacc[i] += t_ - plast; plast = t_; } } while (0)
#else
#define RES_T(i) do {} while (0)
#endif

__device__ __forceinline__ void res_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v) : "memory");
}

// geometry of one mode on one CTA (registers of the caller, passed by value)
struct ResMode {
  int rows, Iq0, pn, pq, Jp, ns;
  int ext[kMaxModes - 2];  // slow modes: extents (slab-local for mode N-1),
  int spt[kMaxModes - 2];  // T strides,
  int sg0[kMaxModes - 2];  // global row of local index 0,
  int suo[kMaxModes - 2];  // replica byte offsets
};

// One pass of a warp: n-tiles [nb, nb + NW) x m-tiles [0, NM) over k4 steps [sb, se) of the flat
// (j', i_q0 / 4) space, into its k-range slice at dst. NM / NW are compile-time so that no MMA is
// predicated off (r02: predicated-off DMMAs still occupied the pipe).
template <int NM, int NW>
static __device__ __forceinline__ void res_pass(const ResMode& md, uint32_t sT, uint32_t sUq, uint32_t sbase,
                                             uint32_t dst, int Cpi, int nb, int sb, int se, int spr) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const int rows = md.rows, Iq0 = md.Iq0, pq = md.pq, ns = md.ns;
  double acc[NM][NW][2];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int q = 0; q < NW; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
  // per n-tile: this lane's (clamped, in-bounds) row offset in T, in bytes
  uint32_t roff[NW];
#pragma unroll
  for (int q = 0; q < NW; ++q) roff[q] = (uint32_t)(min((nb + q) * 8 + gid, rows - 1) * md.pn) * 8u;
  for (int st = sb; st < se;) {
    const int jp = st / spr, k0 = st - jp * spr, k1 = min(spr, k0 + (se - st));
    // j' -> T offset and S_j'(c) for this lane's column c = 8 m + gid of every m-tile
    int toff = 0, rem = jp;
    double sv[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) sv[m] = 1.0;
    for (int z = 0; z < ns; ++z) {
      const int ex = md.ext[z];
      const int dgt = rem % ex;
      rem /= ex;
      toff += dgt * md.spt[z];
      const uint32_t ur = sbase + (uint32_t)md.suo[z] + (uint32_t)((dgt + md.sg0[z]) * Cpi + gid) * 8u;
#pragma unroll
      for (int m = 0; m < NM; ++m) sv[m] *= lds_f64(ur + m * 64u);
    }
    const uint32_t tb = sT + (uint32_t)toff * 8u;
    const int kf = min(k1, Iq0 / 4);  // full k4 steps: no i_q0 padding
    int k = k0;
#pragma unroll 2
    for (; k < kf; ++k) {
      const int iq = k * 4 + tig;
      const uint32_t ua = sUq + (uint32_t)(iq * Cpi + gid) * 8u;
      const uint32_t tq = tb + (uint32_t)(iq * pq) * 8u;
      double av[NM], bv[NW];
#pragma unroll
      for (int m = 0; m < NM; ++m) av[m] = lds_f64(ua + m * 64u) * sv[m];
#pragma unroll
      for (int q = 0; q < NW; ++q) bv[q] = lds_f64(tq + roff[q]);
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int q = 0; q < NW; ++q) dmma_m8n8k4(acc[m][q][0], acc[m][q][1], av[m], bv[q]);
    }
    for (; k < k1; ++k) {  // the ragged last k4 step of the run: A = 0 beyond I_q0
      const int iq = k * 4 + tig;
      const bool ok = iq < Iq0;
      const int iqc = ok ? iq : Iq0 - 1;
      const uint32_t ua = sUq + (uint32_t)(iqc * Cpi + gid) * 8u;
      const uint32_t tq = tb + (uint32_t)(iqc * pq) * 8u;
      double av[NM], bv[NW];
#pragma unroll
      for (int m = 0; m < NM; ++m) av[m] = ok ? lds_f64(ua + m * 64u) * sv[m] : 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) bv[q] = lds_f64(tq + roff[q]);
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int q = 0; q < NW; ++q) dmma_m8n8k4(acc[m][q][0], acc[m][q][1], av[m], bv[q]);
    }
    st += k1 - k0;
  }
  // D[c][i]: this lane holds (c = 8 m + gid, i = 8 n + 2 tig + {0, 1})
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      const int i = (nb + q) * 8 + 2 * tig, c = m * 8 + gid;
      if (i < rows) sts_f64(dst + (uint32_t)(i * Cpi + c) * 8u, acc[m][q][0]);
      if (i + 1 < rows) sts_f64(dst + (uint32_t)((i + 1) * Cpi + c) * 8u, acc[m][q][1]);
    }
}

// This CTA's slab share of M for one mode: warps split the n8 row tiles (TG groups) and the k4
// steps (KG = 8 / TG ranges); partial blocks M_part[kg][i][c] (pitch Cpi) are then summed into
// slice 0 in kg order. sT / sUq / sbase / sMp are 32-bit shared addresses.
static __device__ __forceinline__ void res_mttkrp(const ResMode& md, uint32_t sT, uint32_t sUq, uint32_t sbase,
                                               uint32_t sMp, int Cp, int Cpi) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const int rows = md.rows;
  if (rows <= 0) return;
  const int nM = Cp / 8, nN = (rows + 7) / 8;
  const int TG = res_tgroups(rows), KG = kResWarps / TG;
  const int tg = warp / KG, kg = warp % KG;
  const int n0 = (int)((int64_t)tg * nN / TG), n1 = (int)((int64_t)(tg + 1) * nN / TG);  // this warp's n-tiles
  const int spr = (md.Iq0 + 3) / 4, S = md.Jp * spr;
  const int sb = (int)((int64_t)kg * S / KG), se = (int)((int64_t)(kg + 1) * S / KG);
  const uint32_t dst = sMp + (uint32_t)(kg * rows * Cpi) * 8u;
  for (int nb = n0; nb < n1; nb += kResMaxNw) {  // passes of <= 4 n-tiles
    const int nw = min(kResMaxNw, n1 - nb);
#define RES_PASS(M_, W_) \
  case (M_)*8 + (W_): res_pass<M_, W_>(md, sT, sUq, sbase, dst, Cpi, nb, sb, se, spr); break;
    switch (nM * 8 + nw) {
      RES_PASS(1, 1) RES_PASS(1, 2) RES_PASS(1, 3) RES_PASS(1, 4)
      RES_PASS(2, 1) RES_PASS(2, 2) RES_PASS(2, 3) RES_PASS(2, 4)
      RES_PASS(3, 1) RES_PASS(3, 2) RES_PASS(3, 3) RES_PASS(3, 4)
      RES_PASS(4, 1) RES_PASS(4, 2) RES_PASS(4, 3) RES_PASS(4, 4)
      default: break;
    }
#undef RES_PASS
  }
  if (KG > 1) {
    __syncthreads();
    for (int e = tid; e < rows * Cpi; e += kResThreads) {  // fixed kg order into slice 0
      double x = lds_f64(sMp + (uint32_t)e * 8u);
      for (int q = 1; q < KG; ++q) x += lds_f64(sMp + (uint32_t)(q * rows * Cpi + e) * 8u);
      sts_f64(sMp + (uint32_t)e * 8u, x);
    }
  }
}

// per-CTA scratch of the owner updates and the per-owned-submodel state (dynamic shared memory)
struct ResOwn {
  int sub, it, fl, pad_;
  int64_t pz;
  double nt2, fp;
};
struct ResScr {
  double H[kResMaxOwn][64], Lf[kResMaxOwn][64], Linv[kResMaxOwn][8];
  double tol;
  int use_pinv[kResMaxOwn], any_active;
  ResOwn own[kResMaxOwn];
};

__device__ __forceinline__ double res_warp_sum(double x) {  // fixed tree to lane 0, then broadcast
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  return __shfl_sync(0xffffffffu, x, 0);
}

// ALS update of owned submodel j (slot w of this CTA) after mode n's partial blocks are complete
// (Alg. 3 alg:cals_jk:hadamard .. alg:cals_jk:error), by ONE warp (warp w): no CTA
// barrier on the critical path, and the owned submodels of a CTA update in parallel.
template <int RMAX>
static __device__ __forceinline__ void res_update_warp(const ResArgs& a, ResScr* sc, double* Ms, double* Vs,
                                                       double* Gs, int* Xs, double* Mp, double* Un, int n, int j,
                                                       int w) {
  cgr::cluster_group cl = cgr::this_cluster();
  const int lane = threadIdx.x & 31;
  const int N = a.N, R = a.R, Cpi = a.Cpi, last = N - 1;
  const int In = a.dims[n];
  const int ldm = R | 1;
  const int sub = sc->own[w].sub;
  const int cb = j * R;
  double* H = sc->H[w];
  double* Lf = sc->Lf[w];
  double* Linv = sc->Linv[w];
  // (a3) Hadamard of the cached Gramians of the other modes
  for (int e = lane; e < R * R; e += 32) {
    double hh = 1.0;
    for (int m = 0; m < N; ++m)
      if (m != n) hh *= Gs[(w * N + m) * R * R + e];
    H[e] = hh;
  }
  // (a2) gather M: the cs partial blocks summed in rank order (mode N-1: the slab owner's rows)
  for (int e = lane; e < In * R; e += 32) {
    const int i = e / R, r = e % R;
    double x;
    if (n == last) {
      const double* pm = cl.map_shared_rank(Mp, i / a.slab);
      x = pm[(i % a.slab) * Cpi + cb + r];
    } else {  // all cs remote loads in flight, then the adds in rank order
      double v[16];
#pragma unroll
      for (int qq = 0; qq < 16; ++qq) v[qq] = qq < a.cs ? cl.map_shared_rank(Mp, qq)[i * Cpi + cb + r] : 0.0;
      x = 0.0;
#pragma unroll
      for (int qq = 0; qq < 16; ++qq)
        if (qq < a.cs) x += v[qq];
    }
    Ms[i * ldm + r] = x;
  }
  __syncwarp();
  // (a4) Cholesky H = L L^T (textbook, no pivoting) on lane 0; pinv fallback
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
    sc->use_pinv[w] = ok ? 0 : 1;
    if (ok) {
#pragma unroll
      for (int i = 0; i < RMAX; ++i)
#pragma unroll
        for (int jj = 0; jj <= i; ++jj)
          if (i < R) Lf[i * R + jj] = L[i][jj];
    } else {
      jacobi_pinv<RMAX>(H, R, Lf, 1e-12);
      sc->own[w].fl |= F_PINV;
      a.flags[sub] = sc->own[w].fl;
    }
  }
  __syncwarp();
  const bool pinv = sc->use_pinv[w] != 0;
  const int64_t pz0 = (n == 0) ? sc->own[w].pz : -1, pz1 = (n == 0) ? pz0 + a.d : -1;
  // (a4/a5) V(i,:) = M(i,:) H^-1 (lanes over rows; the left-out rows of mode 0 are zero), with
  // this lane's share of V^T V (upper triangle) and V.M
  constexpr int NQ = RMAX * (RMAX + 1) / 2;
  double accq[NQ + 1];
#pragma unroll
  for (int z = 0; z <= NQ; ++z) accq[z] = 0.0;
  for (int i = lane; i < In; i += 32) {
    double mv[RMAX], v[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) mv[r] = (r < R) ? Ms[i * ldm + r] : 0.0;
    if (i >= pz0 && i < pz1) {
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
      if (r < R) Vs[i * ldm + r] = v[r];
#pragma unroll
      for (int c = r; c < RMAX; ++c, ++z) accq[z] += v[r] * v[c];
    }
#pragma unroll
    for (int r = 0; r < RMAX; ++r) accq[NQ] += v[r] * mv[r];
  }
#pragma unroll
  for (int z = 0; z <= NQ; ++z) accq[z] = res_warp_sum(accq[z]);  // totals, on every lane
  __syncwarp();
  auto vtv = [&](int r, int c) -> double {
    const int lo = r < c ? r : c, hi = r < c ? c : r;
    const int idx = lo * RMAX - lo * (lo - 1) / 2 + (hi - lo);
    double x = 0.0;
#pragma unroll
    for (int z = 0; z < NQ; ++z)
      if (z == idx) x = accq[z];
    return x;
  };
  // (a6) lambda_r = ||V(:,r)||; U = V / lambda (lambda = 0: unchanged)
  double lam[RMAX], il[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    lam[r] = r < R ? sqrt(vtv(r, r)) : 0.0;
    il[r] = lam[r] > 0.0 ? 1.0 / lam[r] : 1.0;
  }
  // the new block, into every CTA's replica (DSMEM stores; the cluster barrier after the updates
  // orders them)
  for (int e = lane; e < In * R; e += 32) {
    const int i = e / R, r = e % R;
    double ir = 1.0;
#pragma unroll
    for (int rr = 0; rr < RMAX; ++rr)
      if (rr == r) ir = il[rr];
    const double u = Vs[i * ldm + r] * ir;
    for (int qq = 0; qq < a.cs; ++qq) cl.map_shared_rank(Un, qq)[i * Cpi + cb + r] = u;
  }
  if (lane == 0) {
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < R; ++c) Gs[(w * N + n) * R * R + r * R + c] = vtv(r, c) * il[r] * il[c];
    if (n == last) {  // (a7) error, fit, history, convergence mask
      for (int r = 0; r < R; ++r) a.lambda[(int64_t)sub * R + r] = lam[r];
      double quad = 0.0;
      for (int r = 0; r < R; ++r)
        for (int c = 0; c < R; ++c) quad += H[r * R + c] * vtv(r, c);
      const double crs = accq[NQ];
      ResOwn& o = sc->own[w];
      const double nt2 = o.nt2;
      const double e = nt2 + quad - 2.0 * crs;
      const int itn = o.it + 1;
      o.it = itn;
      a.iters[sub] = itn;
      a.err[sub] = e;
      a.hist[(int64_t)sub * a.hist_cap + (itn - 1) % a.hist_cap] = e;
      int f = o.fl;
      bool act = true;
      if (!isfinite(e)) {
        f |= F_NONFINITE;
        act = false;
      } else {
        if (e < -1e-9 * nt2) f |= F_BREAKDOWN;
        const double fitv = nt2 > 0.0 ? 1.0 - sqrt(fmax(e, 0.0)) / sqrt(nt2) : 0.0;
        const double tol = sc->tol;
        if (tol > 0.0 && itn >= 2 && fabs(fitv - o.fp) < tol) {
          f |= F_CONVERGED;
          act = false;
        }
        a.fit[sub] = fitv;
        a.fit_prev[sub] = fitv;
        o.fp = fitv;
      }
      a.flags[sub] = f;
      o.fl = f;
      if (!act) {
        a.active[sub] = 0;
        cl.map_shared_rank(Xs, 0)[j] = 0;  // read by every CTA after the sweep's last barrier
      }
    }
  }
  __syncwarp();
}

template <int RMAX>
__global__ void __launch_bounds__(kResThreads, 1) resident_sweep_kernel(ResArgs a) {
  extern __shared__ __align__(16) unsigned char res_smem[];
  cgr::cluster_group cl = cgr::this_cluster();
  const int rank = (int)cl.block_rank();
  const int q = blockIdx.x / a.cs;  // cluster = submodel group
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = a.N, R = a.R, Cp = a.Cp, Cpi = a.Cpi, last = N - 1;
  const int k0 = q * a.kpc, kq = min(a.kpc, a.K - k0);  // the group's blocks [k0, k0 + kq)
  const int Cq = kq * R;
  const int s0 = rank * a.slab, slen = max(0, min(a.slab, a.dims[last] - s0));  // this CTA's slab
  int Imax = 1;
  for (int m = 0; m < N; ++m) Imax = max(Imax, a.dims[m]);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(res_smem);

  double* Ts = reinterpret_cast<double*>(res_smem + a.o_T);
  double* Mp = reinterpret_cast<double*>(res_smem + a.o_M);   // [KG][rows][Cpi]; slice 0 = the CTA's block
  double* Es = reinterpret_cast<double*>(res_smem + a.o_E);   // owner scratch per slot: M, V (Imax x ldm each)
  double* Gs = reinterpret_cast<double*>(res_smem + a.o_G);   // owned Gramians [own][N][R][R]
  int* Xs = reinterpret_cast<int*>(res_smem + a.o_X);         // [0..kpc): activity (CTA 0's copy is the group's)
#define RES_U(m) reinterpret_cast<double*>(res_smem + a.o_U[m])  // mode-m factor replica [I_m][Cpi]
  ResScr* sc = reinterpret_cast<ResScr*>(res_smem + a.o_S);  // owner scratch, owned-submodel state

  // ---------------- load: T slab, factor replicas, owned state, activity
  {
    int nel = slen;
    for (int m = 0; m < last; ++m) nel *= a.dims[m];
    for (int e = tid; e < nel; e += kResThreads) {  // e enumerates (i_0, ..., i_{N-2}, local i_{N-1})
      int rem = e;
      int64_t so = 0, go = 0;
      for (int m = 0; m < last; ++m) {
        const int im = rem % a.dims[m];
        rem /= a.dims[m];
        so += (int64_t)im * a.pitch[m];
        go += (int64_t)im * a.gst[m];
      }
      so += (int64_t)rem * a.pitch[last];
      go += (int64_t)(rem + s0) * a.gst[last];
      Ts[so] = a.T[go];
    }
    for (int m = 0; m < N; ++m)
      for (int e = tid; e < a.dims[m] * Cpi; e += kResThreads) {
        const int i = e / Cpi, c = e % Cpi;
        RES_U(m)[e] = c < Cq ? a.U[m][(int64_t)i * a.ldu + (int64_t)k0 * R + c] : 0.0;
      }
    for (int j = rank, w = 0; j < kq; j += a.cs, ++w) {
      const int sub = a.blk2sub[k0 + j];
      if (tid == 0) {
        sc->own[w].sub = sub;
        sc->own[w].pz = a.pglob[sub];
        sc->own[w].nt2 = a.normT2p[sub];
        sc->own[w].it = a.iters[sub];
        sc->own[w].fl = a.flags[sub];
        sc->own[w].fp = a.fit_prev[sub];
      }
      for (int e = tid; e < N * R * R; e += kResThreads) {
        const int m = e / (R * R), rr = e % (R * R);
        Gs[(w * N + m) * R * R + rr] = a.gram[((int64_t)m * a.nsub + sub) * R * R + rr];
      }
    }
    if (rank == 0)
      for (int j = tid; j < kq; j += kResThreads) Xs[j] = a.active[a.blk2sub[k0 + j]];
    if (tid == 0) sc->tol = *a.tol;
  }
  __syncthreads();
  res_cluster_sync();
  const int* act0 = cl.map_shared_rank(Xs, 0);  // the group's activity flags live in CTA 0

  int sweeps = 0;
#ifdef JK_RES_PROF
  long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, plast = clock64();
#endif
  for (int it = 0; it < a.max_iters; ++it) {
    if (tid == 0) {
      int any = 0;
      for (int j = 0; j < kq; ++j) any |= act0[j];
      sc->any_active = any;
    }
    __syncthreads();
    if (!sc->any_active) break;  // uniform over the cluster: every CTA reads the same flags
    ++sweeps;
    for (int n = 0; n < N; ++n) {
      // ================= MTTKRP share of this CTA (rows: mode-n indices; slab rows at n = N-1)
      {
        ResMode md;
        const int q0 = (n == 0) ? 1 : 0;
        md.rows = (n == last) ? slen : a.dims[n];
        md.Iq0 = a.dims[q0];
        md.pn = a.pitch[n];
        md.pq = a.pitch[q0];
        md.ns = 0;
        md.Jp = 1;
#pragma unroll
        for (int z = 0; z < kMaxModes - 2; ++z) md.ext[z] = 1, md.spt[z] = 0, md.sg0[z] = 0, md.suo[z] = 0;
        for (int m = 0; m < N; ++m) {
          if (m == n || m == q0) continue;
          const int ex = (m == last) ? slen : a.dims[m];
#pragma unroll
          for (int z = 0; z < kMaxModes - 2; ++z)
            if (z == md.ns) {
              md.ext[z] = ex;
              md.spt[z] = a.pitch[m];
              md.sg0[z] = (m == last) ? s0 : 0;
              md.suo[z] = a.o_U[m];
            }
          md.Jp *= ex;
          ++md.ns;
        }
        if (md.Jp == 0) {  // an empty slab contributes zeros
          for (int e = tid; e < md.rows * Cpi; e += kResThreads) Mp[e] = 0.0;
        } else {
          res_mttkrp(md, sbase + a.o_T, sbase + a.o_U[q0], sbase, sbase + a.o_M, Cp, Cpi);
        }
      }
      RES_T(0);
      __syncthreads();
      RES_T(1);
      res_cluster_sync();  // every CTA's partial block is complete (and readable via DSMEM)
      RES_T(2);

      // ================= ALS update of the owned submodels (Alg. 3)
      const int ldm = R | 1;
      {
        const int w = warp, j = rank + warp * a.cs;  // owned slot w on warp w (in parallel)
        if (w < kResMaxOwn && j < kq && act0[j]) {
          double* Ms = Es + (size_t)w * 2 * Imax * ldm;
          res_update_warp<RMAX>(a, sc, Ms, Ms + (size_t)Imax * ldm, Gs, Xs, Mp, RES_U(n), n, j, w);
        }
      }
      RES_T(5);
      RES_T(6);
      res_cluster_sync();  // new blocks visible in every replica; partial blocks free again
      RES_T(7);
    }
  }

  // ---------------- write back the owned submodels' factors (every mode) and Gramians
  for (int j = rank, w = 0; j < kq; j += a.cs, ++w) {
    const int sub = sc->own[w].sub;
    for (int m = 0; m < N; ++m)
      for (int e = tid; e < a.dims[m] * R; e += kResThreads) {
        const int i = e / R, r = e % R;
        a.U[m][(int64_t)i * a.ldu + (int64_t)(k0 + j) * R + r] = RES_U(m)[i * Cpi + j * R + r];
      }
    for (int e = tid; e < N * R * R; e += kResThreads) {
      const int m = e / (R * R), rr = e % (R * R);
      a.gram[((int64_t)m * a.nsub + sub) * R * R + rr] = Gs[(w * N + m) * R * R + rr];
    }
  }
  if (rank == 0 && tid == 0) atomicMax(a.sweeps_out, sweeps);
#ifdef JK_RES_PROF
  if (blockIdx.x == 0 && tid == 0)
    for (int i = 0; i < 8; ++i) a.prof[i] = pacc[i];
#endif
  res_cluster_sync();  // no CTA exits while a peer may still read its shared memory
#undef RES_U
}

}  // namespace jk
