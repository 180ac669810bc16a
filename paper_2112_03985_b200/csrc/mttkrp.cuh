// mttkrp.cuh — fused Khatri-Rao + MTTKRP on the FP64 tensor pipe (sm_100a DMMA).
//
// Computes, for one mode n (Alg. 3 alg:cals_jk:mttkrp; Eq. 1):
//     M(i, c) = sum_j T_(n)(i, j) * KRP(j, c),   KRP(j, c) = prod_{m != n} U_m(i_m(j), c)
// for all fused columns c of all active submodels at once (CALS fusion).
// The KRP is generated tile by tile in shared memory and never touches HBM.
//
// GEMM view: D[c][i] = sum_j A[c][j] * B[j][i] with A = KRP^T (C side = MMA "m"),
// B = T_(n)^T (I_n side = MMA "n"), K = J_n. sm_100a has no FP64 tcgen05 kind, so the
// contraction runs on mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), which the microbenchmark in
// tools/microbench_fp64.cu measured at 37.05 TFLOP/s on B200 (= the chip's FP64 peak).
//
// Work decomposition: "stream-K". The (C/BM) x (I_n/BN) output tiles x (J/BK) k-tiles form
// one linear unit space split evenly over G = #SMs x occupancy CTAs (one wave, balanced to
// +-1 k-tile). A CTA whose range spans tiles writes one partial "piece" per tile; the
// epilogue sums a tile's pieces in a fixed order (deterministic).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace jk {

constexpr int kMaxModes = 8;
constexpr int kBK = 16;  // k-tile depth (j values per shared-memory stage)

struct ModeView {
  int N;                               // number of modes
  int n;                               // the mode being updated
  int nrest;                           // N - 1
  int In;                              // I_n
  int J;                               // prod_{m != n} I_m  (< 2^31, checked on the host)
  int L;                               // prod_{m < n} I_m: stride of i_n in T
  int64_t LIn;                         // L * I_n
  int rdim[kMaxModes - 1];             // I_m of the modes m != n, ascending m
  const double* U[kMaxModes - 1];      // multi-factor of mode m (row-major I_m x ldu)
};

// Per output tile: the first CTA touching it, its number of partial pieces and the base
// index of its pieces in the partial buffer.
struct TileInfo {
  int first_cta;
  int npieces;
  int piece_base;
  int pad_;
};

struct MttkrpGeom {
  int C;          // fused width in use (columns >= C of U are zero up to round_up(C, BM))
  int64_t ldu;    // row pitch of every U_m
  int nMt, nNt;   // output tiles along C and along I_n
  int KT;         // k-tiles: ceil(J / kBK)
  int64_t units;  // nMt * nNt * KT
  int G;          // CTAs launched
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src_size = valid ? 8 : 0;  // src-size 0 => zero fill (OOB rows / tail j)
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_size));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int NT, int WARPS>
struct MttkrpCfg {
  static constexpr int kThreads = WARPS * 32;
  static constexpr int BM = WARPS * 16;                    // fused columns per CTA tile
  static constexpr int BN = NT * 8;                        // rows of M (I_n) per CTA tile
  static constexpr int BMP = BM + 8;                       // 64B-shifted rows: conflict-free
  static constexpr int BNP = (NT % 2 == 0) ? BN + 8 : BN;  // row pitch = 8 mod 16 doubles
  static constexpr size_t kSmemA = 2ull * kBK * BMP * sizeof(double);
  static constexpr size_t kSmemB = 2ull * kBK * BNP * sizeof(double);
  static constexpr size_t kSmemTab = 2ull * kBK * sizeof(int64_t) + 2ull * (kMaxModes - 1) * kBK * sizeof(int);
  static constexpr size_t kSmem = kSmemA + kSmemB + kSmemTab;
};

// Build the per-k-tile index table: for each j of the tile, the T offset without the i_n
// term (l + L*I_n*r with j = l + L*r, Eq. 3) and the row offsets i_m(j)*ldu into every U_m.
__device__ __forceinline__ void build_table(const ModeView& v, int64_t ldu, int kt, int64_t* tofs,
                                            int* koff) {
  int t = threadIdx.x;
  if (t < kBK) {
    int j = kt * kBK + t;
    if (j < v.J) {
      int l = j % v.L, r = j / v.L;
      tofs[t] = (int64_t)l + v.LIn * (int64_t)r;
      int rem = j;
#pragma unroll
      for (int q = 0; q < kMaxModes - 1; ++q) {
        if (q < v.nrest) {
          int i = rem % v.rdim[q];
          rem /= v.rdim[q];
          koff[q * kBK + t] = i * (int)ldu;
        }
      }
    } else {
      tofs[t] = -1;
#pragma unroll
      for (int q = 0; q < kMaxModes - 1; ++q) koff[q * kBK + t] = 0;
    }
  }
}

template <int NT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1)
    mttkrp_dmma_kernel(ModeView v, const double* __restrict__ T, MttkrpGeom g,
                       const TileInfo* __restrict__ tinfo, double* __restrict__ parts) {
  using Cfg = MttkrpCfg<NT, WARPS>;
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BMP = Cfg::BMP, BNP = Cfg::BNP;
  constexpr int THREADS = Cfg::kThreads;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);                     // [2][BK][BMP]
  double* Bs = As + 2 * kBK * BMP;                                      // [2][BK][BNP]
  int64_t* tofs = reinterpret_cast<int64_t*>(Bs + 2 * kBK * BNP);       // [2][BK]
  int* koff = reinterpret_cast<int*>(tofs + 2 * kBK);                   // [2][MAXM-1][BK]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int b = blockIdx.x;
  const int64_t u0 = (int64_t)b * g.units / g.G, u1 = (int64_t)(b + 1) * g.units / g.G;
  const bool lmode = (v.L == 1);  // mode 0: i_n contiguous in T

  int64_t u = u0;
  while (u < u1) {
    const int t = (int)(u / g.KT);
    const int kt0 = (int)(u % g.KT);
    const int64_t kt_end = (int64_t)kt0 + (u1 - u);
    const int kt1 = (int)(kt_end < (int64_t)g.KT ? kt_end : (int64_t)g.KT);
    u += kt1 - kt0;
    const int tm = t % g.nMt, tn = t / g.nMt;
    const int c0 = tm * BM, i0 = tn * BN;
    const bool warp_live = (c0 + warp * 16) < g.C;

    double acc[2][NT][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    auto load_T = [&](int s) {
      const int64_t* tf = tofs + s * kBK;
      double* bs = Bs + s * kBK * BNP;
      for (int e = tid; e < kBK * BN; e += THREADS) {
        int k, i;
        if (lmode) { k = e / BN; i = e % BN; } else { k = e % kBK; i = e / kBK; }
        int gi = i0 + i;
        int64_t off = tf[k];
        bool valid = (gi < v.In) && (off >= 0);
        const double* src = valid ? (T + off + (int64_t)v.L * gi) : T;
        cp_async8(bs + k * BNP + i, src, valid);
      }
      cp_async_commit();
    };
    auto gen_A = [&](int s) {
      const int* ko = koff + s * (kMaxModes - 1) * kBK;
      double* as = As + s * kBK * BMP;
      for (int e = tid; e < kBK * BM; e += THREADS) {
        int k = e / BM, c = e % BM;
        int gc = c0 + c;
        double val = 0.0;
        if (gc < g.C) {
          val = 1.0;
          // descending mode order of Eq. 1
#pragma unroll
          for (int q = kMaxModes - 2; q >= 0; --q)
            if (q < v.nrest) val *= __ldg(v.U[q] + ko[q * kBK + k] + gc);
        }
        as[k * BMP + c] = val;
      }
    };

    build_table(v, g.ldu, kt0, tofs, koff);
    __syncthreads();
    load_T(0);
    gen_A(0);
    for (int kt = kt0; kt < kt1; ++kt) {
      const int s = (kt - kt0) & 1;
      const bool more = (kt + 1) < kt1;
      if (more) build_table(v, g.ldu, kt + 1, tofs + (s ^ 1) * kBK, koff + (s ^ 1) * (kMaxModes - 1) * kBK);
      cp_async_wait_all();
      __syncthreads();
      if (more) load_T(s ^ 1);
      if (warp_live) {
        const double* as = As + s * kBK * BMP + warp * 16 + gid;
        const double* bs = Bs + s * kBK * BNP + gid;
#pragma unroll
        for (int kk = 0; kk < kBK / 4; ++kk) {
          const int kr = kk * 4 + tig;
          double a0 = as[kr * BMP], a1 = as[kr * BMP + 8];
#pragma unroll
          for (int ni = 0; ni < NT; ++ni) {
            if (i0 + ni * 8 < v.In) {
              double bb = bs[kr * BNP + ni * 8];
              dmma_m8n8k4(acc[0][ni][0], acc[0][ni][1], a0, bb);
              dmma_m8n8k4(acc[1][ni][0], acc[1][ni][1], a1, bb);
            }
          }
        }
      }
      if (more) gen_A(s ^ 1);
    }
    __syncthreads();

    // partial piece of tile t written by this CTA
    const TileInfo ti = tinfo[t];
    double* P = parts + ((int64_t)ti.piece_base + (b - ti.first_cta)) * (int64_t)(BN * BM);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        const int cl = warp * 16 + mi * 8 + gid;
        const int il = ni * 8 + 2 * tig;
        P[(int64_t)il * BM + cl] = acc[mi][ni][0];
        P[(int64_t)(il + 1) * BM + cl] = acc[mi][ni][1];
      }
  }
}

// Plain reduction of the partial pieces into a dense row-major M (stand-alone op only; the
// JK-CALS path reduces inside the epilogue instead).
__global__ void reduce_parts_kernel(const double* __restrict__ parts, const TileInfo* __restrict__ tinfo,
                                    int In, int C, int BM, int BN, int nMt, double* __restrict__ M,
                                    int64_t ldm) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)In * C) return;
  int i = (int)(e / C), c = (int)(e % C);
  int tn = i / BN, tm = c / BM;
  TileInfo ti = tinfo[tn * nMt + tm];
  const double* p = parts + (int64_t)ti.piece_base * BN * BM + (int64_t)(i - tn * BN) * BM + (c - tm * BM);
  double s = 0.0;
  for (int pc = 0; pc < ti.npieces; ++pc) s += p[(int64_t)pc * BN * BM];
  M[(int64_t)i * ldm + c] = s;
}

// Materialised Khatri-Rao generation (a1 in SURVEY §8a): K(j, c) = prod_{m != n} U_m(i_m(j), c),
// row-major J x ldk. Each thread owns 4 consecutive columns and a run of kRows consecutive j,
// advancing the mixed-radix index incrementally; stores are 32-byte vectors (st.global.v4.f64).
constexpr int kKrpRows = 64;
__global__ void __launch_bounds__(256) krp_gen_kernel(ModeView v, int C, int64_t ldu, double* __restrict__ K,
                                                      int64_t ldk) {
  const int c = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  if (c >= C) return;
  const int j0 = blockIdx.x * kKrpRows;
  if (j0 >= v.J) return;
  const int j1 = min(v.J, j0 + kKrpRows);
  int idx[kMaxModes - 1];
  int rem = j0;
#pragma unroll
  for (int q = 0; q < kMaxModes - 1; ++q)
    if (q < v.nrest) { idx[q] = rem % v.rdim[q]; rem /= v.rdim[q]; }
  const bool full4 = (c + 4 <= C) && ((ldu & 3) == 0) && ((ldk & 3) == 0);
  for (int j = j0; j < j1; ++j) {
    double r0 = 1.0, r1 = 1.0, r2 = 1.0, r3 = 1.0;
#pragma unroll
    for (int q = kMaxModes - 2; q >= 0; --q) {
      if (q < v.nrest) {
        const double* row = v.U[q] + (int64_t)idx[q] * ldu + c;
        if (full4) {
          double4 x = *reinterpret_cast<const double4*>(row);  // 32B-aligned (ldu % 4 == 0)
          r0 *= x.x; r1 *= x.y; r2 *= x.z; r3 *= x.w;
        } else {
          r0 *= row[0];
          if (c + 1 < C) r1 *= row[1];
          if (c + 2 < C) r2 *= row[2];
          if (c + 3 < C) r3 *= row[3];
        }
      }
    }
    double* dst = K + (int64_t)j * ldk + c;
    if (full4) {
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(dst), "d"(r0), "d"(r1), "d"(r2), "d"(r3)
                   : "memory");
    } else {
      dst[0] = r0;
      if (c + 1 < C) dst[1] = r1;
      if (c + 2 < C) dst[2] = r2;
      if (c + 3 < C) dst[3] = r3;
    }
    // mixed-radix increment (mode order ascending = Eq. 3 column order)
#pragma unroll
    for (int q = 0; q < kMaxModes - 1; ++q) {
      if (q < v.nrest) {
        if (++idx[q] < v.rdim[q]) break;
        idx[q] = 0;
      }
    }
  }
}

}  // namespace jk
