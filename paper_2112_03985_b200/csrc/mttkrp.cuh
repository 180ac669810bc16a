// mttkrp.cuh — fused Khatri-Rao + MTTKRP on the FP64 tensor pipe (sm_100a DMMA).
//
// Computes, for one mode n (Alg. 3 alg:cals_jk:mttkrp; Eq. 1):
//     M(i, c) = sum_j T_(n)(i, j) * KRP(j, c),   KRP(j, c) = prod_{m != n} U_m(i_m(j), c)
// for all fused columns c of all active submodels at once (CALS fusion).
// The KRP is never materialised: with q0 the fastest "rest" mode (Eq. 3 column order) and
// j = i_q0 + I_q0 * j', every KRP row factors as U_q0(i_q0, c) * S_{j'}(c), where
// S_{j'} = prod of the slower rest modes' rows. A k-tile is BK consecutive i_q0 at one j':
// the A operand (KRP^T) of the tile is a BK x BM slab of U_q0 (staged once per i_q0 block and
// reused for all J' tiles) scaled column-wise by one S row (N-2 factor rows, staged per tile).
//
// GEMM view: D[c][i] = sum_j A[c][j] * B[j][i] with A = KRP^T (C side = MMA "m"),
// B = T_(n)^T (I_n side = MMA "n"). sm_100a has no FP64 tcgen05 kind, so the contraction
// runs on mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), measured at 37.05 TFLOP/s on B200
// (tools/microbench_fp64.cu), the chip's FP64 peak.
//
// Data movement: one thread per CTA issues, per k-tile, a 4-D TMA box of T (zero-filled at the
// ragged edges), 1-D bulk copies of the N-2 slow-mode factor rows and, when the i_q0 block
// changes, a 2-D TMA box of the U_q0 slab, all completing on the stage's mbarrier; a
// STAGES-deep shared-memory ring keeps STAGES-1 k-tiles in flight; 2 CTAs/SM.
// Work decomposition: "stream-K" -- the (C/BM) x (I_n/BN) output tiles x KT k-tiles form one
// linear unit space split evenly over G = #SMs x occupancy CTAs (one wave); a CTA spanning
// several tiles writes one partial "piece" per tile, summed in a fixed order later.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace jk {

constexpr int kMaxModes = 8;
constexpr int kBK = 16;      // k-tile depth (i_q0 values per tile)
constexpr int kWarps = 8;    // warps per CTA; each warp owns 16 fused columns
constexpr int kBM = kWarps * 16;
constexpr int kBMP = kBM + 4;  // row pitch = 4 mod 16 doubles: conflict-free 64-bit fragment loads
constexpr int kMaxNT = 8;    // n8 tiles per CTA (BN <= 64)

// generic mode description (stand-alone KRP generator and host helpers)
struct ModeView {
  int N, n, nrest;
  int In;
  int J;                            // prod_{m != n} I_m (< 2^31)
  int L;                            // prod_{m < n} I_m
  int64_t LIn;
  int rdim[kMaxModes - 1];          // I_m of the modes m != n, ascending m
  const double* U[kMaxModes - 1];   // their multi-factors (row-major I_m x ldu)
};

// mode description for the fused kernel (q0 = fastest rest mode, "slow" = the others)
struct MttkrpView {
  int In;                           // I_n
  int Iq0;                          // I_q0
  int nb0;                          // ceil(I_q0 / BK)
  int Jp;                           // J' = prod of the slow rest modes
  int runA;                         // j' = jA + runA * jB (slow modes merged into <= 2 runs for TMA)
  int nslow;                        // N - 2
  int sdim[kMaxModes - 2];          // dims of the slow rest modes, ascending
  const double* Us[kMaxModes - 2];  // slow rest modes' U (row-major I x ldu)
};

struct TileInfo {
  int first_cta;
  int npieces;
  int piece_base;
  int pad_;
};

struct MttkrpGeom {
  int C;          // fused width in use
  int64_t ldu;    // row pitch of every U_m (multiple of 128 doubles)
  int nMt, nNt;   // output tiles along C and along I_n
  int KT;         // k-tiles per output tile: nb0 * J'
  int64_t units;  // nMt * nNt * KT
  int G;          // CTAs launched
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// ---- mbarrier / TMA / bulk-copy primitives (PTX ISA 8.x, sm_90+; SASS UTMALDG / UBLKCP / SYNCS)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int x0, int x1, int x2, int x3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int x0, int x1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(x0), "r"(x1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// one lane of a converged warp (lane 0 when all are active): issue slot for single-thread
// instructions while the whole warp walks the loop, so that every operand stays warp-uniform
// (uniform registers for tcgen05.mma / TMA, no per-lane serialisation loops)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 r;\n.reg .pred p;\nelect.sync r|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Shared-memory layout of one CTA (every buffer 128-byte aligned for TMA):
//   Ub[2][BK][BMP]                       U_q0 slab, double-buffered on b0 parity (2-D TMA, box 132 x 16)
//   STAGES x { Bt (T tile, 4-D TMA box), Ss[nslow][BM] (slow-mode rows, 1-D bulk copies) }
//   full[STAGES] mbarriers
// B layout: KMAJOR=false (n == 0: i_n contiguous in T) -> Bt[k][BNP], box (BNP, 16), BNP = 4 mod 16;
//           KMAJOR=true  (n >= 1: i_q0 contiguous in T) -> Bt[i][BKP], box (20, BN), BKP = 20.
// The 4-double over-fetch of each box row makes the row pitch 4 mod 16 doubles, so the 64-bit
// fragment loads of a half-warp hit 16 distinct bank pairs.
template <int NT, bool KMAJOR, int STAGES, int WM = kWarps, int KB = kBK>
struct MttkrpCfg {
  static constexpr int BM = WM * 16;  // fused columns of a tile: WM consumer warps x 16
  static constexpr int BMP = BM + 4;  // = 4 mod 16 doubles for WM in {5, 8}: conflict-free loads
  static constexpr int BN = NT * 8;
  static constexpr int BNP = BN + ((4 - BN % 16) + 16) % 16;  // BN rounded up to 4 mod 16
  static constexpr int BKP = KB + ((4 - KB % 16) + 16) % 16;  // KB rounded up to 4 mod 16 (16 -> 20, 20 -> 20)
  static constexpr int kBTile = KMAJOR ? BN * BKP : KB * BNP;   // doubles (= TMA box volume)
  static constexpr unsigned kTBytes = kBTile * 8u;
  static constexpr size_t kUb = 2ull * KB * BMP;                // doubles
  __host__ __device__ static size_t stage_doubles(int nslow) { return (size_t)kBTile + (size_t)nslow * BM; }
  __host__ __device__ static size_t smem_bytes(int nslow) {
    return 128 + (kUb + (size_t)STAGES * stage_doubles(nslow)) * sizeof(double) + 2 * STAGES * sizeof(uint64_t);
  }
};

template <int NT, bool KMAJOR, int STAGES, int WM = kWarps, int KB = kBK>
__global__ void __maxnreg__(NT <= 6 ? 96 : 112)
    mttkrp_dmma_kernel(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmU,
                       MttkrpView v, MttkrpGeom g, const TileInfo* __restrict__ tinfo, double* __restrict__ parts) {
  using Cfg = MttkrpCfg<NT, KMAJOR, STAGES, WM, KB>;
  constexpr int BN = Cfg::BN, BNP = Cfg::BNP, BKP = Cfg::BKP, BT = Cfg::kBTile;
  constexpr int BM = Cfg::BM, BMP = Cfg::BMP;
  // (no integer round-trip on the base pointer: it must stay in the shared window so that the
  // fragment loads compile to LDS, not generic LD)
  extern __shared__ __align__(1024) double smem[];
  double* Ub = smem;                                // [2][BK][BMP]
  double* stage0 = smem + Cfg::kUb;                 // STAGES x (BT + nslow*BM)
  const int stage_sz = (int)Cfg::stage_doubles(v.nslow);
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + (size_t)STAGES * stage_sz);  // data landed
  uint64_t* empty = full + STAGES;                                                     // consumers done

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.x;
  const int* cta_u = reinterpret_cast<const int*>(tinfo + g.nMt * g.nNt);  // packed after the tile table
  const int64_t u0 = cta_u[b], u1 = cta_u[b + 1];

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WM);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  // =========================== producer warp (warp WM, one lane) ===========================
  // (r01: a warp-uniform loop with elect.sync measured no faster here -- the FP64 kernel is
  // DMMA-bound -- and 12 % slower on the 4-way config, so the lane-0 producer stays)
  if (warp == WM) {
    if (lane != 0) return;
    const unsigned s_bytes = (unsigned)v.nslow * BM * 8u;
    // programmatic dependent launch: T is constant, so the T tiles of the first STAGES k-tiles
    // are requested BEFORE waiting for the previous grid (the previous mode's epilogue, which
    // writes U); their barriers expect the full tile bytes and complete once the U rows issued
    // after the wait land too. U and the partial buffer are only touched after the wait.
    int npre = 0;
    if (u0 < u1) {
      const int t = (int)(u0 / g.KT);
      const int kt0 = (int)(u0 % g.KT);
      const int64_t kt_end = (int64_t)kt0 + (u1 - u0);
      const int kt1 = (int)(kt_end < (int64_t)g.KT ? kt_end : (int64_t)g.KT);
      npre = kt1 - kt0 < STAGES ? kt1 - kt0 : STAGES;
      const int i0 = (t / g.nMt) * BN;
      int b0 = kt0 / v.Jp, jp = kt0 % v.Jp, ja = jp % v.runA, jb = jp / v.runA, lb0 = -1;
      for (int q = 0; q < npre; ++q) {
        double* st = stage0 + (size_t)q * stage_sz;
        const bool new_slab = (b0 != lb0);
        mbar_expect_tx(&full[q], Cfg::kTBytes + s_bytes + (new_slab ? (unsigned)(KB * BMP * 8) : 0u));
        if (KMAJOR) tma_load_4d(st, &tmT, b0 * KB, ja, i0, jb, &full[q]);
        else tma_load_4d(st, &tmT, i0, b0 * KB, ja, jb, &full[q]);
        lb0 = b0;
        if (++jp == v.Jp) {
          jp = 0;
          ++b0;
        }
        if (++ja == v.runA) {
          ja = 0;
          ++jb;
        }
        if (jp == 0) jb = 0;
      }
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" :::);
    unsigned ld_git = 0;  // tiles issued by this CTA (ring slot + phase)
    for (int64_t u = u0; u < u1;) {
      const int t = (int)(u / g.KT);
      const int kt0 = (int)(u % g.KT);
      const int64_t kt_end = (int64_t)kt0 + (u1 - u);
      const int kt1 = (int)(kt_end < (int64_t)g.KT ? kt_end : (int64_t)g.KT);
      u += kt1 - kt0;
      const int tm = t % g.nMt, tn = t / g.nMt;
      const int c0 = tm * BM, i0 = tn * BN;
      // a new segment reloads the U_q0 slab buffers: wait until every issued tile is consumed
      for (unsigned q = (ld_git >= (unsigned)STAGES ? ld_git - STAGES + 1 : 0); q < ld_git; ++q)
        mbar_wait(&empty[q % STAGES], (q / STAGES) & 1u);
      int ld_b0 = kt0 / v.Jp, ld_jp = kt0 % v.Jp, loaded_b0 = -1;
      int ld_ja = ld_jp % v.runA, ld_jb = ld_jp / v.runA;
      int sidx[kMaxModes - 2];
      {
        int rem = ld_jp;
#pragma unroll
        for (int s = 0; s < kMaxModes - 2; ++s)
          if (s < v.nslow) { sidx[s] = rem % v.sdim[s]; rem /= v.sdim[s]; }
      }
#pragma unroll 1
      for (int kt = kt0; kt < kt1; ++kt) {
        const int slot = (int)(ld_git % STAGES);
        // WAR: the previous use of this slot must have been released by every consumer warp
        if (ld_git >= (unsigned)STAGES) mbar_wait(&empty[slot], ((ld_git / STAGES) - 1) & 1u);
        double* st = stage0 + (size_t)slot * stage_sz;
        uint64_t* bar = &full[slot];
        const bool new_slab = (ld_b0 != loaded_b0);
        // the slab buffer (b0 & 1) was last read by the tiles of block b0 - 2; the slot WAR wait
        // above covers them only when a block spans >= STAGES - 1 tiles, so for very short
        // blocks (tiny tensors) drain every issued tile first
        if (new_slab && loaded_b0 >= 0 && v.Jp < STAGES - 1)
          for (unsigned q = (ld_git >= (unsigned)STAGES ? ld_git - STAGES + 1 : 0); q < ld_git; ++q)
            mbar_wait(&empty[q % STAGES], (q / STAGES) & 1u);
        {
          const bool pre = ld_git < (unsigned)npre;  // T already requested before the wait
          if (!pre) mbar_expect_tx(bar, Cfg::kTBytes + s_bytes + (new_slab ? (unsigned)(KB * BMP * 8) : 0u));
          // U_q0 rows [b0*BK, b0*BK+BK) x columns [c0, c0+BMP): OOB rows are zero
          if (new_slab) tma_load_2d(Ub + (ld_b0 & 1) * (KB * BMP), &tmU, c0, ld_b0 * KB, bar);
          if (!pre) {
            if (KMAJOR) tma_load_4d(st, &tmT, ld_b0 * KB, ld_ja, i0, ld_jb, bar);  // view (q0, runA, n, runB)
            else tma_load_4d(st, &tmT, i0, ld_b0 * KB, ld_ja, ld_jb, bar);
          }
#pragma unroll
          for (int s = 0; s < kMaxModes - 2; ++s)
            if (s < v.nslow) bulk_load(st + BT + s * BM, v.Us[s] + (int64_t)sidx[s] * g.ldu + c0, BM * 8u, bar);
        }
        if (new_slab) loaded_b0 = ld_b0;
        // advance to the next k-tile (j' fastest, then the i_q0 block)
        ++ld_git;
        if (++ld_jp == v.Jp) {
          ld_jp = 0;
          ++ld_b0;
        }
        if (++ld_ja == v.runA) {
          ld_ja = 0;
          ++ld_jb;
        }
        if (ld_jp == 0) ld_jb = 0;
#pragma unroll
        for (int s = 0; s < kMaxModes - 2; ++s) {
          if (s < v.nslow) {
            if (++sidx[s] < v.sdim[s]) break;
            sidx[s] = 0;
          }
        }
      }
    }
    return;
  }
  // consumers: the parts buffer (written at the end) may still be read by the previous grid
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" :::);

  // =========================== consumer warps 0..WM-1 ===========================
  const int gid = lane >> 2, tig = lane & 3;
  unsigned git = 0;  // tiles consumed by this CTA (ring slot + phase)
  for (int64_t u = u0; u < u1;) {
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

    int cmp_b0 = kt0 / v.Jp, cmp_jp = kt0 % v.Jp;
    const int nvalid_n = (v.In - i0 + 7) / 8;
    const bool full_n = nvalid_n >= NT;

    for (int kt = kt0; kt < kt1; ++kt) {
      const int slot = (int)(git % STAGES);
      mbar_wait(&full[slot], (git / STAGES) & 1u);
      if (warp_live) {
        const double* st = stage0 + (size_t)slot * stage_sz;
        const double* Bt = st;
        const double* Ss = st + BT;
        const double* ub = Ub + (cmp_b0 & 1) * (KB * BMP) + warp * 16 + gid;
        const int cl = warp * 16 + gid;
        double s0 = Ss[cl], s1 = Ss[cl + 8];
        for (int s = 1; s < v.nslow; ++s) {
          s0 *= Ss[s * BM + cl];
          s1 *= Ss[s * BM + cl + 8];
        }
        // A fragments of the whole k-tile: KRP^T(c, k) = U_q0(k, c) * S_{j'}(c)
        double a[KB / 4][2];
#pragma unroll
        for (int kk = 0; kk < KB / 4; ++kk) {
          const int kr = kk * 4 + tig;
          a[kk][0] = ub[kr * BMP] * s0;
          a[kk][1] = ub[kr * BMP + 8] * s1;
        }
        const int kvalid = v.Iq0 - cmp_b0 * KB;
        if (kvalid >= KB && full_n) {
          // interior tile: no predicates around the MMAs
#pragma unroll
          for (int kk = 0; kk < KB / 4; ++kk) {
            const int kr = kk * 4 + tig;
#pragma unroll
            for (int ni = 0; ni < NT; ++ni) {
              const double bb = KMAJOR ? Bt[(ni * 8 + gid) * BKP + kr] : Bt[kr * BNP + ni * 8 + gid];
              dmma_m8n8k4(acc[0][ni][0], acc[0][ni][1], a[kk][0], bb);
              dmma_m8n8k4(acc[1][ni][0], acc[1][ni][1], a[kk][1], bb);
            }
          }
        } else {
          // ragged edge: skip whole k4 steps / n8 tiles outside the tensor (warp-uniform)
#pragma unroll
          for (int kk = 0; kk < KB / 4; ++kk) {
            if (kk * 4 < kvalid) {
              const int kr = kk * 4 + tig;
#pragma unroll
              for (int ni = 0; ni < NT; ++ni) {
                if (ni < nvalid_n) {
                  const double bb = KMAJOR ? Bt[(ni * 8 + gid) * BKP + kr] : Bt[kr * BNP + ni * 8 + gid];
                  dmma_m8n8k4(acc[0][ni][0], acc[0][ni][1], a[kk][0], bb);
                  dmma_m8n8k4(acc[1][ni][0], acc[1][ni][1], a[kk][1], bb);
                }
              }
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      ++git;
      if (++cmp_jp == v.Jp) {
        cmp_jp = 0;
        ++cmp_b0;
      }
    }

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
#ifdef JK_TU_HOST

// Plain reduction of the partial pieces into a dense row-major M (stand-alone op only; the
// JK-CALS path reduces inside the epilogue instead).
__global__ void reduce_parts_kernel(const double* __restrict__ parts, const TileInfo* __restrict__ tinfo,
                                    int In, int C, int BN, int nMt, double* __restrict__ M, int64_t ldm,
                                    int BM = kBM) {
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
#endif
#ifdef JK_TU_HOST

// Materialised Khatri-Rao generation (a1 in SURVEY §8a): K(j, c) = prod_{m != n} U_m(i_m(j), c),
// row-major J x ldk. Each thread owns 4 consecutive columns and a run of kKrpRows consecutive j,
// advancing the mixed-radix index incrementally; stores are 32-byte vectors (st.global.v4.f64).
constexpr int kKrpRows = 16;  // r01 sweep: 4-8-16-64-256 rows per CTA -> 16 best (4.0-4.5 TB/s)
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
  // unrolled so that the factor-row loads of several rows are in flight at once (the loop is
  // otherwise one L2 round trip per 32-byte store); streaming (.cs) stores: K is not re-read here
  // S = product of the slower rest-mode rows (q >= 1), the same for I_fast consecutive rows:
  // formed once per j' and kept in registers, so a row reads one factor row (the fastest mode's)
  // instead of nrest -- half the L2 reads for 3-way tensors (r02). Same multiplication order as
  // forming the whole product per row (slowest mode first): bitwise-identical results.
  double s0 = 1.0, s1 = 1.0, s2 = 1.0, s3 = 1.0;
  bool need_s = true;
#pragma unroll 4
  for (int j = j0; j < j1; ++j) {
    if (need_s) {
      s0 = s1 = s2 = s3 = 1.0;
#pragma unroll
      for (int q = kMaxModes - 2; q >= 1; --q) {
        if (q < v.nrest) {
          const double* row = v.U[q] + (int64_t)idx[q] * ldu + c;
          if (full4) {
            double4 x = *reinterpret_cast<const double4*>(row);  // 32B-aligned (ldu % 4 == 0)
            s0 *= x.x; s1 *= x.y; s2 *= x.z; s3 *= x.w;
          } else {
            s0 *= row[0];
            if (c + 1 < C) s1 *= row[1];
            if (c + 2 < C) s2 *= row[2];
            if (c + 3 < C) s3 *= row[3];
          }
        }
      }
      need_s = false;
    }
    double r0 = s0, r1 = s1, r2 = s2, r3 = s3;
    {
      const double* row = v.U[0] + (int64_t)idx[0] * ldu + c;
      if (full4) {
        double4 x = *reinterpret_cast<const double4*>(row);
        r0 *= x.x; r1 *= x.y; r2 *= x.z; r3 *= x.w;
      } else {
        r0 *= row[0];
        if (c + 1 < C) r1 *= row[1];
        if (c + 2 < C) r2 *= row[2];
        if (c + 3 < C) r3 *= row[3];
      }
    }
    double* dst = K + (int64_t)j * ldk + c;
    if (full4) {
      asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(dst), "d"(r0), "d"(r1), "d"(r2), "d"(r3)
                   : "memory");
    } else {
      dst[0] = r0;
      if (c + 1 < C) dst[1] = r1;
      if (c + 2 < C) dst[2] = r2;
      if (c + 3 < C) dst[3] = r3;
    }
#pragma unroll
    for (int q = 0; q < kMaxModes - 1; ++q) {
      if (q < v.nrest) {
        if (++idx[q] < v.rdim[q]) break;
        idx[q] = 0;
        need_s = true;  // a slower index moves: new S
      }
    }
  }
}
#endif

}  // namespace jk
