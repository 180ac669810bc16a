// mttkrp_i8.cuh — EXPERIMENTAL stand-alone FP64-accurate MTTKRP from INT8 tcgen05 MMAs
// (the JK-CALS path under precision JKCALS_FP64_I8, and jkcals_mttkrp_i8).
//
//   M(i, c) = sum_j' S(j', c) * sum_iq0 T(i, iq0, j') U_q0(iq0, c)          (the KRP factorisation)
//
// Both operands of the inner product are split into 7 balanced base-128 digits with power-of-two
// scales (T per mode-n row i, U_q0 per column c): x = 2^e sum_s d_s 2^(-7(s+1)), |d_s| <= 64.
// Products of digits a, b with a + b = dg accumulate exactly (int32) in TMEM accumulator D_dg; per
// j' the drain warps fold sum_dg D_dg 2^(-14-7 dg) times S(j', c) into FP64 registers, and the
// scales 2^(e_T(i) + e_U(c)) are applied when the CTA's partial piece is written. One stream-K
// unit = (output tile, j'); K = I_q0 padded to 64 per unit (4 K64 ring steps for I_q0 = 200).
// Operands are precomputed by slice_t_i8_kernel / slice_u_i8_kernel into GEMM-friendly layouts:
//   Bsl[s][j'][i (InP)][k (KP)]  and  Asl[s][c (CP)][k (KP)]   (int8, k contiguous)
// and loaded per K64 ring step by 3-D TMA boxes (64 B, rows, 7 slices) with SWIZZLE_64B.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "mttkrp_tf32.cuh"

namespace jk {

constexpr int kI8S = 7;          // digits (slices) per operand
constexpr int kI8N = 64;         // UMMA N = rows i of an output tile (7 accumulators x 64 <= 512)
constexpr int kI8K = 64;         // K per ring step (64-byte SWIZZLE_64B rows; 2 UMMA K32 sub-steps)
constexpr int kI8Stages = 2;
constexpr int kI8Threads = 10 * 32;  // warp 0 TMA, warp 1 MMA, warps 2-9 drain (lane quadrant x column half)
constexpr int kI8DWarps = 8;
constexpr int64_t kI8MaxK = 65536;  // I_q0 bound for exact int32 diagonal sums (7 * 4096 * K < 2^31)
constexpr size_t kI8ABytes = (size_t)kI8S * 128 * kI8K;    // 28 KB
constexpr size_t kI8BBytes = (size_t)kI8S * kI8N * kI8K;   // 14 KB
constexpr size_t kI8StageBytes = kI8ABytes + kI8BBytes;
constexpr size_t kI8Smem = 1024 + kI8Stages * kI8StageBytes + 256;
// resident-A variant: when K = I_q0 fits kI8ResKS ring steps (KP <= 192), the CTA keeps the whole U_q0
// digit tile (KS x 56 KB) in shared memory across its j' units -- it is the same for every unit of
// an m-tile -- and streams only the T digits (B) through a 2-stage ring. This cuts the L2 -> SMEM
// traffic per unit from 294 KB to 98 KB (syn200) -- but with only 28 KB of B in flight per SM the
// ring is latency-bound and the variant measured ~6 % slower than streaming (opt-in).
constexpr int kI8ResKS = 3;
constexpr int kI8ResStages = 2;
constexpr size_t kI8SmemRes = 1024 + kI8ResKS * kI8ABytes + kI8ResStages * kI8BBytes + 256;
static_assert(kI8SmemRes <= 232448, "resident-A INT8 MTTKRP exceeds shared memory");
// cluster variant: a pair of CTAs (one thread-block cluster) works on the same (m-tile, j') units
// for two adjacent 64-row n-tiles (a 128-row "pair tile"); each CTA TMA-loads 4 of the (padded to
// 8) U_q0 digit slices and multicasts them into both CTAs' stages, so the A operand crosses L2
// once per pair: 56 KB instead of 84 KB of L2 -> SMEM traffic per pair and K step
constexpr size_t kI8ABytesClu = (size_t)8 * 128 * kI8K;  // 8 slice slots (slot 7: TMA zero fill)
constexpr size_t kI8StageBytesClu = kI8ABytesClu + kI8BBytes;
constexpr size_t kI8SmemClu = 1024 + kI8Stages * kI8StageBytesClu + 256;

__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

struct I8Geom {
  int nMt, nNt;      // output tiles: C / 128, I_n / 64 (padded)
  int Jp, KS;        // j' count, ring steps per unit (KP / kI8K)
  int Kq;            // real K = I_q0 (the K32 sub-steps wholly in the zero padding are skipped)
  int64_t units;     // nMt * nNt * Jp
  int InP;           // padded I_n (rows of a j' block of Bsl)
  int nslow;
  int sdim[kMaxModes - 2];
  const double* Us[kMaxModes - 2];  // slow modes' U (row-major rows x ldu)
  int64_t ldu;
  const int* eT;     // [InP] reference exponent of each row of T_(n) (the largest slab exponent)
  const int8_t* dS;  // [Jp][InP] slab exponent of (row i, j') relative to eT(i), <= 0 (T digits are
                     // scaled per (i, j') slab: a spike costs precision only in its own slab)
  const int* eU;     // [CP] column exponents of U_q0 (kI8Bad: the column holds a non-finite value)
#ifdef JKCALS_DEV_PROBES
  int probe;         // dev timing probe builds only (tools/i8_probe.py)
#endif
};

__device__ __forceinline__ uint64_t umma_desc_sw32(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(256u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)6u << 61);
}
__device__ __forceinline__ uint64_t umma_desc_i8(uint32_t saddr) {
  if constexpr (kI8K == 64)
    return umma_desc_sw64(saddr);
  else
    return umma_desc_sw32(saddr);
}
__device__ __forceinline__ uint32_t umma_idesc_i8(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
}
// kCol: A-operand collector usage (0 none, 1 fill, 2 use, 3 lastuse) -- one A digit slice is read
// from shared memory once and reused by the MMAs of its 7 - a diagonals (halves the smem reads)
template <int kCol>
__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (kCol == 1)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a),
                 "l"(b), "r"(idesc), "r"(acc));
  else if constexpr (kCol == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::use [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a),
                 "l"(b), "r"(idesc), "r"(acc));
  else if constexpr (kCol == 3)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a),
                 "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
                 "r"(acc));
}
// the 28 digit products of one K32 step, A slice a outer: D_{a+b} += A_a B_b
template <int a, int bb>
__device__ __forceinline__ void i8_products(uint32_t tmem, uint32_t a0, uint32_t b0, uint32_t idesc, bool first_k) {
  // a0 / b0 already include the K32 sub-step's byte offset inside the swizzle atom
  if constexpr (a < kI8S) {
    if constexpr (bb <= kI8S - 1 - a) {
      constexpr int last = kI8S - 1 - a;
      constexpr int col = last == 0 ? 0 : (bb == 0 ? 1 : (bb == last ? 3 : 2));
      umma_i8<col>(tmem + (a + bb) * kI8N, umma_desc_i8(a0 + a * 128 * kI8K), umma_desc_i8(b0 + bb * kI8N * kI8K),
                   idesc, (!first_k || a > 0) ? 1u : 0u);
      i8_products<a, bb + 1>(tmem, a0, b0, idesc, first_k);
    } else {
      i8_products<a + 1, 0>(tmem, a0, b0, idesc, first_k);
    }
  }
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// digits of x * 2^-e (|x 2^-e| <= 1/2): 7 balanced base-128 digits, most significant first
__device__ __forceinline__ void i8_digits(double x, int e, int8_t* d) {
  double r = ldexp(x, -e);
#pragma unroll
  for (int s = 0; s < kI8S; ++s) {
    r *= 128.0;
    const double q = rint(r);
    d[s] = (int8_t)q;
    r -= q;
  }
}
constexpr int kI8Bad = 0x7fffffff;   // column-exponent marker of a non-finite U_q0 column
constexpr int kI8ZeroSlab = -100000; // slab-exponent marker of an all-zero slab
__device__ __forceinline__ int i8_exponent(double m) {  // e with m * 2^-e <= 1/2
  if (!(m > 0.0)) return 0;
  int e;
  frexp(m, &e);  // m = f 2^e, f in [0.5, 1)
  return e + 1;
}

template <int kStages, bool kResA, bool kClu = false>
__global__ void __launch_bounds__(kI8Threads, 1)
    mttkrp_i8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, I8Geom g,
                     const TileInfo* __restrict__ tinfo, double* __restrict__ parts) {
  extern __shared__ __align__(1024) unsigned char ism[];
  constexpr size_t kStageB = kResA ? kI8BBytes : (kClu ? kI8StageBytesClu : kI8StageBytes);  // per ring stage
  constexpr size_t kAOff = kClu ? kI8ABytesClu : kI8ABytes;  // B offset inside a streaming stage
  unsigned char* ares = ism;                                       // resident A (kResA)
  unsigned char* stages = ism + (kResA ? kI8ResKS * kI8ABytes : 0);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kStages * kStageB);
  uint64_t* full = bars;
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* a_full = acc_empty + 1;   // resident A loaded
  uint64_t* a_empty = a_full + 1;     // resident A no longer read by the MMAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_empty + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // kClu: the plan's "CTA" is the cluster (pair tile rows = 2 x kI8N); crk = this CTA's half
  const int crk = kClu ? (int)cluster_ctarank() : 0;
  const int b = kClu ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int* cta_u = reinterpret_cast<const int*>(tinfo + g.nMt * g.nNt);
  const int64_t u0 = cta_u[b], u1 = cta_u[b + 1];
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kClu ? 2 : 1);  // kClu: both CTAs' MMAs must be done with the stage
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, kI8DWarps);
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (kClu)
    cluster_sync_all();  // the peer's barriers are initialised before any multicast reaches them
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int KT = g.Jp;  // units per tile

  if (warp == 0) {
    // ---------------- TMA producer: per unit, KS steps of (A box, B box), each all 7 slices
    unsigned it = 0, na = 0;
    int cur_tm = -1;
    for (int64_t u = u0; u < u1; ++u) {
      const int t = (int)(u / KT), jp = (int)(u % KT);
      const int tm = t % g.nMt, tn = t / g.nMt;
      if (kResA && tm != cur_tm) {  // (re)load the m-tile's U_q0 digits once
        if (na >= 1) mbar_wait_safe(a_empty, (na - 1) & 1u);
        if (elect_one()) {
          mbar_expect_tx(a_full, (unsigned)(g.KS * kI8ABytes));
          for (int ks = 0; ks < g.KS; ++ks) tma_load_3d(ares + ks * kI8ABytes, &tmA, ks * kI8K, tm * 128, 0, a_full);
        }
        __syncwarp();
        ++na;
        cur_tm = tm;
      }
      for (int ks = 0; ks < g.KS; ++ks, ++it) {
        const int slot = (int)(it % kStages);
        if (it >= (unsigned)kStages) mbar_wait_safe(&empty[slot], ((it / kStages) - 1) & 1u);
        if (elect_one()) {
          unsigned char* st = stages + slot * kStageB;
          mbar_expect_tx(&full[slot], (unsigned)kStageB);
          if (kClu) {  // my 4 slice slots of A to both CTAs, my own n-tile of B
            tma_load_3d_mc(st + crk * 4 * 128 * kI8K, &tmA, ks * kI8K, tm * 128, crk * 4, &full[slot], (uint16_t)3);
            tma_load_3d(st + kAOff, &tmB, ks * kI8K, jp * g.InP + (2 * tn + crk) * kI8N, 0, &full[slot]);
          } else {
            if (!kResA) tma_load_3d(st, &tmA, ks * kI8K, tm * 128, 0, &full[slot]);
            tma_load_3d(st + (kResA ? 0 : kI8ABytes), &tmB, ks * kI8K, jp * g.InP + tn * kI8N, 0, &full[slot]);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: 28 digit products per K32 step into the 7 diagonal accumulators
    const uint32_t idesc = umma_idesc_i8(kI8N);
    unsigned it = 0, un = 0, na = 0;
    int cur_tm = -1;
    for (int64_t u = u0; u < u1; ++u, ++un) {
      const int tm = (int)((u / KT) % g.nMt);
      if (un >= 1) mbar_wait_safe(acc_empty, (un - 1) & 1u);  // the drain has read the previous unit
      if (kResA && tm != cur_tm) {
        mbar_wait_safe(a_full, na & 1u);
        ++na;
        cur_tm = tm;
      }
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const bool a_last = kResA && (u + 1 == u1 || (int)(((u + 1) / KT) % g.nMt) != tm);
      for (int ks = 0; ks < g.KS; ++ks, ++it) {
        const int slot = (int)(it % kStages);
        mbar_wait_safe(&full[slot], (it / kStages) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t st = smem_u32(stages + slot * kStageB);
        const uint32_t a0 = kResA ? smem_u32(ares + ks * kI8ABytes) : st;
        const uint32_t b0 = kResA ? st : st + (uint32_t)kAOff;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kI8K / 32; ++kk) {
            if (kk > 0 && ks * kI8K + kk * 32 >= g.Kq) break;  // all-zero K32 sub-step of the padding
#ifdef JKCALS_DEV_PROBES  // timing probe builds only: one digit product per K32 step (wrong results)
            if (g.probe == 2)
              umma_i8<0>(tmem, umma_desc_i8(a0 + kk * 32), umma_desc_i8(b0 + kk * 32), idesc, (ks | kk) ? 1u : 0u);
            else
#endif
              i8_products<0, 0>(tmem, a0 + kk * 32, b0 + kk * 32, idesc, ks == 0 && kk == 0);
          }
          if (kClu)
            umma_commit_mc(&empty[slot], (uint16_t)3);  // frees the stage in both CTAs
          else
            umma_commit(&empty[slot]);
          if (ks == g.KS - 1) {
            umma_commit(acc_full);
            if (a_last) umma_commit(a_empty);  // the next unit needs another m-tile's A
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- drain warps: TMEM lane quadrant q <-> fused columns 32q..32q+31 of the tile
    // (a warp may only read the TMEM lanes of its own quadrant, warp % 4); each of the two warps of
    // a quadrant folds one 32-column half of the N = 64 accumulator columns
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int cl = q * 32 + lane;
    double acc[kI8N / 2];
#pragma unroll
    for (int i = 0; i < kI8N / 2; ++i) acc[i] = 0.0;
    unsigned un = 0;
    int64_t seg_t = -1;
    auto flush = [&](int64_t t) {  // write this CTA's piece of tile t (its column half), with the scales
      const int tm = (int)(t % g.nMt), tn = (int)(t / g.nMt);
      const TileInfo ti = tinfo[t];
      constexpr int kBN = kClu ? 2 * kI8N : kI8N;  // rows of a plan tile
      double* P = parts + ((int64_t)ti.piece_base + (b - ti.first_cta)) * (int64_t)(kBN * 128) + cl;
      const int eu = g.eU[tm * 128 + cl];
#pragma unroll
      for (int i = 0; i < kI8N / 2; ++i) {
        const int il = crk * kI8N + h * (kI8N / 2) + i;
        // a non-finite U_q0 column yields NaN, as the FP64 path would (the epilogue flags it)
        P[(int64_t)il * 128] = (eu == kI8Bad) ? __longlong_as_double(0x7ff8000000000000LL)
                                              : ldexp(acc[i], eu + g.eT[tn * kBN + il]);
        acc[i] = 0.0;
      }
    };
    for (int64_t u = u0; u < u1; ++u, ++un) {
      const int64_t t = u / KT;
      const int jp = (int)(u % KT);
      if (seg_t >= 0 && t != seg_t) flush(seg_t);
      seg_t = t;
      const int c = (int)(t % g.nMt) * 128 + cl;
      // this thread's 32 rows: their slab exponents relative to the row reference (broadcast loads)
      uint4 dsw[2];
      {
        constexpr int kBNr = kClu ? 2 * kI8N : kI8N;
        const int tn = (int)(t / g.nMt);
        const uint4* dp = reinterpret_cast<const uint4*>(g.dS + (int64_t)jp * g.InP + tn * kBNr + crk * kI8N +
                                                          h * (kI8N / 2));
        dsw[0] = __ldg(dp);
        dsw[1] = __ldg(dp + 1);
      }
      // S(j', c) = prod of the slow modes' rows (FP64, from L2; overlaps this unit's MMAs)
      double s = 1.0;
      {
        int rem = jp;
        for (int m = 0; m < g.nslow; ++m) {
          const int idx = rem % g.sdim[m];
          rem /= g.sdim[m];
          s *= g.Us[m][(int64_t)idx * g.ldu + c];
        }
      }
      mbar_wait_safe(acc_full, un & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#ifdef JKCALS_DEV_PROBES  // timing probe builds only: drain skipped (wrong results)
      if (g.probe == 1) {
        acc[0] += s;
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
        continue;
      }
#endif
      const uint32_t lb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * (kI8N / 2));
#pragma unroll
      for (int cg = 0; cg < kI8N / 2; cg += 16) {
        // all 7 diagonals of these 16 columns in flight, one wait
        uint32_t r[kI8S][16];
#pragma unroll
        for (int dg = 0; dg < kI8S; ++dg)
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
              : "=r"(r[dg][0]), "=r"(r[dg][1]), "=r"(r[dg][2]), "=r"(r[dg][3]), "=r"(r[dg][4]), "=r"(r[dg][5]),
                "=r"(r[dg][6]), "=r"(r[dg][7]), "=r"(r[dg][8]), "=r"(r[dg][9]), "=r"(r[dg][10]), "=r"(r[dg][11]),
                "=r"(r[dg][12]), "=r"(r[dg][13]), "=r"(r[dg][14]), "=r"(r[dg][15])
              : "r"(lb + (uint32_t)(dg * kI8N + cg)));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (cg + 16 == kI8N / 2) {
          // the accumulators are all in registers: release TMEM to the next unit's MMAs before the
          // last chunk's recombination (overlaps it with the MMA stream)
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          // exact integer recombination of the diagonals (|D_dg| < 2^31, K <= kI8MaxK):
          //   hi = D0 2^21 + D1 2^14 + D2 2^7 + D3 (< 2^50),  lo = D4 2^14 + D5 2^7 + D6 (< 2^46),
          // each converted exactly by the 1.5 * 2^52 bias trick (no I2F), one rounding in the fma
          const int64_t hi = (int64_t)(int)r[0][i] * (1 << 21) + (int64_t)(int)r[1][i] * (1 << 14) +
                             (int64_t)(int)r[2][i] * (1 << 7) + (int64_t)(int)r[3][i];
          const int64_t lo = (int64_t)(int)r[4][i] * (1 << 14) + (int64_t)(int)r[5][i] * (1 << 7) + (int64_t)(int)r[6][i];
          const double hd = __longlong_as_double(hi + 0x4338000000000000LL) - 6755399441055744.0;
          const double ld = __longlong_as_double(lo + 0x4338000000000000LL) - 6755399441055744.0;
          const double v = fma(ld, 0x1p-56, hd * 0x1p-35);  // D_dg carries 2^(-14 - 7 dg)
          // 2^(e_S(i, j') - e_T(i)) built from its exponent bits (exact; -126 <= d <= 0)
          const int row = cg + i;
          const uint32_t wd = (row < 16) ? ((row < 8) ? ((row < 4) ? dsw[0].x : dsw[0].y) : ((row < 12) ? dsw[0].z : dsw[0].w))
                                         : ((row < 24) ? ((row < 20) ? dsw[1].x : dsw[1].y) : ((row < 28) ? dsw[1].z : dsw[1].w));
          const int dsl = (int)(int8_t)(wd >> (8 * (row & 3)));
          const double sc = __longlong_as_double((long long)(1023 + dsl) << 52);
          acc[cg + i] = fma(s * sc, v, acc[cg + i]);
        }
      }
    }
    if (seg_t >= 0) flush(seg_t);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
  if (kClu) cluster_sync_all();  // no multicast or remote arrive may target an exited peer
}

#ifdef JK_TU_HOST
// ---- operand preparation -----------------------------------------------------------------
// slab exponents of T_(n): e_S(i, j') with max_k |T(i, k, j')| 2^-e <= 1/2 (kI8ZeroSlab for an
// all-zero slab); one thread per (j', i), k = i_q0 the contraction index
__global__ void slab_exp_t_kernel(const double* __restrict__ T, int N, const int64_t* __restrict__ st_dev,
                                  const int* __restrict__ dims_dev, int n, int q0, int In, int InP, int Iq0,
                                  int64_t Jp, int* __restrict__ eS) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= Jp * InP) return;
  const int64_t jp = e / InP;
  const int i = (int)(e % InP);
  int ex = kI8ZeroSlab;
  if (i < In) {
    int64_t rem = jp, off = (int64_t)i * st_dev[n];
    for (int m = 0; m < N; ++m) {
      if (m == n || m == q0) continue;
      off += (rem % dims_dev[m]) * st_dev[m];
      rem /= dims_dev[m];
    }
    double mx = 0.0;
    for (int k = 0; k < Iq0; ++k) mx = fmax(mx, fabs(T[off + (int64_t)k * st_dev[q0]]));
    if (mx > 0.0) ex = i8_exponent(mx);
  }
  eS[e] = ex;
}

// row reference exponents e_T(i) = max_j' e_S(i, j') and the relative slab exponents
// dS = e_S - e_T in [-126, 0] (an all-zero slab, or one 126+ binades below its row, is -126: its
// digits are all zero or its contribution is below 2^-126 of the row's largest)
__global__ void row_ref_exp_kernel(const int* __restrict__ eS, int InP, int64_t Jp, int* __restrict__ eT,
                                   int8_t* __restrict__ dS) {
  const int i = blockIdx.x;
  int m = kI8ZeroSlab;
  for (int64_t jp = threadIdx.x; jp < Jp; jp += blockDim.x) m = max(m, eS[jp * InP + i]);
  __shared__ int red[256];
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = max(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  const int ref = red[0] == kI8ZeroSlab ? 0 : red[0];
  if (threadIdx.x == 0) eT[i] = ref;
  for (int64_t jp = threadIdx.x; jp < Jp; jp += blockDim.x) {
    const int es = eS[jp * InP + i];
    dS[jp * InP + i] = (int8_t)(es == kI8ZeroSlab ? -126 : max(-126, es - ref));
  }
}

// Bsl[s][j'][i][k] = digit s of T(i_n = i, i_q0 = k, j') * 2^-e_S(i, j'); zero padding outside
__global__ void slice_t_i8_kernel(const double* __restrict__ T, int N, const int64_t* __restrict__ st_dev,
                                  const int* __restrict__ dims_dev, int n, int q0, int In, int InP, int Iq0, int KP,
                                  int64_t Jp, const int* __restrict__ eS, int8_t* __restrict__ B) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)InP * KP;
  if (e >= Jp * per) return;
  const int64_t jp = e / per;
  const int i = (int)((e % per) / KP), k = (int)(e % KP);
  int8_t d[kI8S] = {0, 0, 0, 0, 0, 0, 0};
  if (i < In && k < Iq0) {
    int64_t rem = jp, off = (int64_t)i * st_dev[n] + (int64_t)k * st_dev[q0];
    for (int m = 0; m < N; ++m) {
      if (m == n || m == q0) continue;
      off += (rem % dims_dev[m]) * st_dev[m];
      rem /= dims_dev[m];
    }
    const int es = eS[jp * InP + i];
    if (es != kI8ZeroSlab) i8_digits(T[off], es, d);
  }
  const int64_t slice = Jp * per;
#pragma unroll
  for (int s = 0; s < kI8S; ++s) B[(int64_t)s * slice + e] = d[s];
}

// column exponents of U_q0 and Asl[s][c][k] = digit s of U_q0(k, c) * 2^-e_U(c)
// 32 columns x 8 row groups per 256-thread block: coalesced along c, max-reduced across the groups
__global__ void __launch_bounds__(256) col_exp_u_kernel(const double* __restrict__ U, int64_t ldu, int rows, int C,
                                                        int CP, int* __restrict__ eU) {
  __shared__ double red[8][32];
  const int cx = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cx;
  double m = 0.0;
  if (c < C)
    for (int k = ry; k < rows; k += 8) {
      const double x = fabs(U[(int64_t)k * ldu + c]);
      m = (x <= 1.7976931348623157e308) ? fmax(m, x) : __longlong_as_double(0x7ff0000000000000LL);  // NaN/Inf -> Inf
    }
  red[ry][cx] = m;
  __syncthreads();
  if (ry == 0 && c < CP) {
#pragma unroll
    for (int r = 1; r < 8; ++r) m = fmax(m, red[r][cx]);
    eU[c] = isinf(m) ? kI8Bad : i8_exponent(m);
  }
}
__global__ void slice_u_i8_kernel(const double* __restrict__ U, int64_t ldu, int rows, int C, int CP, int KP,
                                  const int* __restrict__ eU, int8_t* __restrict__ A) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)CP * KP) return;
  const int c = (int)(e / KP), k = (int)(e % KP);
  int8_t d[kI8S] = {0, 0, 0, 0, 0, 0, 0};
  if (c < C && k < rows && eU[c] != kI8Bad) i8_digits(U[(int64_t)k * ldu + c], eU[c], d);
  const int64_t slice = (int64_t)CP * KP;
#pragma unroll
  for (int s = 0; s < kI8S; ++s) A[(int64_t)s * slice + e] = d[s];
}

#endif  // JK_TU_HOST

}  // namespace jk
