// mttkrp_tf32.cuh — the FP32 path of the fused KRP + MTTKRP on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), FP32-accurate via the 3xTF32 split.
//
// Same product as mttkrp.cuh (Alg. 3 alg:cals_jk:mttkrp; Eq. 1):
//     D[c][i] = sum_j KRP(j, c) * T_(n)(i, j)   (M = fused columns c, N = I_n, K = J_n)
// Every operand x is split x = hi + lo with hi = x truncated to TF32 (10-bit mantissa) and
// lo = x - hi, and D += A_hi B_hi^T + A_hi B_lo^T + A_lo B_hi^T (the lo*lo term is below FP32
// rounding) — "3xTF32", which a single TF32 pass would fail (1.5e-4 > 1e-4).
//
// Roles (one CTA per SM, 14 warps):
//   warps 0-7   A producers: build the KRP^T tile of a k-tile in shared memory, already split into
//               hi/lo and laid out in the UMMA K-major SWIZZLE_64B canonical layout, from the
//               U_q0 slab (TMA) scaled by the S_{j'} rows (bulk copies) -- the KRP never hits HBM.
//   warps 8-11  drain: per FP32 accumulation chain, tcgen05.ld of the TMEM accumulator (one lane
//               quadrant each) added into the FP64 partial piece read by the FP64 path's epilogue.
//   warp 12     TMA producer (one lane): T_hi / T_lo boxes (4-D tensor maps, 64-B swizzle), the
//               S rows and the U_q0 slab, on the stage's mbarriers.
//   warp 13     MMA issuer (one lane): 3 x (16/8) tcgen05.mma per j' sub-tile, tcgen05.commit to
//               the stage's `empty` barrier and, per chain, to `acc_full`.
// Variants (r02): PAIR -- a 2-CTA cluster on a 256-column super tile with cta_group::2 MMAs
// (M = 256), each CTA holding half of the T tile; JM -- 1, 2 or 4 j' values per k-tile, to
// amortise the ring handshakes on narrow tiles.
// T is stored as FP32 hi/lo copies (built once at create): the original layout for n >= 1
// (i_0 contiguous) and a mode-(1,0,2,..) permuted copy for n = 0 so that B is always K-major.
#pragma once
#ifdef JKCALS_DEV_PROBES
#include <cstdio>
#endif
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "mttkrp.cuh"

namespace jk {

constexpr int kTfBK = 16;         // k (i_q0 values) per stage: one 64-byte swizzle atom of fp32
constexpr int kTfAWarps = 8;      // A producers: thread = (row of the A tile, half of the k-tile)
constexpr int kTfDWarps = 4;      // TMEM drain warps (8..11: lane quadrants warp % 4)
constexpr int kTfThreads = (kTfAWarps + kTfDWarps + 2) * 32;
constexpr int kTfTmaWarp = kTfAWarps + kTfDWarps, kTfMmaWarp = kTfTmaWarp + 1;
constexpr int kTfMaxN = 256;      // UMMA N (fp32 accumulator columns) per output tile
constexpr uint32_t kTfTmemCols = 512;  // two accumulator buffers of kTfMaxN columns
// FP32 accumulation chains are cut every kTfChunk k-tiles (128 products x 3): the TMEM buffer is
// drained into the FP64 partial piece while the MMAs continue in the other buffer.
constexpr int kTfChunk = 8;  // r02: 48 left the fluorescence-shaped eem R5 at 2.2e-4 (bar 1e-4), 16 at 1.2e-4 (lambda, full size)
constexpr int kTfMaxStages = 8;

struct TfGeom {
  int C;          // fused width in use
  int64_t ldu;    // pitch of the FP64 multi-factors (multiple of 128)
  int nMt, nNt;   // output tiles (C / 128 -- C / 256 super tiles when paired --, I_n / BN)
  int nMt1;       // 128-column tiles per tile row (the piece table; = nMt unless paired)
  int BN;         // UMMA N of an output tile (multiple of 16, <= 256)
  int KT;         // k-tiles per output tile (nb0 * J')
  int64_t units;
  int G;
  int stages;     // shared-memory ring depth (as many as fit, <= kTfMaxStages)
  int chunk;      // k-tiles per FP32 accumulation chain (kTfChunk / jm unless tuned)
  int jm;         // j' values per k-tile (1, 2 or 4): a k-tile is 16 i_q0 x jm j' (r02)
  int probe;      // dev timing probe builds only (JKCALS_DEV_PROBES)
};

// one ring stage = jm sub-tiles of {A_hi, A_lo (128 x 64 B each), B_hi, B_lo (BN x 64 B), S rows}
__host__ __device__ constexpr size_t tf_stage_bytes(int BN, int nslow, int jm = 1) {
  return (size_t)jm * (2u * 128u * 64u + 2u * (size_t)BN * 64u + (size_t)nslow * kBM * 8u);
}
__host__ __device__ constexpr size_t tf_slab_bytes() { return 2ull * kBK * kBMP * 8ull; }
// drain staging: two buffers of 16 TMEM columns x 128 lanes in FP64 ([16 rows i][128 columns c])
constexpr size_t kTfStgBytes = 2u * 16u * 128u * 8u;
__host__ __device__ constexpr size_t tf_smem_bytes(int BN, int nslow, int stages, int jm = 1) {
  // 1 KB alignment slack + drain staging + slab + stages + barriers (4 per stage + 4) + TMEM address
  return 1024 + kTfStgBytes + tf_slab_bytes() + stages * tf_stage_bytes(BN, nslow, jm) + (4 * stages + 4) * 8 + 16;
}
// bulk (TMA-engine) moves of a drained FP64 block into the partial piece: plain copy for the first
// chain of a segment, f64 add (UBLKRED.ADD.F64) for the next ones -- no L2 round trip on the drain
__device__ __forceinline__ void bulk_store_f64(double* dst, const void* src, unsigned bytes, bool add) {
  if (add)
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
  else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void drain_bar() {  // the 4 drain warps only (named barrier 1)
  asm volatile("bar.sync 1, %0;\n" ::"n"(kTfDWarps * 32) : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_64B, 8-row groups of 64-byte rows (SBO 512 B)
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(512u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)4u << 61);
}
// instruction descriptor: D fp32, A/B tf32, both K-major, M = 128, N = BN
__device__ __forceinline__ uint32_t umma_idesc_tf32(int BN, uint32_t M = 128) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
// mbarrier wait that traps (illegal-instruction error) instead of spinning forever if the
// barrier never completes -- a protocol bug must not hang the GPU
__device__ __forceinline__ void mbar_wait_safe(uint64_t* bar, unsigned parity) {
  uint32_t done = 0;
  for (uint64_t it = 0; it < (1ull << 26); ++it) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
  }
  __trap();
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// ---- CTA-pair (cta_group::2) helpers
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t smem_peer(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// arrive on an mbarrier given by its shared::cluster address (default .release.cta semantics: the
// data it publishes -- A tiles after fence.proxy.async, drained TMEM -- is consumed by the tensor
// core through the async proxy, not by generic loads of the peer, so no cluster-scope release is
// needed; r02: .release.cluster compiled to MEMBAR.ALL.GPU per arrive and the acquire.cluster wait
// to CCTL.IVALL, making the pair kernel 1.8x slower than the one-CTA kernel)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cbar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cbar) : "memory");
}
// TMA of one CTA's half of a paired operand; completion is counted on the LEADER's barrier
__device__ __forceinline__ void tma_load_4d_pair(void* dst, const CUtensorMap* tm, int x0, int x1, int x2, int x3,
                                                 uint32_t leader_bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// commit the pair's MMAs to the barrier at the same offset in both CTAs
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ uint32_t tf32_trunc(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

template <int NSTEP>  // 32 lanes x NSTEP fp32 columns
__device__ __forceinline__ void tmem_ld_32x32b(uint32_t taddr, float* v) {
  static_assert(NSTEP == 16, "");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}

// PAIR: a CTA pair (2-CTA cluster, cta_group::2) computes a 256-column super tile -- UMMA M = 256,
// each CTA builds its own 128 columns of A and TMA-loads HALF of the T tile's rows (B), and the
// leader's single MMA thread reads both halves: the shared-memory operand traffic per SM drops
// from (A + B) to (A + B/2) per MMA. Pieces stay per 128-column tile (CTA rank r writes tile
// 2 * tm2 + r), so the epilogue is unchanged.
template <int kTfStages, bool PAIR = false, int JMT = 1>
__global__ void __launch_bounds__(kTfThreads, 1)
    mttkrp_tf32_kernel(const __grid_constant__ CUtensorMap tmThi, const __grid_constant__ CUtensorMap tmTlo,
                       const __grid_constant__ CUtensorMap tmU, MttkrpView v, TfGeom g,
                       const TileInfo* __restrict__ tinfo, double* __restrict__ parts) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  unsigned char* base = tsm;  // dynamic smem is 1 KB aligned (__align__(1024) on the declaration)
  double* stg = reinterpret_cast<double*>(base);                                  // drain staging
  double* Ub = reinterpret_cast<double*>(base + kTfStgBytes);                      // [2][BK][BMP] fp64
  unsigned char* stages = base + kTfStgBytes + tf_slab_bytes();
  const int BNl = PAIR ? g.BN / 2 : g.BN;  // rows of the T tile held by this CTA
  constexpr int JM = JMT;                    // j' per k-tile (compile-time: loops unrolled)
  const int KTJ = (v.Jp + JM - 1) / JM;       // k-tiles per i_q0 block
  const size_t stage_sz = tf_stage_bytes(BNl, v.nslow, JM);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kTfStages * stage_sz);
  uint64_t* fullB = bars;                      // TMA data landed (count 1 + tx)
  uint64_t* fullA = bars + kTfStages;          // A tile written (count kTfAWarps)
  uint64_t* empty = bars + 2 * kTfStages;      // MMAs of the stage done (tcgen05.commit)
  uint64_t* acc_full = bars + 3 * kTfStages;   // [2] accumulator buffer holds a finished chunk
  uint64_t* acc_empty = acc_full + 2;          // [2] accumulator buffer drained
  uint64_t* fullS = acc_empty + 2;             // [STAGES] S rows (+ U_q0 slab) landed: A may start
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fullS + kTfStages);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int crk = PAIR ? (int)cluster_ctarank() : 0;
  const bool leader = crk == 0;
  const int b = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;  // the plan's CTA (a pair when PAIR)
  const int nMt1 = PAIR ? g.nMt1 : g.nMt;  // 128-column tiles per tile row (the piece table)
  const int* cta_u = reinterpret_cast<const int*>(tinfo + nMt1 * g.nNt);
  const int64_t u0 = cta_u[b], u1 = cta_u[b + 1];
  const int BN = g.BN;

  // stage layout: A_hi[JM] | A_lo[JM] | B_hi[JM] | B_lo[JM] | S[JM][nslow][128] (sub-tile jj of a
  // stage is j' = jp0 + jj; every sub-tile base is a multiple of 512 B, the SWIZZLE_64B period)
  auto stA_hi = [&](int s, int jj) { return stages + s * stage_sz + (size_t)jj * 8192; };
  auto stA_lo = [&](int s, int jj) { return stages + s * stage_sz + (size_t)(JM + jj) * 8192; };
  auto stB_hi = [&](int s, int jj) { return stages + s * stage_sz + (size_t)JM * 16384 + (size_t)jj * BNl * 64; };
  auto stB_lo = [&](int s, int jj) {
    return stages + s * stage_sz + (size_t)JM * 16384 + (size_t)(JM + jj) * BNl * 64;
  };
  auto stS = [&](int s, int jj) {
    return reinterpret_cast<double*>(stages + s * stage_sz + (size_t)JM * 16384 + (size_t)2 * JM * BNl * 64 +
                                     (size_t)jj * v.nslow * kBM * 8);
  };

  if (tid == 0) {
    for (int s = 0; s < kTfStages; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&fullS[s], 1);
      mbar_init(&fullA[s], PAIR ? 2 * kTfAWarps : kTfAWarps);  // (PAIR: both CTAs' A warps)
      mbar_init(&empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&acc_full[q], 1);
      mbar_init(&acc_empty[q], PAIR ? 2 * kTfDWarps : kTfDWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (PAIR) {
    __syncthreads();
    cluster_sync_all();  // the peer's barriers are initialised before any remote arrive / commit
  }
  if (warp == 0) {  // TMEM accumulator: 128 lanes x 256 fp32 columns (x 2 CTAs when PAIR)
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                   "n"(kTfTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                   "n"(kTfTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" :::);

  if (warp == kTfTmaWarp) {
    // ======================= TMA producer (whole warp walks the loop, one elected lane issues) ===
    {
      const unsigned s_bytes = (unsigned)v.nslow * kBM * 8u;
      const unsigned t_bytes = 2u * (unsigned)BNl * 64u;  // this CTA's B bytes per stage
      unsigned ld_git = 0;
      for (int64_t u = u0; u < u1;) {
        const int t = (int)(u / g.KT);
        const int kt0 = (int)(u % g.KT);
        const int64_t kt_end = (int64_t)kt0 + (u1 - u);
        const int kt1 = (int)(kt_end < (int64_t)g.KT ? kt_end : (int64_t)g.KT);
        u += kt1 - kt0;
        const int tm = t % g.nMt, tn = t / g.nMt;
        const int c0 = (PAIR ? 2 * tm + crk : tm) * kBM, i0 = tn * BN + crk * BNl;
        for (unsigned q = (ld_git >= (unsigned)kTfStages ? ld_git - kTfStages + 1 : 0); q < ld_git; ++q)
          mbar_wait_safe(&empty[q % kTfStages], (q / kTfStages) & 1u);
        int loaded_b0 = -1;
        // running j' state (divisions only at a segment start: a per-k-tile div/mod chain in
        // this single issuing lane made the TMA loop the bottleneck)
        int ld_b0 = kt0 / KTJ, ld_jp = (kt0 % KTJ) * JM;
        int ld_ja = ld_jp % v.runA, ld_jb = ld_jp / v.runA;
        int sidx[kMaxModes - 2];
        {
          int rem = ld_jp;
#pragma unroll
          for (int q = 0; q < kMaxModes - 2; ++q)
            if (q < v.nslow) { sidx[q] = rem % v.sdim[q]; rem /= v.sdim[q]; }
        }
#pragma unroll 1
        for (int kt = kt0; kt < kt1; ++kt) {
          const int nv = v.Jp - ld_jp < JM ? v.Jp - ld_jp : JM;  // j' sub-tiles of this k-tile
          const int slot = (int)(ld_git % kTfStages);
          if (ld_git >= (unsigned)kTfStages) mbar_wait_safe(&empty[slot], ((ld_git / kTfStages) - 1) & 1u);
          uint64_t* bar = &fullB[slot];
          const bool new_slab = (ld_b0 != loaded_b0);
          if (new_slab && KTJ < kTfStages - 1) {  // short i_q0 blocks: drain before reusing a slab buffer
            for (unsigned q = (ld_git >= (unsigned)kTfStages ? ld_git - kTfStages + 1 : 0); q < ld_git; ++q)
              mbar_wait_safe(&empty[q % kTfStages], (q / kTfStages) & 1u);
          }
          uint64_t* sbar = &fullS[slot];
          if (elect_one()) {
            // the A producers only need the slow-mode rows and the U_q0 slab: their own barrier
            mbar_expect_tx(sbar, (unsigned)nv * s_bytes + (new_slab ? (unsigned)(kBK * kBMP * 8) : 0u));
            if (new_slab) tma_load_2d(Ub + (ld_b0 & 1) * (kBK * kBMP), &tmU, c0, ld_b0 * kBK, sbar);
            // (c0s: the dead second half of an odd last super tile reads a valid row; unused)
            const int c0s = c0 < nMt1 * kBM ? c0 : c0 - kBM;
            {
              int si[kMaxModes - 2];  // slow-mode indices of j' = ld_jp + jj (mixed radix, Eq. 3)
#pragma unroll
              for (int q = 0; q < kMaxModes - 2; ++q) si[q] = sidx[q];
              for (int jj = 0; jj < JM && jj < nv; ++jj) {
#pragma unroll
                for (int q = 0; q < kMaxModes - 2; ++q)
                  if (q < v.nslow)
                    bulk_load(stS(slot, jj) + q * kBM, v.Us[q] + (int64_t)si[q] * g.ldu + c0s, kBM * 8u, sbar);
#pragma unroll
                for (int q = 0; q < kMaxModes - 2; ++q) {
                  if (q < v.nslow) {
                    if (++si[q] < v.sdim[q]) break;
                    si[q] = 0;
                  }
                }
              }
            }
            // view (q0, runA, n, runB) for every mode (the n = 0 view is the permuted copy)
#ifdef JKCALS_DEV_PROBES  // timing probe builds only: no T tiles (wrong results)
            if (g.probe == 3 || g.probe == 6) {
              if (!PAIR || leader) mbar_expect_tx(bar, 0);
            } else
#endif
            {
              // both halves of a pair complete on the leader's barrier; the leader expects both
              if (!PAIR || leader) mbar_expect_tx(bar, (unsigned)nv * (PAIR ? 2 * t_bytes : t_bytes));
              const uint32_t lb = PAIR ? smem_peer(bar, 0) : 0u;
              int ja = ld_ja, jb = ld_jb;
              for (int jj = 0; jj < JM && jj < nv; ++jj) {
                if (PAIR) {
                  tma_load_4d_pair(stB_hi(slot, jj), &tmThi, ld_b0 * kTfBK, ja, i0, jb, lb);
                  tma_load_4d_pair(stB_lo(slot, jj), &tmTlo, ld_b0 * kTfBK, ja, i0, jb, lb);
                } else {
                  tma_load_4d(stB_hi(slot, jj), &tmThi, ld_b0 * kTfBK, ja, i0, jb, bar);
                  tma_load_4d(stB_lo(slot, jj), &tmTlo, ld_b0 * kTfBK, ja, i0, jb, bar);
                }
                if (++ja == v.runA) {
                  ja = 0;
                  ++jb;
                }
              }
            }
          }
          __syncwarp();
          if (new_slab) loaded_b0 = ld_b0;
          ++ld_git;
          // advance the running j' state by the nv j' of this k-tile (every lane, uniformly)
          for (int jj = 0; jj < JM && jj < nv; ++jj) {
            if (++ld_ja == v.runA) {
              ld_ja = 0;
              ++ld_jb;
            }
#pragma unroll
            for (int q = 0; q < kMaxModes - 2; ++q) {
              if (q < v.nslow) {
                if (++sidx[q] < v.sdim[q]) break;
                sidx[q] = 0;
              }
            }
          }
          ld_jp += nv;
          if (ld_jp == v.Jp) {  // next i_q0 block: j' restarts at 0
            ld_jp = 0;
            ++ld_b0;
            ld_ja = ld_jb = 0;
#pragma unroll
            for (int q = 0; q < kMaxModes - 2; ++q) sidx[q] = 0;
          }
        }
      }
    }
  } else if (warp == kTfMmaWarp) {
    // ======================= MMA issuer (whole warp walks the loop, one elected lane issues) ===
    // (PAIR: the leader CTA's warp issues for both; the peer's MMA warp idles)
    if (leader) {
      const uint32_t idesc = umma_idesc_tf32(BN, PAIR ? 256u : 128u);
      unsigned git = 0, gc = 0;  // k-tiles consumed, chunks issued (accumulator buffer = gc & 1)
#ifdef JKCALS_DEV_PROBES
      long long pw_b = 0, pw_a = 0, pw_t0 = clock64();
#endif
      for (int64_t u = u0; u < u1;) {
        const int kt0 = (int)(u % g.KT);
        const int64_t kt_end = (int64_t)kt0 + (u1 - u);
        const int kt1 = (int)(kt_end < (int64_t)g.KT ? kt_end : (int64_t)g.KT);
        u += kt1 - kt0;
        bool first = true;
        uint32_t dacc = tmem;
        int cmp_b0 = kt0 / KTJ, cmp_g = kt0 % KTJ;  // running (i_q0 block, j' group)
        for (int kt = kt0; kt < kt1; ++kt) {
          const int cpos = (kt - kt0) % g.chunk;
          if (cpos == 0) {  // new chunk: its accumulator buffer must have been drained
            if (gc >= 2) {
              mbar_wait_safe(&acc_empty[gc & 1], ((gc >> 1) - 1) & 1u);
            }
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            dacc = tmem + (gc & 1) * kTfMaxN;
            first = true;
          }
          const int slot = (int)(git % kTfStages);
#ifdef JKCALS_DEV_PROBES  // phase clocks of the MMA warp (probe 5: printed by CTA 0 at the end)
          long long pc0 = clock64();
#endif
          mbar_wait_safe(&fullB[slot], (git / kTfStages) & 1u);
#ifdef JKCALS_DEV_PROBES
          long long pc1 = clock64();
#endif
          mbar_wait_safe(&fullA[slot], (git / kTfStages) & 1u);
#ifdef JKCALS_DEV_PROBES
          long long pc2 = clock64();
          pw_b += pc1 - pc0;
          pw_a += pc2 - pc1;
#endif
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const int nv = v.Jp - cmp_g * JM < JM ? v.Jp - cmp_g * JM : JM;
          const int kvalid = v.Iq0 - cmp_b0 * kTfBK;
          const int nks = kvalid >= kTfBK ? kTfBK / 8 : (kvalid + 7) / 8;
          if (elect_one()) {
            // sub-tile jj of the stage sits at a fixed stride from sub-tile 0 (A: 8 KB, B: BNl x 64 B)
            const uint32_t ahi0 = smem_u32(stA_hi(slot, 0)), alo0 = smem_u32(stA_lo(slot, 0));
            const uint32_t bhi0 = smem_u32(stB_hi(slot, 0)), blo0 = smem_u32(stB_lo(slot, 0));
            const uint32_t bstride = (uint32_t)BNl * 64u;
            for (int jj = 0; jj < JM && jj < nv; ++jj) {
              const uint32_t ahi = ahi0 + jj * 8192u, alo = alo0 + jj * 8192u;
              const uint32_t bhi = bhi0 + jj * bstride, blo = blo0 + jj * bstride;
              for (int kk = 0; kk < nks; ++kk) {
                const uint32_t ko = kk * 32;  // 8 tf32 = 32 bytes along K inside the 64-byte atom
#ifdef JKCALS_DEV_PROBES  // timing probe builds only: one MMA per k-tile (wrong results)
                if ((g.probe == 1 || g.probe == 6) && (jj > 0 || kk > 0)) break;
                if (g.probe == 1 || g.probe == 6) {
                  if (PAIR) umma_tf32_pair(dacc, umma_desc_sw64(ahi + ko), umma_desc_sw64(bhi + ko), idesc, 1u);
                  else umma_tf32(dacc, umma_desc_sw64(ahi + ko), umma_desc_sw64(bhi + ko), idesc, 1u);
                  continue;
                }
#endif
                if (PAIR) {
                  umma_tf32_pair(dacc, umma_desc_sw64(alo + ko), umma_desc_sw64(bhi + ko), idesc, first ? 0u : 1u);
                  umma_tf32_pair(dacc, umma_desc_sw64(ahi + ko), umma_desc_sw64(blo + ko), idesc, 1u);
                  umma_tf32_pair(dacc, umma_desc_sw64(ahi + ko), umma_desc_sw64(bhi + ko), idesc, 1u);
                } else {
                  umma_tf32(dacc, umma_desc_sw64(alo + ko), umma_desc_sw64(bhi + ko), idesc, first ? 0u : 1u);
                  umma_tf32(dacc, umma_desc_sw64(ahi + ko), umma_desc_sw64(blo + ko), idesc, 1u);
                  umma_tf32(dacc, umma_desc_sw64(ahi + ko), umma_desc_sw64(bhi + ko), idesc, 1u);
                }
                first = false;
              }
            }
            // frees the stage (in both CTAs when PAIR) once these MMAs have read it
            if (PAIR) umma_commit_pair(&empty[slot]);
            else umma_commit(&empty[slot]);
            if (cpos == g.chunk - 1 || kt == kt1 - 1) {  // -> drain warps
              if (PAIR) umma_commit_pair(&acc_full[gc & 1]);
              else umma_commit(&acc_full[gc & 1]);
            }
          }
          __syncwarp();
          first = false;
          ++git;
          if (cpos == g.chunk - 1 || kt == kt1 - 1) ++gc;
          if (++cmp_g == KTJ) {
            cmp_g = 0;
            ++cmp_b0;
          }
        }
      }
#ifdef JKCALS_DEV_PROBES
      if (g.probe == 5 && blockIdx.x == 0 && lane == 0)
        printf("TFPROF cta0 k-tiles %u total %lld waitB %lld waitA %lld\n", git, clock64() - pw_t0, pw_b, pw_a);
#endif
    }
  } else if (warp >= kTfAWarps) {
    // ======================= TMEM drain warps (8..11) =======================
    // per chain: tcgen05.ld 16 TMEM columns at a time -> FP64 -> a shared staging block laid out
    // like the piece ([16 rows][128 fused columns], 16 KB contiguous) -> one bulk copy (first chain of
    // a segment) or bulk f64 add (later chains) by one thread. r02: the former read-modify-write
    // through L2 made the drain the bottleneck at 128-product chains.
    const int quad = warp & 3;               // TMEM lane quadrant of this warp
    const int row = quad * 32 + lane;        // fused column c0 + row <-> TMEM lane
    const bool issuer = (warp == kTfAWarps && lane == 0);
    unsigned gc = 0, rnd = 0;  // chains drained, staging rounds (buffer rnd & 1)
    for (int64_t u = u0; u < u1;) {
      const int t = (int)(u / g.KT);
      const int kt0 = (int)(u % g.KT);
      const int64_t kt_end = (int64_t)kt0 + (u1 - u);
      const int kt1 = (int)(kt_end < (int64_t)g.KT ? kt_end : (int64_t)g.KT);
      u += kt1 - kt0;
      const int tm1 = PAIR ? 2 * (t % g.nMt) + crk : t % g.nMt;  // this CTA's 128-column tile
      const bool wr = tm1 < nMt1;  // (PAIR: the second half of an odd last super tile is dead)
      const TileInfo ti = tinfo[(t / g.nMt) * nMt1 + (wr ? tm1 : 0)];
      double* P = parts + ((int64_t)ti.piece_base + (b - ti.first_cta)) * (int64_t)(BN * kBM);
      const int nch = (kt1 - kt0 + g.chunk - 1) / g.chunk;
      for (int ch = 0; ch < nch; ++ch, ++gc) {
        mbar_wait_safe(&acc_full[gc & 1], (gc >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16) + (gc & 1) * kTfMaxN;
        int bn_drain = wr ? BN : 0;
#ifdef JKCALS_DEV_PROBES  // timing probe builds only: drain skipped (wrong results)
        if (g.probe == 4 || g.probe == 6) bn_drain = 0;
#endif
        // the previous chain's adds into this piece must have landed before this chain's are issued
        if (issuer) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
        for (int col = 0; col < bn_drain; col += 16, ++rnd) {
          double* sb = stg + (rnd & 1) * 2048;
          if (rnd >= 2) {  // staging buffer rnd & 1 was read by the bulk op of round rnd - 2
            if (issuer) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
            drain_bar();
          }
          float vals[16];
          tmem_ld_32x32b<16>(lane_base + (uint32_t)col, vals);
#pragma unroll
          for (int q = 0; q < 16; ++q) sb[q * 128 + row] = (double)vals[q];
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic -> bulk copy
          drain_bar();
          if (issuer) bulk_store_f64(P + (int64_t)col * kBM, sb, 16u * 128u * 8u, ch != 0);
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (PAIR) mbar_arrive_cluster(smem_peer(&acc_empty[gc & 1], 0));
          else mbar_arrive(&acc_empty[gc & 1]);
        }
      }
    }
    if (issuer) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // pieces complete
  } else {
    // ======================= A producers (warps 0-7) =======================
    const int row = tid & (kBM - 1);  // fused column c0 + row of the A tile
    const int kh = tid >> 7;          // which half of the k-tile (chunks 2kh, 2kh+1)
    unsigned git = 0;
    for (int64_t u = u0; u < u1;) {
      const int t = (int)(u / g.KT);
      const int kt0 = (int)(u % g.KT);
      const int64_t kt_end = (int64_t)kt0 + (u1 - u);
      const int kt1 = (int)(kt_end < (int64_t)g.KT ? kt_end : (int64_t)g.KT);
      u += kt1 - kt0;
      const int tm = t % g.nMt;
      const int c0 = (PAIR ? 2 * tm + crk : tm) * kBM;
      const bool live = (c0 + row) < g.C;
      // swizzled (SWIZZLE_64B, K-major) byte offset of this row's 16-byte chunk ch
      const uint32_t rbase = (uint32_t)(row >> 3) * 512u + (uint32_t)(row & 7) * 64u;
      const uint32_t sw = (uint32_t)((row & 7) >> 1) & 3u;
      // this thread's 8 U_q0 values (its row, its k half) stay in registers for the J' tiles of
      // an i_q0 block; they are re-read from the FP64 slab only when the block changes
      float uv[8];
      int uv_b0 = -1;
      int cmp_b0 = kt0 / KTJ, cmp_g = kt0 % KTJ;  // running (i_q0 block, j' group)
      for (int kt = kt0; kt < kt1; ++kt) {
        const int nv = v.Jp - cmp_g * JM < JM ? v.Jp - cmp_g * JM : JM;
        const int slot = (int)(git % kTfStages);
        if (git >= (unsigned)kTfStages) mbar_wait_safe(&empty[slot], ((git / kTfStages) - 1) & 1u);
        mbar_wait_safe(&fullS[slot], (git / kTfStages) & 1u);
        if (uv_b0 != cmp_b0) {
          const double* ub = Ub + (cmp_b0 & 1) * (kBK * kBMP) + row;
#pragma unroll
          for (int e = 0; e < 8; ++e) uv[e] = (float)ub[(kh * 8 + e) * kBMP];
          uv_b0 = cmp_b0;
        }
        for (int jj = 0; jj < JM && jj < nv; ++jj) {  // one A sub-tile per j' of the k-tile
          const double* Ss = stS(slot, jj);
          float s = 0.0f;
          if (live) {
            double sd = Ss[row];
            for (int q = 1; q < v.nslow; ++q) sd *= Ss[q * kBM + row];
            s = (float)sd;
          }
          unsigned char* ah = stA_hi(slot, jj) + rbase;
          unsigned char* al = stA_lo(slot, jj) + rbase;
#ifdef JKCALS_DEV_PROBES  // timing probe builds only: A tile not built (wrong results)
          if (g.probe != 2 && g.probe != 6)
#endif
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int ch = kh * 2 + cc;
            float4 h4, l4;
            float* hp = &h4.x;
            float* lp = &l4.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float a = uv[cc * 4 + e] * s;  // KRP^T(c, k) = U_q0(k, c) * S(c), FP32 product
              const uint32_t hb = tf32_trunc(a);
              hp[e] = __uint_as_float(hb);
              lp[e] = a - __uint_as_float(hb);
            }
            const uint32_t off = ((uint32_t)ch ^ sw) * 16u;
            *reinterpret_cast<float4*>(ah + off) = h4;
            *reinterpret_cast<float4*>(al + off) = l4;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> tensor core
        __syncwarp();
        if (lane == 0) {
          if (PAIR) mbar_arrive_cluster(smem_peer(&fullA[slot], 0));
          else mbar_arrive(&fullA[slot]);
        }
        ++git;
        if (++cmp_g == KTJ) {
          cmp_g = 0;
          ++cmp_b0;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (PAIR) cluster_sync_all();  // no remote arrive / commit / operand read may target an exited peer
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTfTmemCols));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kTfTmemCols));
  }
}
#ifdef JK_TU_HOST

// FP32 hi/lo copies of T for the TF32 path. dst layout: dims permuted by `perm01` (swap modes 0
// and 1 when set), first-dim pitch ld_dst (multiple of 4 floats => 16-byte TMA strides).
__global__ void split_tf32_kernel(const double* __restrict__ T, int64_t I0, int64_t I0p, int64_t I1, int64_t rest,
                                  int perm01, int64_t ld_dst, float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= I0 * I1 * rest) return;
  const int64_t i0 = e % I0, i1 = (e / I0) % I1, r = e / (I0 * I1);
  const double x = T[i0 + I0p * (i1 + I1 * r)];
  const float h = __uint_as_float(__float_as_uint((float)x) & 0xFFFFE000u);
  const float l = (float)(x - (double)h);
  const int64_t d = perm01 ? (i1 + ld_dst * (i0 + I0 * r)) : (i0 + ld_dst * (i1 + I1 * r));
  hi[d] = h;
  lo[d] = l;
}
#endif

}  // namespace jk
