// jkcals.cu — host orchestration and C ABI (include/jkcals.h) of the B200 JK-CALS path.
//
// One handle = one shard of submodels on one GPU. The workspace (caller-owned, e.g. a torch
// uint8 tensor) is carved by a deterministic bump layout; a sweep (N x [fused MTTKRP +
// per-submodel epilogue]) is captured once into a CUDA graph and replayed max_iters times
// (CS1 in SURVEY §3). With tol > 0 the host reads one int per sweep (active count) and, when
// enough submodels have converged, compacts them out (a8) and re-captures the graph.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: host ranges for nsys timelines
#include <vector>

#define JK_TU_HOST  // this TU defines the small non-template kernels; the heavy ones live in k_*.cu
#include "../../include/jkcals.h"
#include "align.cuh"
#include "aux_kernels.cuh"
#include "epilogue_large.cuh"
#include "kernels.h"

using namespace jk;

namespace {

constexpr size_t kAlign = 256;
constexpr size_t kTfSmemMax = 227 * 1024;  // opt-in dynamic shared memory per CTA on sm_100

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }

// ---------------------------------------------------------------- tuning overrides
// Every environment knob the library reads, parsed once per process. None changes results (each
// selects among kernels / tilings that are all parity-tested) and none is needed in production: the
// defaults are the calibrated cost models below. They exist for the tuning sweeps recorded in
// DESIGN.md §9c (tools/*.py) and for the tests that pin one kernel path.
//   JKCALS_FORCE_NT=<mode>:<NT>[,...]  N tile (n8 tiles) per mode        JKCALS_FORCE_WM=<8|5>  tile width
//   JKCALS_FORCE_KB=<16|20>            k-tile depth                       JKCALS_SK_ALPHA=<a>    stream-K weight
//   JKCALS_RED_PIECES=<n>              pre-reduce threshold (0: never)
//   JKCALS_RESIDENT=<0|1|2>            0 streamed only, 1 cluster-resident, 2 warp-resident (unset: auto);
//                                      read at each plan (tests pin the path per handle), see resident_mode()
//   JKCALS_TF32_MIN_NNT / JKCALS_TF32_MAX_STAGES   FP32 path N tiles / ring depth
//   JKCALS_TF32_PAIR=0                 FP32 path: one-CTA kernel only (no cta_group::2 pairs)
//   JKCALS_TF32_CHUNK=<k>              FP32 path: k-tiles per FP32 accumulation chain (accuracy!)
//   JKCALS_MAX_CTAS=<g>                FP64 MTTKRP: cap on the stream-K grid
//   JKCALS_TF32_JM=<1|2|4>             FP32 path: j' values per k-tile
//   JKCALS_MAX_PIECES=<p>              FP64 MTTKRP: stream-K pieces per tile when < 4 tiles (48)
//   JKCALS_I8_RESIDENT / JKCALS_I8_CLUSTER         FP64_I8 kernel variant
//   JKCALS_I8_PROBE                    timing-probe builds only (-DJKCALS_DEV_PROBES; wrong results)
//   JKCALS_TOL_HOST_LOOP=1             tol mode: host check after every sweep (no WHILE graph node)
struct Tuning {
  std::string force_nt;
  int force_wm = 0, force_kb = 0, red_pieces = -1;
  double sk_alpha = -1.0;
  // tf32_max_stages: 4 by default (r02: the MTTKRP is not ring-depth bound -- 3, 4, 6, 8 stages
  // within 1 % per launch -- while a 4-stage ring leaves room for the dependent epilogue's CTAs
  // to become resident under PDL: syn200 FP32 38.7 -> 36.3 ms, eem R5 -1.8 %, 4-way -0.4 %)
  int tf32_min_nnt = 0, tf32_max_stages = 4, i8_resident = 0, i8_cluster = 1, i8_probe = 0;
  int tol_host_loop = 0, tf32_pair = 1, tf32_chunk = 0, max_ctas = 0, tf32_jm = 0, max_pieces = 0;
};
const Tuning& tuning() {
  static const Tuning t = [] {
    Tuning v;
    auto geti = [](const char* k, int d) { const char* e = getenv(k); return e ? atoi(e) : d; };
    if (const char* e = getenv("JKCALS_FORCE_NT")) v.force_nt = e;
    v.force_wm = geti("JKCALS_FORCE_WM", 0);
    v.force_kb = geti("JKCALS_FORCE_KB", 0);
    v.red_pieces = geti("JKCALS_RED_PIECES", -1);
    if (const char* e = getenv("JKCALS_SK_ALPHA")) v.sk_alpha = atof(e);
    v.tf32_min_nnt = geti("JKCALS_TF32_MIN_NNT", 0);
    v.tf32_max_stages = geti("JKCALS_TF32_MAX_STAGES", 4);
    v.i8_resident = geti("JKCALS_I8_RESIDENT", 0);
    v.i8_cluster = geti("JKCALS_I8_CLUSTER", 1);
    v.i8_probe = geti("JKCALS_I8_PROBE", 0);
    v.tol_host_loop = geti("JKCALS_TOL_HOST_LOOP", 0);
    v.tf32_pair = geti("JKCALS_TF32_PAIR", 1);
    v.tf32_chunk = geti("JKCALS_TF32_CHUNK", 0);
    v.max_ctas = geti("JKCALS_MAX_CTAS", 0);
    v.tf32_jm = geti("JKCALS_TF32_JM", 0);
    v.max_pieces = geti("JKCALS_MAX_PIECES", 0);
    return v;
  }();
  return t;
}
int resident_mode() {
  const char* e = getenv("JKCALS_RESIDENT");
  return e ? atoi(e) : -1;
}

// ---------------------------------------------------------------- kernel dispatch tables
struct KernelInfo {
  MttkrpFn fn[kNumKB][kNumWM][2][2][kMaxNT];         // [k depth kKBs][tile width kWMs][KMAJOR][STAGES==4][NT-1]
  SmemFn smem[kNumKB][kNumWM][2][2][kMaxNT];
  int occ[kNumKB][kNumWM][2][2][kMaxNT][kMaxModes];  // [..][nslow]
  int nsm;
  int i8clusters;                    // co-resident 2-CTA clusters of the INT8 cluster kernel (0: none)
  int tfpairs = 0;                   // co-resident CTA pairs of the FP32 cta_group::2 kernel (0: none)
};

KernelInfo* kernel_info(int device, std::string* err) {
  static KernelInfo info[16];
  static bool ready[16] = {false};
  if (device < 0 || device >= 16) return nullptr;
  if (ready[device]) return &info[device];
  KernelInfo& ki = info[device];
  {
    MttkrpFn f[kNumKB][2][kNumWM][2][kMaxNT];
    SmemFn sm[kNumKB][2][kNumWM][2][kMaxNT];
    dmma_kernels_km0_kb16(f[0][0], sm[0][0]);
    dmma_kernels_km1_kb16(f[0][1], sm[0][1]);
    dmma_kernels_km0_kb20(f[1][0], sm[1][0]);
    dmma_kernels_km1_kb20(f[1][1], sm[1][1]);
    for (int kv = 0; kv < kNumKB; ++kv)
      for (int wv = 0; wv < kNumWM; ++wv)
        for (int km = 0; km < 2; ++km)
          for (int st = 0; st < 2; ++st)
            for (int t = 0; t < kMaxNT; ++t) {
              ki.fn[kv][wv][km][st][t] = f[kv][km][wv][st][t];
              ki.smem[kv][wv][km][st][t] = sm[kv][km][wv][st][t];
            }
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaDeviceGetAttribute(&ki.nsm, cudaDevAttrMultiProcessorCount, device);
  {
    cudaError_t e = cudaSuccess;
    for (bool pair : {false, true})
      for (int st : {2, 3, 4})
        for (int jm : {1, 2, 4})
          if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tf32_kernel(st, pair, jm), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kTfSmemMax);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(i8_kernel(0), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kI8Smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(i8_kernel(1), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kI8SmemRes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(i8_kernel(2), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kI8SmemClu);
    // epilogue kernels: opt-in dynamic shared memory (per device, once)
    for (EpiFns f : {epi_kernels_2(), epi_kernels_4(), epi_kernels_6(), epi_kernels_8(), epi_kernels_10(),
                     epi_kernels_12(), epi_kernels_16()})
      for (EpiFn k : {f.smem, f.mixed})
        if (e == cudaSuccess) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(epi_large_kernel(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)epi_large_smem_bytes());
    ki.i8clusters = 0;
    if (e == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(2 * (ki.nsm / 2));
      cfg.blockDim = dim3(kI8Threads);
      cfg.dynamicSmemBytes = kI8SmemClu;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, i8_kernel(2), &cfg) == cudaSuccess)
        ki.i8clusters = ncl;
      cudaGetLastError();  // the query is advisory: 0 falls back to the one-CTA kernel
      // CTA pairs of the FP32 path (one CTA per SM): co-resident pairs at the largest ring
      cfg.blockDim = dim3(kTfThreads);
      cfg.dynamicSmemBytes = kTfSmemMax;
      ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, tf32_kernel(4, true), &cfg) == cudaSuccess)
        ki.tfpairs = ncl;
      cudaGetLastError();
    }
    if (e != cudaSuccess) {
      if (err) *err = std::string("cudaFuncSetAttribute(tf32): ") + cudaGetErrorString(e);
      cudaSetDevice(prev);
      return nullptr;
    }
  }
  for (int kv = 0; kv < kNumKB; ++kv)
    for (int wv = 0; wv < kNumWM; ++wv)
      for (int km = 0; km < 2; ++km)
        for (int st = 0; st < 2; ++st)
          for (int t = 0; t < kMaxNT; ++t) {
            cudaError_t e = cudaFuncSetAttribute(ki.fn[kv][wv][km][st][t], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)ki.smem[kv][wv][km][st][t](kMaxModes - 2));
            if (e != cudaSuccess) {
              if (err) *err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
              cudaSetDevice(prev);
              return nullptr;
            }
            for (int ns = 1; ns <= kMaxModes - 2; ++ns) {
              int occ = 0;
              cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ki.fn[kv][wv][km][st][t], (kWMs[wv] + 1) * 32,
                                                            ki.smem[kv][wv][km][st][t](ns));
              ki.occ[kv][wv][km][st][t][ns] = std::max(1, occ);
            }
          }
  cudaSetDevice(prev);
  ready[device] = true;
  return &ki;
}

// ---------------------------------------------------------------- per-mode plan
// q0 = fastest rest mode (mode 1 when n == 0, else mode 0); J' = product of the others.
struct ModeGeo {
  int64_t In, Iq0, Jp;
  int q0, nslow;
};

ModeGeo mode_geo(int N, const int64_t* dims, int n) {
  ModeGeo g;
  g.In = dims[n];
  g.q0 = (n == 0) ? 1 : 0;
  g.Iq0 = dims[g.q0];
  g.Jp = 1;
  for (int m = 0; m < N; ++m)
    if (m != n && m != g.q0) g.Jp *= dims[m];
  g.nslow = N - 2;
  return g;
}

struct ModePlan {
  int NT = 1, KM = 0, ST4 = 1, BN = 8, nMt = 1, nNt = 1, KT = 1, G = 1;
  int WV = 0, BM = kBM;  // FP64 kernel tile width: kWMs[WV] consumer warps x 16 = BM fused columns
  int KV = 0, KB = kBK;  // FP64 kernel k-tile depth kKBs[KV] (i_q0 values per k-tile)
  int64_t units = 1;
  int ntiles = 1, npieces = 1;
  size_t smem = 0;
  std::vector<TileInfo> tinfo;
  std::vector<int> cta_u;  // CTA b processes units [cta_u[b], cta_u[b+1])
  int tf32 = 0;
  int pair = 0, nMt2 = 1;  // FP32 path: CTA-pair kernel on 256-column super tiles (nMt2 per tile row)
  int JM = 1;              // FP32 path: j' values per k-tile
};

// stream-K CTA ranges, per-tile piece bookkeeping (shared by the FP64 and TF32 plans).
// CTA b processes units [cta_u[b], cta_u[b+1]) of the (tile, k-tile) space, split uniformly.
// (r01 measurement: weighting units by their DMMA count made the CTAs on ragged tiles the
// stragglers -- the per-k-tile time is dominated by its fixed part -- so the split is uniform.)
// Stream-K split of the (tile, k-tile) units over G CTAs. A unit of a ragged tile (the last
// M tile when C is not a multiple of 128, the last N tile) costs less than a full one: cost =
// alpha + (1 - alpha) * (live DMMA fraction of the tile), alpha the per-k-tile fixed share
// (barriers, fragment loads, KRP scaling). alpha = 1 is the uniform split.
void finish_plan(ModePlan& p, const ModeGeo& mg, int64_t C = 0, double alpha = 1.0) {
  p.cta_u.assign(p.G + 1, 0);
  if (alpha >= 1.0 || C <= 0) {
    for (int b = 0; b <= p.G; ++b) p.cta_u[b] = (int)((int64_t)b * p.units / p.G);
  } else {
    std::vector<double> w(p.ntiles), cum(p.ntiles + 1, 0.0);
    for (int t = 0; t < p.ntiles; ++t) {
      const int tm = t % p.nMt, tn = t / p.nMt;
      const int64_t lc = std::min<int64_t>(p.BM, C - (int64_t)tm * p.BM);
      const int64_t lr = std::min<int64_t>(p.BN, mg.In - (int64_t)tn * p.BN);
      const double f = (double)rup(lc, 16) / p.BM * (double)rup(lr, 8) / p.BN;
      w[t] = alpha + (1.0 - alpha) * f;
      cum[t + 1] = cum[t] + w[t] * p.KT;
    }
    int t = 0;
    for (int b = 0; b <= p.G; ++b) {
      const double target = cum[p.ntiles] * b / p.G;
      while (t < p.ntiles - 1 && cum[t + 1] < target) ++t;
      int64_t u = (int64_t)t * p.KT + (int64_t)std::llround((target - cum[t]) / w[t]);
      u = std::min<int64_t>(std::max<int64_t>(u, 0), p.units);
      p.cta_u[b] = (int)u;
    }
    p.cta_u[0] = 0;
    p.cta_u[p.G] = (int)p.units;
    for (int b = 1; b <= p.G; ++b) p.cta_u[b] = std::max(p.cta_u[b], p.cta_u[b - 1]);
  }
  // drop empty ranges so that the CTAs touching a tile are consecutive and the piece index of
  // CTA b in tile t is b - first_cta[t]
  p.cta_u.erase(std::unique(p.cta_u.begin(), p.cta_u.end()), p.cta_u.end());
  p.G = (int)p.cta_u.size() - 1;
  std::vector<int> first(p.ntiles, -1), lastc(p.ntiles, -1);
  for (int b = 0; b < p.G; ++b) {
    int64_t u0 = p.cta_u[b], u1 = p.cta_u[b + 1];
    if (u0 >= u1) continue;
    int64_t t0 = u0 / p.KT, t1 = (u1 - 1) / p.KT;
    for (int64_t t = t0; t <= t1; ++t) {
      if (first[t] < 0) first[t] = b;
      lastc[t] = b;
    }
  }
  p.tinfo.resize(p.ntiles);
  int base = 0;
  for (int t = 0; t < p.ntiles; ++t) {
    p.tinfo[t].first_cta = first[t];
    p.tinfo[t].npieces = lastc[t] - first[t] + 1;
    p.tinfo[t].piece_base = base;
    p.tinfo[t].pad_ = 0;
    base += p.tinfo[t].npieces;
  }
  p.npieces = base;
}


ModePlan make_plan(const ModeGeo& mg, int n, int64_t C, const KernelInfo& ki, bool tf32 = false) {
  ModePlan p;
  if (tf32) {
    // FP32 (3xTF32 tcgen05) path: UMMA M = 128 fused columns, N = whole I_n up to 256 per tile
    p.tf32 = 1;
    p.nNt = (int)cdiv(mg.In, kTfMaxN);
    p.nNt = std::max<int>(p.nNt, tuning().tf32_min_nnt);
    p.BN = (int)rup(cdiv(mg.In, p.nNt), 16);
    p.NT = p.BN / 8;
    p.KM = 1;
    p.nMt = (int)std::max<int64_t>(1, cdiv(C, kBM));
    // CTA pairs (cta_group::2, UMMA M = 256) whenever there are two 128-column tiles to pair:
    // each SM then reads A + B/2 instead of A + B from shared memory per MMA
    p.pair = (p.nMt >= 2 && ki.tfpairs > 0 && tuning().tf32_pair) ? 1 : 0;
    const int BNl = p.pair ? p.BN / 2 : p.BN;
    // j' values per k-tile (JM): more MMA work per ring handshake (r02); at most
    // what a 2-stage ring fits
    // per mode (r02, profiles/r02_fp32_jm.txt): a k-tile of I_n >= 192 rows already carries enough
    // MMA work per handshake (syn200: JM = 2 was 7 % slower), narrower tiles gain from 4 j' per
    // k-tile (eem mode 2, I_n = 61: 172 -> 111 us; 4-way mode 3, I_n = 30: 412 -> 277 us)
    { const int jm = tuning().tf32_jm > 0 ? tuning().tf32_jm : (p.BN >= 192 ? 1 : 4);
      p.JM = jm >= 4 ? 4 : jm >= 2 ? 2 : 1; }
    while (p.JM > 1 && tf_smem_bytes(BNl, mg.nslow, 2, p.JM) > kTfSmemMax) p.JM /= 2;
    p.KT = (int)(cdiv(mg.Iq0, kTfBK) * cdiv(mg.Jp, p.JM));
    // deepest ring of {4, 3, 2} stages that fits under the cap (JKCALS_TF32_MAX_STAGES, default 4)
    const int cap = tuning().tf32_max_stages;
    p.ST4 = 2;
    for (int st : {4, 3})  // (deeper rings measured no faster, r02)
      if (st <= cap && tf_smem_bytes(BNl, mg.nslow, st, p.JM) <= kTfSmemMax) { p.ST4 = st; break; }
    p.smem = tf_smem_bytes(BNl, mg.nslow, p.ST4, p.JM);
    if (!p.pair) {
      p.ntiles = p.nMt * p.nNt;
      p.units = (int64_t)p.ntiles * p.KT;
      p.G = (int)std::min<int64_t>(p.units, std::min<int64_t>((int64_t)ki.nsm, 48 * (int64_t)p.ntiles));
      finish_plan(p, mg);
      return p;
    }
    // stream-K over super tiles (pairs are the plan's CTAs), then one piece table entry per
    // 128-column tile: both halves of a super tile share its CTA range and piece count
    ModePlan q = p;
    q.nMt = (int)cdiv(p.nMt, 2);
    q.ntiles = q.nMt * q.nNt;
    q.units = (int64_t)q.ntiles * q.KT;
    q.G = (int)std::min<int64_t>(q.units, std::min<int64_t>((int64_t)ki.tfpairs, 48 * (int64_t)q.ntiles));
    finish_plan(q, mg);
    p.nMt2 = q.nMt;
    p.units = q.units;
    p.G = q.G;
    p.cta_u = q.cta_u;
    p.ntiles = p.nMt * p.nNt;
    p.tinfo.resize(p.ntiles);
    int base = 0;
    for (int tn = 0; tn < p.nNt; ++tn)
      for (int tm = 0; tm < p.nMt; ++tm) {
        const TileInfo& st = q.tinfo[tn * q.nMt + tm / 2];
        TileInfo& ti = p.tinfo[tn * p.nMt + tm];
        ti.first_cta = st.first_cta;
        ti.npieces = st.npieces;
        ti.piece_base = base;
        ti.pad_ = 0;
        base += st.npieces;
      }
    p.npieces = base;
    return p;
  }
  // N tiling: NT n8 tiles per CTA tile. Score = useful/issued n8 slots x NT/(NT + 1), the second
  // factor modelling the per-k-tile cost that does not scale with NT (A fragments, S scaling,
  // barriers): I_n = 200 (25 n8) -> 5 x 5 exactly rather than 4 x 7 with 3 idle slots.
  const int64_t nI8 = cdiv(mg.In, 8);
  double best = -1.0;
  for (int nt = 1; nt <= kMaxNT; ++nt) {
    const int64_t ntiles_n = cdiv(nI8, nt);
    // variants that fit 2 CTAs/SM (<= 96 regs: NT <= 6) hide the per-k-tile latency better:
    // measured +7 % on syn200 (r01), modelled as a 1.08 factor
    const int km = (n != 0) ? 1 : 0, st4 = (mg.Jp >= 3) ? 1 : 0;
    const double occ_bonus = ki.occ[0][0][km][st4][nt - 1][mg.nslow] >= 2 ? 1.08 : 1.0;
    const double score = (double)nI8 / (double)(ntiles_n * nt) * (double)nt / (nt + 1.0) * occ_bonus;
    if (score > best + 1e-12) {
      best = score;
      p.NT = nt;
      p.nNt = (int)ntiles_n;
    }
  }
  // JKCALS_FORCE_NT=<mode>:<NT>[,<mode>:<NT>...] overrides the model (tuning experiments only)
  if (!tuning().force_nt.empty()) {
    for (const char* q = tuning().force_nt.c_str(); *q;) {
      int mm = -1, nt = 0, used = 0;
      if (sscanf(q, "%d:%d%n", &mm, &nt, &used) != 2) break;
      if (mm == n && nt >= 1 && nt <= kMaxNT) {
        p.NT = nt;
        p.nNt = (int)cdiv(nI8, nt);
      }
      q += used;
      if (*q == ',') ++q;
    }
  }
  p.BN = p.NT * 8;
  p.KM = (n != 0) ? 1 : 0;
  p.ST4 = (mg.Jp >= 3) ? 1 : 0;  // the U_q0 slab double buffer needs J' >= STAGES - 1
  // tile width: kWMs[wv] consumer warps x 16 columns. Cost model (warp-k-tiles per k-tile row):
  // a tile with w live warps costs max(w, 0.7 WM) -- the per-k-tile fixed share, r01's alpha --
  // so a mostly idle last tile is charged 70 % of a full one. 4-way C = 400: 8 warps -> 3 full +
  // 1 one-warp tile = 29.6; 5 warps -> 5 full 80-column tiles = 25 / 0.90 (r02: 370 vs 393 us on
  // modes 1-2). The wider tile is kept unless the narrower one is >= 3 % cheaper.
  // JKCALS_FORCE_WM=<8|5> overrides (tuning).
  {
    double cost[kNumWM];
    for (int wv = 0; wv < kNumWM; ++wv) {
      const int WM = kWMs[wv], BM = WM * 16;
      const int64_t tiles = std::max<int64_t>(1, cdiv(C, BM));
      const int64_t w_last = cdiv(C - (tiles - 1) * BM, 16);
      cost[wv] = (double)(tiles - 1) * WM + std::max((double)w_last, 0.7 * WM);
      // per-warp efficiency of the narrow tile relative to the wide one (r02 on B200): its
      // per-k-tile fixed work is shared by fewer warps -- 0.90 with NT >= 6 n8 tiles (4-way modes
      // 0-2), 0.75 below (syn200 NT = 5: 23.2 vs 30.7 TF/s; 4-way mode 3, NT = 4, slower too)
      if (WM < kWMs[0]) cost[wv] /= (p.NT >= 6 ? 0.90 : 0.75);
    }
    p.WV = (cost[1] < 0.97 * cost[0]) ? 1 : 0;
    const int force_wm = tuning().force_wm;
    for (int wv = 0; wv < kNumWM; ++wv)
      if (force_wm == kWMs[wv]) p.WV = wv;
    p.BM = kWMs[p.WV] * 16;
  }
  p.nMt = (int)std::max<int64_t>(1, cdiv(C, p.BM));
  // k-tile depth: 16 or 20 i_q0 values. A k-tile costs phi (its fixed share: barriers, TMA, the
  // A-fragment build) + its live depth / 16; a ragged last block pays phi for a partial depth.
  // Calibrated on B200 (r02, phi = 0.12, 2 % margin): I_q0 = 200 / 100 / 50 take 20 (syn200
  // 157.2 -> 149.9 ms, 4-way modes 1-3 -8 to -13 %, the "All" pool -5 %), I_q0 = 201 / 268 keep 16
  // (eem R6 was 4 % slower with 20). The 20-deep variant is also skipped when it fits fewer CTAs per
  // SM. JKCALS_FORCE_KB=<16|20> overrides (tuning).
  {
    constexpr double phi = 0.12;
    double cost[kNumKB];
    for (int kv = 0; kv < kNumKB; ++kv) {
      const int KB = kKBs[kv];
      const int64_t full = mg.Iq0 / KB, rem = mg.Iq0 % KB;
      cost[kv] = (double)full * (phi + KB / 16.0) + (rem ? phi + rem / 16.0 : 0.0);
    }
    p.KV = (mg.Jp >= 3 && cost[1] < 0.98 * cost[0] &&
            ki.occ[1][p.WV][p.KM][1][p.NT - 1][mg.nslow] >= ki.occ[0][p.WV][p.KM][1][p.NT - 1][mg.nslow])
               ? 1 : 0;  // (the 20-deep variants need STAGES = 4: J' >= 3)
    const int force_kb = tuning().force_kb;
    for (int kv = 0; kv < kNumKB; ++kv)
      if (force_kb == kKBs[kv] && (kv == 0 || mg.Jp >= 3)) p.KV = kv;
    p.KB = kKBs[p.KV];
  }
  p.KT = (int)(cdiv(mg.Iq0, p.KB) * mg.Jp);
  p.ntiles = p.nMt * p.nNt;
  p.units = (int64_t)p.ntiles * p.KT;
  p.smem = ki.smem[p.KV][p.WV][p.KM][p.ST4][p.NT - 1](mg.nslow);
  int64_t gmax = (int64_t)ki.nsm * ki.occ[p.KV][p.WV][p.KM][p.ST4][p.NT - 1][mg.nslow];
  if (tuning().max_ctas > 0) gmax = std::min<int64_t>(gmax, tuning().max_ctas);
  // at most kMaxPieces partial pieces per output tile: small problems (few tiles) would
  // otherwise write and re-read a BN x BM piece per CTA for ~1 k-tile of work each
  // (only for < 4 tiles: a single 128-column M tile x 5 N tiles -- a syn200 shard at 8 GPUs --
  // must still fill both CTA slots of every SM, r01 +20 %; such tiles are pre-reduced, kRedPieces)
  const int64_t kMaxPieces = tuning().max_pieces > 0 ? tuning().max_pieces : 48;
  if (p.ntiles < 4) gmax = std::min<int64_t>(gmax, kMaxPieces * p.ntiles);
  p.G = (int)std::min<int64_t>(p.units, gmax);
  // cost-weighted split only when a tile is mostly idle (e.g. 4-way C = 400: the last M tile
  // has 16 of 128 columns): r01 measured alpha = 0.7 +6 % there, while nearly-full ragged tiles
  // (syn200: 104 of 128) are best with the uniform split. JKCALS_SK_ALPHA overrides (tuning).
  const double env_alpha = tuning().sk_alpha;
  const double live_m = (double)rup(C - (int64_t)(p.nMt - 1) * p.BM, 16) / p.BM;
  const double alpha = env_alpha >= 0.0 ? env_alpha : (live_m < 0.5 ? 0.7 : 1.0);
  finish_plan(p, mg, C, alpha);
  return p;
}

constexpr int kRedPieces = 16;  // pre-reduce when a tile has more partial pieces than this

int64_t plan_parts_doubles(const ModePlan& p) { return (int64_t)p.npieces * p.BN * p.BM; }

// device plan table: TileInfo[ntiles] followed by int cta_u[G+1] (read by the kernel)
size_t plan_table_bytes(int ntiles, int G) { return ntiles * sizeof(TileInfo) + (size_t)(G + 1) * sizeof(int); }
std::vector<char> pack_plan(const ModePlan& p) {
  std::vector<char> buf(plan_table_bytes(p.ntiles, p.G));
  memcpy(buf.data(), p.tinfo.data(), p.ntiles * sizeof(TileInfo));
  memcpy(buf.data() + p.ntiles * sizeof(TileInfo), p.cta_u.data(), (p.G + 1) * sizeof(int));
  return buf;
}

// upper bound for workspace sizing (any C' <= C)
void plan_bounds(const ModeGeo& mg, int n, int64_t C, const KernelInfo& ki, int64_t* parts, int* tiles,
                 bool tf32 = false) {
  ModePlan p = make_plan(mg, n, C, ki, tf32);
  // any later (compacted, smaller-C) plan has G <= 8 nsm CTAs and <= ntiles tiles
  // (x kBM: the widest tile; a narrower-tile plan has more tiles, bounded by nMt(80) <= 2 nMt(128))
  *parts = (int64_t)(std::max<int64_t>(p.G, 8 * (int64_t)ki.nsm) + 2 * p.ntiles) * p.BN * kBM;
  *tiles = 2 * p.ntiles;
}

MttkrpView make_mview(int N, const int64_t* dims, int n, const double* const* Uall, int KB = kBK) {
  ModeGeo mg = mode_geo(N, dims, n);
  MttkrpView v;
  v.In = (int)mg.In;
  v.Iq0 = (int)mg.Iq0;
  v.nb0 = (int)cdiv(mg.Iq0, KB);
  v.Jp = (int)mg.Jp;
  // slow modes merged into <= 2 runs: n == 0 -> one run (modes 2..N-1);
  // n >= 1 -> run A = modes 1..n-1, run B = modes n+1..N-1 (j' = jA + runA * jB, Eq. 3 order)
  int64_t runA = 1;
  if (n == 0) {
    for (int m = 2; m < N; ++m) runA *= dims[m];
  } else {
    for (int m = 1; m < n; ++m) runA *= dims[m];
  }
  v.runA = (int)runA;
  v.nslow = N - 2;
  int s = 0;
  for (int m = 0; m < N; ++m) {
    if (m == n || m == mg.q0) continue;
    v.sdim[s] = (int)dims[m];
    v.Us[s] = Uall[m];
    ++s;
  }
  for (; s < kMaxModes - 2; ++s) {
    v.sdim[s] = 1;
    v.Us[s] = nullptr;
  }
  return v;
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// T (FP64, column-major, mode-0 pitch I0p even so that every stride is a multiple of 16 B)
// viewed for mode n as a 4-D box source with non-decreasing strides:
//   n == 0: (i_0 [In], i_1 [q0], modes 2.. [run], 1)       box (BNP, 16, 1, 1)
//   n >= 1: (i_0 [q0], modes 1..n-1 [runA], i_n, modes n+1.. [runB])   box (20, 1, BN, 1)
bool make_tmap_T(CUtensorMap* tm, const double* T, int N, const int64_t* dims, int64_t I0p, int n, int BN, int BNP,
                 int KB = kBK) {
  auto enc = encode_fn();
  if (!enc) return false;
  int64_t st[kMaxModes + 1];
  st[0] = 1;
  st[1] = I0p;
  for (int m = 2; m <= N; ++m) st[m] = st[m - 1] * dims[m - 1];
  const int64_t total = st[N];
  cuuint64_t gdim[4], gstr[3];
  cuuint32_t box[4], est[4] = {1, 1, 1, 1};
  if (n == 0) {
    int64_t run = 1;
    for (int m = 2; m < N; ++m) run *= dims[m];
    gdim[0] = dims[0]; gdim[1] = dims[1]; gdim[2] = run; gdim[3] = 1;
    gstr[0] = st[1] * 8; gstr[1] = st[2] * 8; gstr[2] = total * 8;
    box[0] = BNP; box[1] = KB; box[2] = 1; box[3] = 1;
  } else {
    int64_t runA = 1, runB = 1;
    for (int m = 1; m < n; ++m) runA *= dims[m];
    for (int m = n + 1; m < N; ++m) runB *= dims[m];
    gdim[0] = dims[0]; gdim[1] = runA; gdim[2] = dims[n]; gdim[3] = runB;
    gstr[0] = st[1] * 8; gstr[1] = st[n] * 8; gstr[2] = (n + 1 < N ? st[n + 1] : total) * 8;
    box[0] = KB + ((4 - KB % 16) + 16) % 16; box[1] = 1; box[2] = BN; box[3] = 1;  // row pitch 4 mod 16
  }
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(T), gdim, gstr, box, est,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// U_q0 (row-major rows x ldu): 2-D box (BMP columns, BK rows); OOB rows/columns read as zero.
// FP32 hi/lo copy viewed as (q0 [contiguous], runA, n, runB), box (16, 1, BN, 1) with the 64-byte
// swizzle that the UMMA K-major SWIZZLE_64B operand layout expects.
bool make_tmap_T32(CUtensorMap* tm, const float* T, const int64_t gdim_in[4], const int64_t gstride_elems[3], int BN) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[4], gstr[3];
  for (int d = 0; d < 4; ++d) gdim[d] = (cuuint64_t)gdim_in[d];
  for (int d = 0; d < 3; ++d) gstr[d] = (cuuint64_t)gstride_elems[d] * 4;
  cuuint32_t box[4] = {(cuuint32_t)kTfBK, 1, (cuuint32_t)BN, 1}, est[4] = {1, 1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(T), gdim, gstr, box, est,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_U(CUtensorMap* tm, const double* U, int64_t rows, int64_t ldu, int bmp = kBMP, int KB = kBK) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)ldu, (cuuint64_t)rows}, gstr[1] = {(cuuint64_t)ldu * 8};
  cuuint32_t box[2] = {(cuuint32_t)bmp, (cuuint32_t)KB}, est[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(U), gdim, gstr, box, est,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int bnp_of(int NT) {
  const int BN = NT * 8;
  return BN + ((4 - BN % 16) + 16) % 16;
}

// ---------------------------------------------------------------- INT8-sliced MTTKRP plans (§9b)
struct I8Plan {
  int64_t In, Iq0, Jp, InP, KP, CP;
  int nMt, nNt;
  int variant;  // 0 streaming, 1 resident A (opt-in), 2 2-CTA cluster with multicast A (default)
  ModePlan p;
};
int i8_variant(const KernelInfo& ki, int64_t KP);
I8Plan make_i8_plan(int ndims, const int64_t* dims, int n, int64_t C, const KernelInfo& ki) {
  I8Plan q;
  const ModeGeo mg = mode_geo(ndims, dims, n);
  q.In = mg.In;
  q.Iq0 = mg.Iq0;
  q.Jp = mg.Jp;
  q.KP = rup(q.Iq0, kI8K);
  q.variant = i8_variant(ki, q.KP);
  const int bn = q.variant == 2 ? 2 * kI8N : kI8N;  // plan tile rows (a pair of n-tiles per cluster)
  q.InP = rup(q.In, bn);
  q.CP = rup(C, 128);
  q.nMt = (int)(q.CP / 128);
  q.nNt = (int)(q.InP / bn);
  ModePlan& p = q.p;
  p.nMt = q.nMt;
  p.nNt = q.nNt;
  p.BN = bn;
  p.KT = (int)q.Jp;
  p.ntiles = p.nMt * p.nNt;
  p.units = (int64_t)p.ntiles * p.KT;
  p.G = (int)std::min<int64_t>(p.units, q.variant == 2 ? (int64_t)ki.i8clusters : (int64_t)ki.nsm);
  finish_plan(p, mg);
  return q;
}
// launch the variant the plan chose (the cluster kernel's grid is 2 CTAs per plan "CTA")
cudaError_t launch_i8(const I8Plan& q, const CUtensorMap& tmA, const CUtensorMap& tmB, const I8Geom& g,
                      const TileInfo* ti, double* parts, cudaStream_t s) {
  if (q.variant == 1) {
    i8_kernel(1)<<<q.p.G, kI8Threads, kI8SmemRes, s>>>(tmA, tmB, g, ti, parts);
    return cudaGetLastError();
  }
  if (q.variant == 0) {
    i8_kernel(0)<<<q.p.G, kI8Threads, kI8Smem, s>>>(tmA, tmB, g, ti, parts);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(2 * q.p.G);
  cfg.blockDim = dim3(kI8Threads);
  cfg.dynamicSmemBytes = kI8SmemClu;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, i8_kernel(2), tmA, tmB, g, ti, parts);
}
// exact int32 accumulation: a diagonal sums <= 7 digit products of magnitude <= 64 * 64 per k, so
// the contraction length K = I_q0 (padded) must stay below 2^31 / (7 * 4096) = 74898
// INT8 kernel variant: the 2-CTA cluster kernel with multicast A by default;
// tuning knobs JKCALS_I8_RESIDENT=1 (resident A where I_q0 <= 192; latency-bound, slower) and
// JKCALS_I8_CLUSTER=0 (the one-CTA streaming kernel)
int i8_variant(const KernelInfo& ki, int64_t KP) {
  const int res = tuning().i8_resident, clu = tuning().i8_cluster;
  if (res && KP / kI8K <= kI8ResKS) return 1;
  if (clu && ki.i8clusters >= 1) return 2;
  return 0;
}
bool i8_k_ok(int ndims, const int64_t* dims) {
  return rup(dims[1], kI8K) <= kI8MaxK && rup(dims[0], kI8K) <= kI8MaxK && ndims >= 3;
}
bool make_tmap_i8(CUtensorMap* tm, const int8_t* base, int64_t kp, int64_t rows, int box_rows, int box_slices = kI8S) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)kI8S};
  cuuint64_t gstr[2] = {(cuuint64_t)kp, (cuuint64_t)(kp * rows)};
  cuuint32_t box[3] = {(cuuint32_t)kI8K, (cuuint32_t)box_rows, (cuuint32_t)box_slices}, est[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), gdim, gstr, box, est,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, kI8K == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- workspace layout
struct Layout {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = off;
    off = rup((int64_t)(off + bytes), kAlign);
    return o;
  }
};

struct Offsets {
  size_t T, T32hi, T32lo, T1hi, T1lo, U[2][kMaxModes], Ures, parts, tinfo[kMaxModes], tinfo1[kMaxModes], red, gram,
      tinfo64, tinfo164,
      lambda, normT2p, fit, fit_prev, err, hist,
      slice, slice_part, stage, iters, flags, active, blk2sub, map, pglob, misc, srcoff, srcld, subR, subRc, blkcol,
      dstoff, pref[kMaxModes], aln, aperm, asign, acong, asrc, asld, srcpg;
  size_t i8B[kMaxModes], i8eT[kMaxModes], i8dS[kMaxModes], i8A, i8eU, i8st, i8dims;  // INT8-sliced MTTKRP (§9b)
  int64_t parts_cap;
  int tiles_cap;
  int slice_nb;
  int64_t stage_cap;
  size_t total;
};

// R: the largest rank in the handle (Rs); sumRm: sum of the pool's model ranks (staging of P)
bool compute_offsets(int N, const int64_t* dims, int R, int64_t nsub, int hist_cap, const KernelInfo& ki,
                     Offsets* o, bool tf32 = false, int64_t sumRm = 0, bool i8 = false) {
  int64_t P = 1, sumI = 0, maxI = 0;
  for (int k = 0; k < N; ++k) {
    P *= dims[k];
    sumI += dims[k];
    maxI = std::max(maxI, dims[k]);
  }
  const int64_t C = nsub * R, ldu = rup(std::max<int64_t>(C, 1), 128);
  Layout L;
  o->T = L.take(rup(dims[0], 2) * (P / dims[0]) * 8);  // mode-0 pitch padded to even (TMA strides)
  o->T32hi = o->T32lo = o->T1hi = o->T1lo = 0;
  if (tf32) {  // FP32 hi/lo copies (16-byte strides): original layout and modes (1,0,2,..) permuted
    o->T32hi = L.take(rup(dims[0], 4) * (P / dims[0]) * 4);
    o->T32lo = L.take(rup(dims[0], 4) * (P / dims[0]) * 4);
    o->T1hi = L.take(rup(dims[1], 4) * (P / dims[1]) * 4);
    o->T1lo = L.take(rup(dims[1], 4) * (P / dims[1]) * 4);
  }
  for (int s = 0; s < 2; ++s)
    for (int k = 0; k < N; ++k) o->U[s][k] = L.take(dims[k] * ldu * 8);
  o->Ures = L.take(nsub * sumI * R * 8);
  o->parts_cap = 0;
  o->tiles_cap = 0;
  for (int n = 0; n < N; ++n) {
    int64_t pc;
    int tc;
    if (i8) {
      const I8Plan q = make_i8_plan(N, dims, n, C, ki);
      pc = (std::max<int64_t>(q.p.G, ki.nsm) + q.p.ntiles) * q.p.BN * kBM;
      tc = q.p.ntiles;
    } else {
      plan_bounds(mode_geo(N, dims, n), n, C, ki, &pc, &tc, tf32);
    }
    o->parts_cap = std::max(o->parts_cap, pc);
    o->tiles_cap = std::max(o->tiles_cap, tc);
  }
  if (tf32) {  // the FP32 path runs its last mode on the FP64 kernel when tol > 0 (reading A24)
    int64_t pc;
    int tc;
    plan_bounds(mode_geo(N, dims, N - 1), N - 1, C, ki, &pc, &tc, false);
    o->parts_cap = std::max(o->parts_cap, pc);
    o->tiles_cap = std::max(o->tiles_cap, tc);
  }
  o->parts = L.take(o->parts_cap * 8);
  for (int n = 0; n < N; ++n) o->tinfo[n] = L.take(plan_table_bytes(o->tiles_cap, ki.nsm * 8));
  // pre-reduced pieces (one per tile) for tiles split over many CTAs, and their 1-piece tables
  int64_t red_cap = 0;
  for (int n = 0; n < N; ++n) {
    const ModePlan q = i8 ? make_i8_plan(N, dims, n, C, ki).p : make_plan(mode_geo(N, dims, n), n, C, ki, tf32);
    red_cap = std::max<int64_t>(red_cap, (int64_t)q.ntiles * q.BN * kBM);
  }
  if (tf32) {
    const ModePlan q = make_plan(mode_geo(N, dims, N - 1), N - 1, C, ki, false);
    red_cap = std::max<int64_t>(red_cap, (int64_t)q.ntiles * q.BN * kBM);
  }
  o->tinfo64 = L.take(plan_table_bytes(o->tiles_cap, ki.nsm * 8));
  o->tinfo164 = L.take(o->tiles_cap * sizeof(TileInfo));
  o->red = L.take(red_cap * 8);
  for (int n = 0; n < N; ++n) o->tinfo1[n] = L.take(o->tiles_cap * sizeof(TileInfo));
  o->gram = L.take((size_t)N * nsub * R * R * 8);
  o->lambda = L.take(nsub * R * 8);
  o->normT2p = L.take(nsub * 8);
  o->fit = L.take(nsub * 8);
  o->fit_prev = L.take(nsub * 8);
  o->err = L.take(nsub * 8);
  o->hist = L.take(nsub * (int64_t)hist_cap * 8);
  o->slice = L.take(dims[0] * 8);
  int64_t J0 = P / dims[0];
  o->slice_nb = (int)std::min<int64_t>(J0, 2 * (int64_t)ki.nsm);
  o->slice_part = L.take((int64_t)o->slice_nb * dims[0] * 8);
  o->stage_cap = std::max<int64_t>(std::max<int64_t>(3 * maxI * R, nsub * maxI * R), 64);
  o->stage_cap = std::max<int64_t>(o->stage_cap, maxI * sumRm);
  o->stage = L.take(o->stage_cap * 8);
  o->iters = L.take(nsub * 4);
  o->flags = L.take(nsub * 4);
  o->active = L.take(nsub * 4);
  o->blk2sub = L.take(nsub * 4);
  o->map = L.take(ldu * 12);  // compaction column map (ldu ints) / converged-block table (3 per block)
  o->pglob = L.take(nsub * 8);
  o->srcoff = L.take(nsub * 8);
  o->srcld = L.take(nsub * 8);
  o->subR = L.take(nsub * 4);
  o->subRc = L.take(nsub * 4);
  o->blkcol = L.take(nsub * 4);
  o->dstoff = L.take(nsub * 8);
  for (int k = 0; k < kMaxModes; ++k) o->i8B[k] = o->i8eT[k] = o->i8dS[k] = 0;
  o->i8A = o->i8eU = o->i8st = o->i8dims = 0;
  if (i8) {  // per-mode T digits (fixed) + the U_q0 digits of the mode being updated
    int64_t amax = 0, cpmax = 0;
    for (int n = 0; n < N; ++n) {
      const I8Plan q = make_i8_plan(N, dims, n, C, ki);
      o->i8B[n] = L.take((size_t)kI8S * q.Jp * q.InP * q.KP);
      o->i8eT[n] = L.take((size_t)q.InP * 4);
      o->i8dS[n] = L.take((size_t)q.Jp * q.InP);
      // (the slab exponents are formed at create in the pieces buffer: Jp x InP ints)
      o->parts_cap = std::max<int64_t>(o->parts_cap, (int64_t)cdiv(q.Jp * q.InP * 4, 8));
      amax = std::max<int64_t>(amax, (int64_t)kI8S * q.CP * q.KP);
      cpmax = std::max<int64_t>(cpmax, q.CP);
    }
    o->i8A = L.take(amax);
    o->i8eU = L.take(cpmax * 4);
    o->i8st = L.take(kMaxModes * 8);
    o->i8dims = L.take(kMaxModes * 4);
  }
  // the pool's reference models (warm starts): mode n is col-major I_n x sumRm
  for (int k = 0; k < N; ++k) o->pref[k] = L.take(dims[k] * std::max<int64_t>(sumRm, R) * 8);
  o->aln = L.take(nsub * sumI * R * 8);  // aligned factors (NEXT #3), slot layout as Ures
  o->aperm = L.take(nsub * R * 4);
  o->asign = L.take(nsub * N * R * 4);
  o->acong = L.take(nsub * R * 8);
  o->asrc = L.take(nsub * N * 8);
  o->asld = L.take(nsub * N * 8);
  o->srcpg = L.take(nsub * 8);
  o->misc = L.take(256);  // [0] normT2 (double), [8] tol (double), [16] active_count (int), [24] sweeps (int)
  o->total = L.off + kAlign;  // slack for re-alignment of the caller's pointer
  return true;
}

bool valid_dims(int N, const int64_t* dims, int R) {
  if (N < 3 || N > JKCALS_MAX_MODES || !dims || R < 1 || R > kLgRMax) return false;
  int64_t P = 1;
  for (int k = 0; k < N; ++k) {
    if (dims[k] < 1) return false;
    P *= dims[k];
    if (P > ((int64_t)1 << 40)) return false;
  }
  if (dims[0] < 2) return false;
  for (int k = 0; k < N; ++k)
    if (P / dims[k] >= ((int64_t)1 << 31)) return false;  // J_n indexes in int32
  return true;
}

}  // namespace

// ---------------------------------------------------------------- the handle
struct jkcals_s {
  int N = 0;
  int64_t dims[kMaxModes] = {0};
  int R = 0;
  int64_t sub_begin = 0, sub_end = 0;  // group indices g; group g leaves out rows [g d, min(g d + d, I_0))
  int64_t d = 1;                       // delete-d group size (1 = leave-one-out)
  int64_t ngroups = 0;                 // ceil(I_0 / d); submodel s = model * ngroups + group
  int nmodels = 1;
  std::vector<int> ranks;              // rank of each pooled model
  bool mixed = false;                  // blocks of different widths (per-block rank / column tables)
  std::vector<int> h_subR, h_subRc, h_model;  // per local submodel: rank, rank prefix of its model, model
  std::vector<int64_t> h_group;        // per local submodel: group index g
  std::vector<int> h_blkcol;           // per live block: first column
  int64_t sumRm = 0;                   // sum of the pool's model ranks (reference store width)
  // slots: nsub = owned-at-create + spare; h_id[q] = global submodel id held by slot q (-1 free).
  // Submodels migrate between handles (tol-mode rebalancing) through export / import.
  std::vector<int64_t> h_id;
  int spare = 0;
  bool aligned = false;                // the aligned store holds jkcals_align's result
  int nsub = 0, K = 0, C = 0;
  int64_t ldu = 0, P = 0, I0p = 0;
  int hist_cap = 1;
  int device = 0;
  cudaStream_t stream = nullptr;  // the caller's stream: all work is ordered on it
  cudaStream_t cap = nullptr;     // private non-blocking stream used only for graph capture
  cudaStream_t es = nullptr;      // stream the enqueue_* helpers target (stream, or cap while capturing)
  char* ws = nullptr;
  size_t ws_bytes = 0;
  Offsets off;
  KernelInfo* ki = nullptr;
  int cur = 0;
  ModePlan plan[kMaxModes];
  CUtensorMap tmT[kMaxModes];
  CUtensorMap tmU[2][kMaxModes];
  std::vector<char> table[kMaxModes];  // host copy of each mode's device plan table
  bool red_on[kMaxModes] = {false};    // pieces of this mode pre-reduced before the epilogue
  std::vector<TileInfo> table1[kMaxModes];
  int tf32 = 0;                        // precision JKCALS_FP32: 3xTF32 tcgen05 MTTKRP
  // JKCALS_FP32 with tol > 0: the last mode's MTTKRP runs on the FP64 kernel so that the error and
  // fit behind the convergence test are FP64-accurate (reading A24)
  bool f64last = false;
  ModePlan plan64;
  CUtensorMap tmT64, tmU64[2];  // its T view and U_q0 slab maps (box width = its tile width + 4)
  bool red64 = false;
  std::vector<char> table64;
  std::vector<TileInfo> table164;
  // small tensors: the whole iterate as one cluster-resident launch (resident.cuh)
  struct {
    bool on = false, dirty = true;
    int cs = 1, Q = 1, kpc = 1, Cp = 4, slab = 1, rclass = 2;
    size_t smem = 0;
    ResArgs a;
    bool warp = false;  // tiny tensors: the warp-per-submodel kernel instead (warp_resident.cuh)
  } res;
  int i8 = 0;                          // precision JKCALS_FP64_I8: INT8-sliced FP64-accurate MTTKRP
  I8Plan i8q[kMaxModes];
  CUtensorMap tmA8[kMaxModes], tmB8[kMaxModes];
  CUtensorMap tmThi[kMaxModes], tmTlo[kMaxModes];
  cudaGraphExec_t gexec = nullptr;
  bool graph_ok = false;
  // tolerance mode: a CUDA-graph WHILE node repeats the sweep until the device-side trigger
  // (tol_decide_kernel) sees the call's sweep budget spent or enough convergence to compact
  cudaGraphExec_t gexec_tol = nullptr;
  bool tol_graph_bad = false;  // conditional nodes unavailable: per-sweep host check
  bool inited = false;
  bool ran = false;
  double tol_host = 0.0;
  int* pinned_count = nullptr;
  std::vector<int> h_blk2sub, h_stored;
  bool instrument = false;
  bool pdl = true;  // programmatic dependent launch between the sweep's kernels
  cudaEvent_t ev[2 * 2 * kMaxModes + 2] = {};
  double t_mttkrp[kMaxModes] = {0}, t_epi[kMaxModes] = {0};
  int64_t launches = 0;
  std::string err;

  template <class T>
  T* ptr(size_t o) { return reinterpret_cast<T*>(ws + o); }
  double* U(int n) { return ptr<double>(off.U[cur][n]); }
};

namespace {

// RAII NVTX range around the host API calls (iterate, compaction, re-plan, create)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

jkcals_status fail(jkcals_t h, jkcals_status st, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    h->err = buf;
  }
  return st;
}

#define CKH(h, x)                                                                                       \
  do {                                                                                                  \
    cudaError_t e_ = (x);                                                                               \
    if (e_ != cudaSuccess) return fail(h, JKCALS_E_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                             \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

jkcals_status replan(jkcals_t h) {
  NvtxRange nv("jkcals replan");
  h->res.dirty = true;
  for (int n = 0; n < h->N; ++n) {
    if (h->i8) {
      h->i8q[n] = make_i8_plan(h->N, h->dims, n, h->C, *h->ki);
      h->plan[n] = h->i8q[n].p;
    } else {
      h->plan[n] = make_plan(mode_geo(h->N, h->dims, n), n, h->C, *h->ki, h->tf32 != 0);
    }
    const ModePlan& p = h->plan[n];
    if (plan_parts_doubles(p) > h->off.parts_cap || p.ntiles > h->off.tiles_cap)
      return fail(h, JKCALS_E_OOM, "internal: plan exceeds workspace bounds");
    h->table[n] = pack_plan(p);
    CKH(h, cudaMemcpyAsync(h->ptr<TileInfo>(h->off.tinfo[n]), h->table[n].data(), h->table[n].size(),
                           cudaMemcpyHostToDevice, h->stream));
    // many pieces per tile: pre-reduce them with the whole GPU (kRedPieces, r01: G = 8 shard)
    int maxp = 0;
    for (const TileInfo& ti : p.tinfo) maxp = std::max(maxp, ti.npieces);
    const int red_thr = tuning().red_pieces >= 0 ? tuning().red_pieces : kRedPieces;
    // ... and only when each epilogue CTA would sum many pieces over many rows (r01: a syn200 shard
    // at G = 8, I_n x pieces = 200 x 59, gains 14 %; syn50, 50 x 48, loses 20 % to the extra launch)
    h->red_on[n] = red_thr > 0 && maxp > red_thr && (h->dims[n] * maxp > 8192 || tuning().red_pieces >= 0);
    h->table1[n].assign(p.ntiles, TileInfo{});
    for (int t = 0; t < p.ntiles; ++t) {
      h->table1[n][t].first_cta = 0;
      h->table1[n][t].npieces = 1;
      h->table1[n][t].piece_base = t;
      h->table1[n][t].pad_ = 0;
    }
    CKH(h, cudaMemcpyAsync(h->ptr<TileInfo>(h->off.tinfo1[n]), h->table1[n].data(), p.ntiles * sizeof(TileInfo),
                           cudaMemcpyHostToDevice, h->stream));
    if (h->i8) {  // 3-D boxes over the U_q0 digits (rebuilt each mode) and this mode's T digits
      const I8Plan& q = h->i8q[n];
      if (!make_tmap_i8(&h->tmA8[n], h->ptr<int8_t>(h->off.i8A), q.KP, q.CP, 128, q.variant == 2 ? 4 : kI8S) ||
          !make_tmap_i8(&h->tmB8[n], h->ptr<int8_t>(h->off.i8B[n]), q.KP, q.Jp * q.InP, kI8N))
        return fail(h, JKCALS_E_CUDA, "cuTensorMapEncodeTiled failed for the int8 digits of mode %d", n);
      continue;
    }
    // TMA descriptors: the tensor view of mode n and the U_q0 slab source of both U buffer sets
    if (!make_tmap_T(&h->tmT[n], h->ptr<double>(h->off.T), h->N, h->dims, h->I0p, n, p.BN, bnp_of(p.NT), p.KB))
      return fail(h, JKCALS_E_CUDA, "cuTensorMapEncodeTiled failed for the tensor view of mode %d", n);
    const int q0 = (n == 0) ? 1 : 0;
    for (int set = 0; set < 2; ++set)
      if (!make_tmap_U(&h->tmU[set][n], h->ptr<double>(h->off.U[set][q0]), h->dims[q0], h->ldu, p.BM + 4, p.KB))
        return fail(h, JKCALS_E_CUDA, "cuTensorMapEncodeTiled failed for U_%d", q0);
    if (h->tf32) {
      int64_t gd[4], gs[3];
      if (n == 0) {  // permuted copy (i_1, i_0, rest): q0 = i_1 contiguous, n = i_0
        const int64_t ld1 = rup(h->dims[1], 4), rest = h->P / (h->dims[0] * h->dims[1]);
        gd[0] = h->dims[1]; gd[1] = 1; gd[2] = h->dims[0]; gd[3] = rest;
        gs[0] = ld1; gs[1] = ld1; gs[2] = ld1 * h->dims[0];
        if (!make_tmap_T32(&h->tmThi[n], h->ptr<float>(h->off.T1hi), gd, gs, p.pair ? p.BN / 2 : p.BN) ||
            !make_tmap_T32(&h->tmTlo[n], h->ptr<float>(h->off.T1lo), gd, gs, p.pair ? p.BN / 2 : p.BN))
          return fail(h, JKCALS_E_CUDA, "cuTensorMapEncodeTiled failed for the fp32 view of mode 0");
      } else {
        const int64_t ld0 = rup(h->dims[0], 4);
        int64_t runA = 1, runB = 1, st_n = ld0;
        for (int m = 1; m < n; ++m) { runA *= h->dims[m]; st_n *= h->dims[m]; }
        for (int m = n + 1; m < h->N; ++m) runB *= h->dims[m];
        gd[0] = h->dims[0]; gd[1] = runA; gd[2] = h->dims[n]; gd[3] = runB;
        gs[0] = ld0; gs[1] = st_n; gs[2] = st_n * h->dims[n];
        if (!make_tmap_T32(&h->tmThi[n], h->ptr<float>(h->off.T32hi), gd, gs, p.pair ? p.BN / 2 : p.BN) ||
            !make_tmap_T32(&h->tmTlo[n], h->ptr<float>(h->off.T32lo), gd, gs, p.pair ? p.BN / 2 : p.BN))
          return fail(h, JKCALS_E_CUDA, "cuTensorMapEncodeTiled failed for the fp32 view of mode %d", n);
      }
    }
  }
  if (h->tf32) {  // the FP64 plan of the last mode (used when tol > 0)
    const int n = h->N - 1;
    h->plan64 = make_plan(mode_geo(h->N, h->dims, n), n, h->C, *h->ki, false);
    const ModePlan& p = h->plan64;
    if (plan_parts_doubles(p) > h->off.parts_cap || p.ntiles > h->off.tiles_cap)
      return fail(h, JKCALS_E_OOM, "internal: plan exceeds workspace bounds");
    h->table64 = pack_plan(p);
    CKH(h, cudaMemcpyAsync(h->ptr<TileInfo>(h->off.tinfo64), h->table64.data(), h->table64.size(),
                           cudaMemcpyHostToDevice, h->stream));
    int maxp = 0;
    for (const TileInfo& ti : p.tinfo) maxp = std::max(maxp, ti.npieces);
    h->red64 = maxp > kRedPieces && h->dims[n] * maxp > 8192;
    h->table164.assign(p.ntiles, TileInfo{});
    for (int t = 0; t < p.ntiles; ++t) h->table164[t] = TileInfo{0, 1, t, 0};
    CKH(h, cudaMemcpyAsync(h->ptr<TileInfo>(h->off.tinfo164), h->table164.data(), p.ntiles * sizeof(TileInfo),
                           cudaMemcpyHostToDevice, h->stream));
    if (!make_tmap_T(&h->tmT64, h->ptr<double>(h->off.T), h->N, h->dims, h->I0p, n, p.BN, bnp_of(p.NT), p.KB))
      return fail(h, JKCALS_E_CUDA, "cuTensorMapEncodeTiled failed for the FP64 view of mode %d", n);
    for (int set = 0; set < 2; ++set)  // q0 = 0 for the last mode (N >= 3)
      if (!make_tmap_U(&h->tmU64[set], h->ptr<double>(h->off.U[set][0]), h->dims[0], h->ldu, p.BM + 4, p.KB))
        return fail(h, JKCALS_E_CUDA, "cuTensorMapEncodeTiled failed for U_0 (FP64 last mode)");
  }
  CKH(h, cudaStreamSynchronize(h->stream));  // tinfo host vectors may change on the next replan
  if (h->gexec) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  if (h->gexec_tol) {
    cudaGraphExecDestroy(h->gexec_tol);
    h->gexec_tol = nullptr;
  }
  h->graph_ok = false;
  return JKCALS_OK;
}

EpiFns epi_fns(int rclass) {
  switch (rclass) {
    case 2: return epi_kernels_2();
    case 4: return epi_kernels_4();
    case 6: return epi_kernels_6();
    case 8: return epi_kernels_8();
    case 10: return epi_kernels_10();
    case 12: return epi_kernels_12();
    default: return epi_kernels_16();
  }
}

void launch_epi(jkcals_t h, int rclass, const EpiArgs& a, bool pdl) {
  const size_t dyn = (size_t)2 * a.In * (a.R | 1) * sizeof(double);  // odd row stride (epilogue.cuh)
  constexpr size_t kMaxDyn = 96 * 1024;  // opt-in set per device in kernel_info()
  const EpiFns f = epi_fns(rclass);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.gridDim = dim3(h->K);
  cfg.stream = h->es;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (dyn <= kMaxDyn && h->mixed) {
    cfg.blockDim = dim3(kEpi2Threads);
    cfg.dynamicSmemBytes = dyn;
    cudaLaunchKernelEx(&cfg, f.mixed, a);
  } else if (dyn <= kMaxDyn) {
    cfg.blockDim = dim3(kEpi2Threads);
    cfg.dynamicSmemBytes = dyn;
    cudaLaunchKernelEx(&cfg, f.smem, a);
  } else {
    cfg.blockDim = dim3(kEpiThreads);
    cfg.dynamicSmemBytes = 0;
    cudaLaunchKernelEx(&cfg, f.rows, a);
  }
}

jkcals_status enqueue_mode(jkcals_t h, int n, bool timed) {
  double* Uall[kMaxModes];
  for (int m = 0; m < h->N; ++m) Uall[m] = h->U(m);
  const bool f64 = h->tf32 && h->f64last && n == h->N - 1;  // FP32 path, tol > 0: last mode in FP64
  const ModePlan& p = f64 ? h->plan64 : h->plan[n];
  MttkrpView v = make_mview(h->N, h->dims, n, Uall, p.KB);
  MttkrpGeom g;
  g.C = h->C;
  g.ldu = h->ldu;
  g.nMt = p.nMt;
  g.nNt = p.nNt;
  g.KT = p.KT;
  g.units = p.units;
  g.G = p.G;
  const TileInfo* ti = h->ptr<TileInfo>(f64 ? h->off.tinfo64 : h->off.tinfo[n]);
  double* parts = h->ptr<double>(h->off.parts);
  if (timed) CKH(h, cudaEventRecord(h->ev[4 * n + 0], h->es));
  if (h->i8) {
    // U_q0 digits of the just-updated factor, then the INT8 MMAs
    const I8Plan& q = h->i8q[n];
    const int q0 = (n == 0) ? 1 : 0;
    int* eU = h->ptr<int>(h->off.i8eU);
    int8_t* A = h->ptr<int8_t>(h->off.i8A);
    col_exp_u_kernel<<<(int)cdiv(q.CP, 32), 256, 0, h->es>>>(Uall[q0], h->ldu, (int)q.Iq0, h->C, (int)q.CP, eU);
    CKH(h, cudaGetLastError());
    slice_u_i8_kernel<<<(int)cdiv(q.CP * q.KP, 256), 256, 0, h->es>>>(Uall[q0], h->ldu, (int)q.Iq0, h->C, (int)q.CP,
                                                                     (int)q.KP, eU, A);
    CKH(h, cudaGetLastError());
    I8Geom ig;
    ig.nMt = q.nMt;
    ig.nNt = q.nNt;
    ig.Jp = (int)q.Jp;
    ig.KS = (int)(q.KP / kI8K);
    ig.Kq = (int)q.Iq0;
    ig.units = p.units;
    ig.InP = (int)q.InP;
    ig.nslow = h->N - 2;
    int sl = 0;
    for (int m = 0; m < h->N; ++m) {
      if (m == n || m == q0) continue;
      ig.sdim[sl] = (int)h->dims[m];
      ig.Us[sl] = Uall[m];
      ++sl;
    }
    for (; sl < kMaxModes - 2; ++sl) {
      ig.sdim[sl] = 1;
      ig.Us[sl] = nullptr;
    }
    ig.ldu = h->ldu;
#ifdef JKCALS_DEV_PROBES  // timing-probe builds only (tools/i8_probe.py); results are wrong when set
    ig.probe = tuning().i8_probe;
#endif
    ig.eT = h->ptr<int>(h->off.i8eT[n]);
    ig.dS = h->ptr<int8_t>(h->off.i8dS[n]);
    ig.eU = eU;
    CKH(h, launch_i8(q, h->tmA8[n], h->tmB8[n], ig, ti, parts, h->es));
  } else if (h->tf32 && !f64) {
    TfGeom tg;
    tg.C = h->C;
    tg.ldu = h->ldu;
    tg.nMt = p.pair ? p.nMt2 : p.nMt;
    tg.nMt1 = p.nMt;
    tg.nNt = p.nNt;
    tg.BN = p.BN;
    tg.KT = p.KT;
    tg.units = p.units;
    tg.G = p.G;
    if (n == 0) v.runA = 1;  // the n = 0 fp32 view carries j' in its runB coordinate
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (h->pdl && !timed) ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;  // (PAIR: 2-CTA clusters)
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.gridDim = dim3(p.pair ? 2 * p.G : p.G);
    cfg.blockDim = dim3(kTfThreads);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = h->es;
    cfg.attrs = attr;
    cfg.numAttrs = p.pair ? 2 : 1;
    tg.stages = p.ST4;
    tg.jm = p.JM;  // (the chain length stays 128 products x 3: kTfChunk 16-k sub-tiles)
    tg.chunk = tuning().tf32_chunk > 0 ? tuning().tf32_chunk : std::max(1, kTfChunk / p.JM);
    tg.probe = 0;
#ifdef JKCALS_DEV_PROBES  // timing-probe builds only (results are wrong when set)
    tg.probe = tuning().i8_probe;
#endif
    CKH(h, cudaLaunchKernelEx(&cfg, tf32_kernel(p.ST4, p.pair != 0, p.JM), h->tmThi[n], h->tmTlo[n], h->tmU[h->cur][n], v,
                              tg, ti, parts));
  } else {
    MttkrpFn fn = h->ki->fn[p.KV][p.WV][p.KM][p.ST4][p.NT - 1];
    // programmatic dependent launch: this grid may start (prologue) while the previous kernel
    // drains; the kernel waits (griddepcontrol.wait) before touching its inputs
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (h->pdl && !timed) ? 1 : 0;
    cfg.gridDim = dim3(p.G);
    cfg.blockDim = dim3((kWMs[p.WV] + 1) * 32);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = h->es;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CKH(h, cudaLaunchKernelEx(&cfg, fn, f64 ? h->tmT64 : h->tmT[n], f64 ? h->tmU64[h->cur] : h->tmU[h->cur][n], v,
                              g, ti, parts));
  }
  CKH(h, cudaGetLastError());
  if (timed) CKH(h, cudaEventRecord(h->ev[4 * n + 1], h->es));
  const double* epi_parts = parts;
  const TileInfo* epi_ti = ti;
  if (f64 ? h->red64 : h->red_on[n]) {  // pre-reduce the pieces across the whole GPU (PDL-chained)
    const int tile_elems = p.BN * p.BM;
    const int64_t tot = (int64_t)p.ntiles * tile_elems;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (h->pdl && !timed) ? 1 : 0;
    cfg.gridDim = dim3((unsigned)(tot / 32));  // one CTA per 32 elements (tile_elems % 32 == 0)
    cfg.blockDim = dim3(32 * kRedWarps);
    cfg.stream = h->es;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    double* red = h->ptr<double>(h->off.red);
    CKH(h, cudaLaunchKernelEx(&cfg, reduce_pieces_kernel, (const double*)parts, ti, p.ntiles, tile_elems, red));
    epi_parts = red;
    epi_ti = h->ptr<TileInfo>(f64 ? h->off.tinfo164 : h->off.tinfo1[n]);
  }
  EpiArgs a;
  a.N = h->N;
  a.n = n;
  a.R = h->R;
  a.subR = h->mixed ? h->ptr<int>(h->off.subR) : nullptr;
  a.blkcol = h->mixed ? h->ptr<int>(h->off.blkcol) : nullptr;
  a.In = (int)h->dims[n];
  a.ldu = h->ldu;
  a.nsub = h->nsub;
  a.U = Uall[n];
  a.blk2sub = h->ptr<int>(h->off.blk2sub);
  a.pglob = h->ptr<int64_t>(h->off.pglob);
  a.d = (int)h->d;
  a.parts = epi_parts;
  a.tinfo = epi_ti;
  a.BM = p.BM;
  a.BN = p.BN;
  a.nMt = p.nMt;
  a.gram = h->ptr<double>(h->off.gram);
  a.lambda = h->ptr<double>(h->off.lambda);
  a.normT2p = h->ptr<double>(h->off.normT2p);
  a.fit = h->ptr<double>(h->off.fit);
  a.fit_prev = h->ptr<double>(h->off.fit_prev);
  a.err = h->ptr<double>(h->off.err);
  a.iters = h->ptr<int>(h->off.iters);
  a.flags = h->ptr<int>(h->off.flags);
  a.active = h->ptr<int>(h->off.active);
  a.hist = h->ptr<double>(h->off.hist);
  a.hist_cap = h->hist_cap;
  a.tol = reinterpret_cast<const double*>(h->ws + h->off.misc + 8);
  a.active_count = reinterpret_cast<int*>(h->ws + h->off.misc + 16);
  const bool pdl = h->pdl && !timed;
  if (h->R > 16) {  // ranks 17..32: the streaming large-rank epilogue (any I_n, mixed pools too)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.gridDim = dim3(h->K);
    cfg.blockDim = dim3(kLgThreads);
    cfg.dynamicSmemBytes = epi_large_smem_bytes();
    cfg.stream = h->es;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (!a.subR) a.subR = h->ptr<int>(h->off.subR);  // the large kernel reads per-block ranks
    if (!a.blkcol) a.blkcol = h->ptr<int>(h->off.blkcol);
    cudaLaunchKernelEx(&cfg, epi_large_kernel(), a);
  } else {
    launch_epi(h, h->R <= 2 ? 2 : h->R <= 4 ? 4 : h->R <= 6 ? 6 : h->R <= 8 ? 8 : h->R <= 10 ? 10 : h->R <= 12 ? 12 : 16,
               a, pdl);
  }
  CKH(h, cudaGetLastError());
  if (timed) CKH(h, cudaEventRecord(h->ev[4 * n + 2], h->es));
  return JKCALS_OK;
}

jkcals_status enqueue_sweep(jkcals_t h, bool timed) {
  // (the per-sweep active counter is reset by the mode-0 epilogue, so a sweep is kernels only)
  for (int n = 0; n < h->N; ++n) {
    jkcals_status st = enqueue_mode(h, n, timed);
    if (st != JKCALS_OK) return st;
  }
  return JKCALS_OK;
}

jkcals_status ensure_graph(jkcals_t h) {
  if (h->graph_ok) return JKCALS_OK;
  cudaGraph_t graph = nullptr;
  // capture on a private stream (the caller's may be the legacy default stream, which
  // cannot be captured); the instantiated graph is then launched on the caller's stream
  CKH(h, cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
  h->es = h->cap;
  jkcals_status st = enqueue_sweep(h, false);
  h->es = h->stream;
  cudaError_t e = cudaStreamEndCapture(h->cap, &graph);
  if (st != JKCALS_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return fail(h, JKCALS_E_CUDA, "graph capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&h->gexec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(h, JKCALS_E_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
  h->graph_ok = true;
  return JKCALS_OK;
}

// Tolerance mode without a host round trip per sweep: graph = WHILE(cond) { sweep; tol_decide },
// the condition set on the device from the active-submodel count (misc+16) against the compaction
// threshold and this call's sweep budget (misc+32 / +36, written by the host before each launch).
// The host wakes only when the loop exits: to compact (a8), or at the end of the call.
jkcals_status ensure_tol_graph(jkcals_t h) {
  if (h->gexec_tol || h->tol_graph_bad || tuning().tol_host_loop) return JKCALS_OK;
  cudaGraph_t graph = nullptr;
  cudaGraphConditionalHandle hnd;
  auto bad = [&](cudaError_t e) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    h->tol_graph_bad = true;  // (logged in last_error; iterate falls back to the per-sweep check)
    h->err = std::string("conditional graph unavailable: ") + cudaGetErrorString(e);
    return JKCALS_OK;
  };
  cudaError_t e = cudaGraphCreate(&graph, 0);
  if (e != cudaSuccess) return bad(e);
  e = cudaGraphConditionalHandleCreate(&hnd, graph, 1, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) return bad(e);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hnd;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, graph, nullptr, 0, &cp);
  if (e != cudaSuccess) return bad(e);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(h->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return bad(e);
  h->es = h->cap;
  jkcals_status st = enqueue_sweep(h, false);
  tol_decide_kernel<<<1, 1, 0, h->cap>>>(reinterpret_cast<int*>(h->ws + h->off.misc), hnd);
  h->es = h->stream;
  cudaGraph_t got = nullptr;
  e = cudaStreamEndCapture(h->cap, &got);
  if (st != JKCALS_OK) {
    cudaGraphDestroy(graph);
    return st;
  }
  if (e != cudaSuccess) return bad(e);
  e = cudaGraphInstantiate(&h->gexec_tol, graph, 0);
  if (e != cudaSuccess) {
    h->gexec_tol = nullptr;
    return bad(e);
  }
  cudaGraphDestroy(graph);
  return JKCALS_OK;
}

template <int RMAX>
void launch_gram(jkcals_t h, int n) {
  gram_kernel<RMAX><<<h->K, kEpiThreads, 0, h->stream>>>(h->U(n), (int)h->dims[n], h->ldu, h->R,
                                                          h->ptr<int>(h->off.blk2sub), h->ptr<int>(h->off.blkcol),
                                                          h->ptr<int>(h->off.subR), h->nsub, n,
                                                          h->ptr<double>(h->off.gram));
}

jkcals_status compute_grams(jkcals_t h) {
  for (int n = 0; n < h->N; ++n) {
    if (h->R <= 4) launch_gram<4>(h, n);
    else if (h->R <= 8) launch_gram<8>(h, n);
    else if (h->R <= 16) launch_gram<16>(h, n);
    else
      gram_large_kernel_fn()<<<h->K, kLgThreads, 0, h->stream>>>(h->U(n), (int)h->dims[n], h->ldu, h->R,
                                                            h->ptr<int>(h->off.blk2sub), h->ptr<int>(h->off.blkcol),
                                                            h->ptr<int>(h->off.subR), h->nsub, n,
                                                            h->ptr<double>(h->off.gram));
    CKH(h, cudaGetLastError());
  }
  return JKCALS_OK;
}

// upload the live-block column table (prefix sums of the live blocks' ranks) and set C
jkcals_status set_blocks(jkcals_t h, const std::vector<int>& b2s) {
  h->h_blk2sub = b2s;
  h->K = (int)b2s.size();
  h->h_blkcol.assign(h->K, 0);
  int c = 0;
  for (int k = 0; k < h->K; ++k) {
    h->h_blkcol[k] = c;
    c += h->h_subR[b2s[k]];
  }
  h->C = c;
  if (h->K > 0) {
    CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.blk2sub), b2s.data(), sizeof(int) * h->K, cudaMemcpyHostToDevice,
                           h->stream));
    CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.blkcol), h->h_blkcol.data(), sizeof(int) * h->K,
                           cudaMemcpyHostToDevice, h->stream));
  }
  CKH(h, cudaStreamSynchronize(h->stream));  // host vectors are the copy sources
  return JKCALS_OK;
}

int64_t sum_dims(const jkcals_s* h) {
  int64_t sumI = 0;
  for (int n = 0; n < h->N; ++n) sumI += h->dims[n];
  return sumI;
}

// gather the blocks of `keep` (in that order, all currently live) to the front of the other
// multi-factor buffer set and re-plan
jkcals_status relayout(jkcals_t h, const std::vector<int>& keep) {
  std::vector<int> colmap;
  for (int sub : keep) {
    int k = -1;
    for (int j = 0; j < h->K; ++j)
      if (h->h_blk2sub[j] == sub) k = j;
    if (k < 0) return fail(h, JKCALS_E_STATE, "internal: slot %d is not live", sub);
    for (int r = 0; r < h->h_subR[sub]; ++r) colmap.push_back(h->h_blkcol[k] + r);
  }
  const int Cnew = (int)colmap.size();
  if (Cnew > 0)
    CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.map), colmap.data(), sizeof(int) * Cnew, cudaMemcpyHostToDevice,
                           h->stream));
  const int other = h->cur ^ 1;
  for (int n = 0; n < h->N; ++n) {
    int64_t tot = h->dims[n] * h->ldu;
    gather_blocks_kernel<<<(int)cdiv(tot, 256), 256, 0, h->stream>>>(
        h->U(n), h->ptr<double>(h->off.U[other][n]), (int)h->dims[n], h->ldu, h->ptr<int>(h->off.map), Cnew);
    CKH(h, cudaGetLastError());
  }
  jkcals_status st = set_blocks(h, keep);  // synchronises (colmap is a host temporary)
  if (st != JKCALS_OK) return st;
  h->cur = other;
  if (!keep.empty()) return replan(h);
  return JKCALS_OK;
}

// (a8) compact: store converged live blocks, gather the active ones to the front.
jkcals_status compact(jkcals_t h) {
  NvtxRange nv("jkcals compact");
  std::vector<int> act(h->nsub);
  CKH(h, cudaMemcpyAsync(act.data(), h->ptr<int>(h->off.active), sizeof(int) * h->nsub, cudaMemcpyDeviceToHost,
                         h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  const int64_t sumI = sum_dims(h);
  std::vector<int> keep, tab;  // tab: (column, rank, slot) of each block to store
  int rmax = 1;
  for (int k = 0; k < h->K; ++k) {
    const int sub = h->h_blk2sub[k], R = h->h_subR[sub], col = h->h_blkcol[k];
    if (act[sub]) {
      keep.push_back(sub);
    } else if (!h->h_stored[sub]) {
      tab.insert(tab.end(), {col, R, sub});
      rmax = std::max(rmax, R);
      h->h_stored[sub] = 1;
    }
  }
  if (!tab.empty()) {  // one launch per mode for all newly converged blocks (r02: was N per block)
    const int nst = (int)tab.size() / 3;
    int* dtab = h->ptr<int>(h->off.map);  // (free here: relayout uploads its column map after these)
    CKH(h, cudaMemcpyAsync(dtab, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice, h->stream));
    int64_t sumIprev = 0;
    for (int n = 0; n < h->N; ++n) {
      const int I = (int)h->dims[n];
      store_blocks_kernel<<<dim3((unsigned)cdiv((int64_t)I * rmax, 256), (unsigned)nst), 256, 0, h->stream>>>(
          h->U(n), I, h->ldu, dtab, sumI * h->R, sumIprev, h->ptr<double>(h->off.Ures));
      CKH(h, cudaGetLastError());
      sumIprev += I;
    }
  }
  if ((int)keep.size() == h->K) return JKCALS_OK;
  return relayout(h, keep);
}

// slot holding global submodel id p, or -1
int slot_of(const jkcals_s* h, int64_t p) {
  if (p >= h->sub_begin && p < h->sub_end && p - h->sub_begin < h->nsub && h->h_id[p - h->sub_begin] == p)
    return (int)(p - h->sub_begin);
  for (int q = 0; q < h->nsub; ++q)
    if (h->h_id[q] == p && p >= 0) return q;
  return -1;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

// pool geometry shared by the workspace-size query and creation
struct PoolGeo {
  int Rs = 0;          // largest rank a slot may hold (all models' max when there are spare slots)
  int64_t sumRm = 0;   // sum of all model ranks
  int64_t ngroups = 0;
  int64_t C = 0;       // fused width of the owned submodels
  int64_t nslot = 0;   // owned + spare
};

static bool pool_geo(const jkcals_config* c, PoolGeo* g) {
  if (!c || c->nmodels < 1 || !c->ranks || !c->dims || c->ndims < 3 || c->ndims > JKCALS_MAX_MODES) return false;
  const int64_t* dims = c->dims;
  const int64_t d = c->d;
  if (dims[0] < 2 || d < 0 || (d > 1 && 2 * d > dims[0]) || c->spare < 0 || c->hist_cap < 1) return false;
  if (c->prec != JKCALS_FP64 && c->prec != JKCALS_FP32 && c->prec != JKCALS_FP64_I8) return false;
  for (int m = 0; m < c->nmodels; ++m)
    if (c->ranks[m] < 1 || c->ranks[m] > kLgRMax) return false;
  if (c->prec == JKCALS_FP64_I8 && !i8_k_ok(c->ndims, dims)) return false;
  // d = 0: plain CALS (§3.3): one model per id, nothing left out
  g->ngroups = d == 0 ? 1 : (dims[0] + d - 1) / d;
  if (c->sub_begin < 0 || c->sub_end <= c->sub_begin || c->sub_end > (int64_t)c->nmodels * g->ngroups) return false;
  g->Rs = 0;
  g->C = 0;
  g->sumRm = 0;
  int rmax = 0;
  for (int m = 0; m < c->nmodels; ++m) {
    g->sumRm += c->ranks[m];
    rmax = std::max(rmax, c->ranks[m]);
  }
  for (int64_t s = c->sub_begin; s < c->sub_end; ++s) {
    const int R = c->ranks[s / g->ngroups];
    g->Rs = std::max(g->Rs, R);
    g->C += R;
  }
  if (c->spare > 0) g->Rs = rmax;
  g->nslot = c->sub_end - c->sub_begin + c->spare;
  return valid_dims(c->ndims, dims, g->Rs) && g->nslot * g->Rs <= (1 << 24);
}

size_t jkcals_config_workspace_bytes(const jkcals_config* c) {
  PoolGeo g;
  if (!pool_geo(c, &g)) return 0;
  KernelInfo* ki = kernel_info(c->device, nullptr);
  if (!ki) return 0;
  Offsets o;
  compute_offsets(c->ndims, c->dims, g.Rs, g.nslot, c->hist_cap, *ki, &o, c->prec == JKCALS_FP32, g.sumRm,
                  c->prec == JKCALS_FP64_I8);
  return o.total;
}

static jkcals_config make_cfg(int ndims, const int64_t* dims, int nmodels, const int* ranks, int64_t d,
                              int64_t sub_begin, int64_t sub_end, jkcals_precision prec, int hist_cap, int device) {
  jkcals_config c = {};
  c.ndims = ndims;
  c.dims = dims;
  c.nmodels = nmodels;
  c.ranks = ranks;
  c.d = d;
  c.sub_begin = sub_begin;
  c.sub_end = sub_end;
  c.spare = 0;
  c.prec = prec;
  c.hist_cap = hist_cap;
  c.device = device;
  return c;
}

size_t jkcals_pool_workspace_bytes(int ndims, const int64_t* dims, int nmodels, const int* ranks, int64_t d,
                                   int64_t sub_begin, int64_t sub_end, jkcals_precision prec, int hist_cap,
                                   int device) {
  jkcals_config c = make_cfg(ndims, dims, nmodels, ranks, d, sub_begin, sub_end, prec, hist_cap, device);
  return jkcals_config_workspace_bytes(&c);
}

size_t jkcals_workspace_bytes(int ndims, const int64_t* dims, int rank, int64_t n_sub, jkcals_precision prec,
                              int hist_cap, int device) {
  if (!dims || ndims < 3 || n_sub < 1 || n_sub > dims[0]) return 0;
  return jkcals_pool_workspace_bytes(ndims, dims, 1, &rank, 1, 0, n_sub, prec, hist_cap, device);
}

// rows of mode 0 left out by group g (the last group may be smaller)
static int64_t group_rows(const jkcals_s* h, int64_t g) { return std::min(h->d, h->dims[0] - g * h->d); }

jkcals_status jkcals_create(jkcals_t* out, int ndims, const int64_t* dims, int rank, int64_t sub_begin,
                            int64_t sub_end, const double* tensor, int tensor_is_device, jkcals_precision prec,
                            int device, void* cuda_stream, void* workspace, size_t workspace_bytes, int hist_cap) {
  return jkcals_create_pool(out, ndims, dims, 1, &rank, 1, sub_begin, sub_end, tensor, tensor_is_device, prec,
                            device, cuda_stream, workspace, workspace_bytes, hist_cap);
}

jkcals_status jkcals_create_d(jkcals_t* out, int ndims, const int64_t* dims, int rank, int64_t d, int64_t sub_begin,
                              int64_t sub_end, const double* tensor, int tensor_is_device, jkcals_precision prec,
                              int device, void* cuda_stream, void* workspace, size_t workspace_bytes, int hist_cap) {
  if (d < 1) return JKCALS_E_ARG;
  return jkcals_create_pool(out, ndims, dims, 1, &rank, d, sub_begin, sub_end, tensor, tensor_is_device, prec,
                            device, cuda_stream, workspace, workspace_bytes, hist_cap);
}

jkcals_status jkcals_create_pool(jkcals_t* out, int ndims, const int64_t* dims, int nmodels, const int* ranks,
                                 int64_t d, int64_t sub_begin, int64_t sub_end, const double* tensor,
                                 int tensor_is_device, jkcals_precision prec, int device, void* cuda_stream,
                                 void* workspace, size_t workspace_bytes, int hist_cap) {
  jkcals_config c = make_cfg(ndims, dims, nmodels, ranks, d, sub_begin, sub_end, prec, hist_cap, device);
  return jkcals_create_config(out, &c, tensor, tensor_is_device, cuda_stream, workspace, workspace_bytes);
}

jkcals_status jkcals_create_config(jkcals_t* out, const jkcals_config* cfg, const double* tensor,
                                   int tensor_is_device, void* cuda_stream, void* workspace,
                                   size_t workspace_bytes) {
  if (!out) return JKCALS_E_ARG;
  *out = nullptr;
  NvtxRange nv("jkcals_create");
  PoolGeo pg0;
  if (!pool_geo(cfg, &pg0) || !tensor || !workspace) return JKCALS_E_ARG;
  const int ndims = cfg->ndims, nmodels = cfg->nmodels, hist_cap = cfg->hist_cap, device = cfg->device;
  const int64_t* dims = cfg->dims;
  const int* ranks = cfg->ranks;
  const int64_t d = cfg->d, sub_begin = cfg->sub_begin, sub_end = cfg->sub_end;
  const jkcals_precision prec = cfg->prec;
  DeviceGuard dg(device);
  std::string kerr;
  KernelInfo* ki = kernel_info(device, &kerr);
  if (!ki) return JKCALS_E_CUDA;
  jkcals_t h = new jkcals_s();
  h->N = ndims;
  for (int k = 0; k < ndims; ++k) h->dims[k] = dims[k];
  h->R = pg0.Rs;
  h->sub_begin = sub_begin;
  h->sub_end = sub_end;
  h->d = d;
  h->ngroups = pg0.ngroups;
  h->nmodels = nmodels;
  h->ranks.assign(ranks, ranks + nmodels);
  h->sumRm = pg0.sumRm;
  h->spare = cfg->spare;
  h->nsub = (int)pg0.nslot;
  const int nown = (int)(sub_end - sub_begin);
  std::vector<int> rc(nmodels, 0);
  for (int m = 1; m < nmodels; ++m) rc[m] = rc[m - 1] + ranks[m - 1];
  for (int q = 0; q < h->nsub; ++q) {
    if (q < nown) {
      const int64_t s = sub_begin + q;
      const int m = (int)(s / h->ngroups);
      h->h_id.push_back(s);
      h->h_model.push_back(m);
      h->h_group.push_back(s % h->ngroups);
      h->h_subR.push_back(ranks[m]);
      h->h_subRc.push_back(rc[m]);
      if (ranks[m] != h->R) h->mixed = true;
    } else {  // spare slot
      h->h_id.push_back(-1);
      h->h_model.push_back(-1);
      h->h_group.push_back(0);
      h->h_subR.push_back(0);
      h->h_subRc.push_back(0);
    }
  }
  if (h->spare > 0)
    for (int m = 0; m < nmodels; ++m)
      if (ranks[m] != h->R) h->mixed = true;
  h->K = nown;
  h->C = (int)pg0.C;
  h->ldu = rup(std::max<int64_t>(pg0.C + (int64_t)h->spare * h->R, 1), 128);  // room for imports
  h->P = 1;
  for (int k = 0; k < ndims; ++k) h->P *= dims[k];
  h->I0p = rup(dims[0], 2);
  h->hist_cap = hist_cap;
  h->device = device;
  h->stream = static_cast<cudaStream_t>(cuda_stream);
  h->es = h->stream;
  h->ki = ki;
  h->tf32 = (prec == JKCALS_FP32) ? 1 : 0;
  h->i8 = (prec == JKCALS_FP64_I8) ? 1 : 0;
  compute_offsets(ndims, dims, h->R, h->nsub, hist_cap, *ki, &h->off, h->tf32 != 0, pg0.sumRm, h->i8 != 0);
  // align the caller's pointer
  uintptr_t base = reinterpret_cast<uintptr_t>(workspace);
  uintptr_t aligned = (base + kAlign - 1) & ~(uintptr_t)(kAlign - 1);
  if (workspace_bytes < h->off.total) {
    delete h;
    return JKCALS_E_OOM;
  }
  h->ws = reinterpret_cast<char*>(aligned);
  h->ws_bytes = workspace_bytes - (aligned - base);
  *out = h;

  CKH(h, cudaMallocHost(&h->pinned_count, 4 * sizeof(int)));
  CKH(h, cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
  for (auto& e : h->ev) CKH(h, cudaEventCreate(&e));
  // T into the workspace with its mode-0 pitch padded to I0p (zero pad row when I0 is odd)
  if (h->I0p != dims[0])
    CKH(h, cudaMemsetAsync(h->ptr<double>(h->off.T), 0, sizeof(double) * h->I0p * (h->P / dims[0]), h->stream));
  CKH(h, cudaMemcpy2DAsync(h->ptr<double>(h->off.T), sizeof(double) * h->I0p, tensor, sizeof(double) * dims[0],
                           sizeof(double) * dims[0], h->P / dims[0],
                           tensor_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, h->stream));
  std::vector<int64_t> pg(h->nsub);
  std::vector<int> b2s(nown);
  for (int q = 0; q < h->nsub; ++q) pg[q] = h->h_group[q] * d;  // first left-out row of the group
  for (int q = 0; q < nown; ++q) b2s[q] = q;
  h->h_stored.assign(h->nsub, 0);
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.pglob), pg.data(), sizeof(int64_t) * h->nsub,
                         cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.subR), h->h_subR.data(), sizeof(int) * h->nsub, cudaMemcpyHostToDevice,
                         h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.subRc), h->h_subRc.data(), sizeof(int) * h->nsub,
                         cudaMemcpyHostToDevice, h->stream));
  {
    jkcals_status st0 = set_blocks(h, b2s);
    if (st0 != JKCALS_OK) return st0;
  }
  // (a0) slice norms, ||T||^2, ||T_-p||^2
  const int64_t I0 = dims[0], J0 = h->P / I0;
  const int nb = h->off.slice_nb;
  const int64_t chunk = cdiv(J0, nb);
  const int nb_eff = (int)cdiv(J0, chunk);
  slice_norms_partial_kernel<<<nb_eff, 256, 0, h->stream>>>(h->ptr<double>(h->off.T), I0, h->I0p, J0, chunk,
                                                             h->ptr<double>(h->off.slice_part));
  CKH(h, cudaGetLastError());
  slice_norms_final_kernel<<<1, 256, 0, h->stream>>>(h->ptr<double>(h->off.slice_part), nb_eff, I0,
                                                     h->ptr<double>(h->off.slice),
                                                     reinterpret_cast<double*>(h->ws + h->off.misc),
                                                     h->ptr<int64_t>(h->off.pglob), (int)d, h->nsub,
                                                     h->ptr<double>(h->off.normT2p));
  CKH(h, cudaGetLastError());
  double nt2 = 0;
  CKH(h, cudaMemcpyAsync(&nt2, h->ws + h->off.misc, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  if (!std::isfinite(nt2)) return fail(h, JKCALS_E_NONFINITE, "tensor contains non-finite values");
  if (h->tf32) {  // FP32 hi/lo copies of T for the 3xTF32 path (original + modes-(1,0) permuted)
    const int64_t I1 = dims[1], rest = h->P / (dims[0] * dims[1]);
    const int64_t ld0 = rup(dims[0], 4), ld1 = rup(dims[1], 4);
    CKH(h, cudaMemsetAsync(h->ptr<float>(h->off.T32hi), 0, ld0 * (h->P / dims[0]) * 4, h->stream));
    CKH(h, cudaMemsetAsync(h->ptr<float>(h->off.T32lo), 0, ld0 * (h->P / dims[0]) * 4, h->stream));
    CKH(h, cudaMemsetAsync(h->ptr<float>(h->off.T1hi), 0, ld1 * (h->P / dims[1]) * 4, h->stream));
    CKH(h, cudaMemsetAsync(h->ptr<float>(h->off.T1lo), 0, ld1 * (h->P / dims[1]) * 4, h->stream));
    const int nbk = (int)cdiv(h->P, 256);
    split_tf32_kernel<<<nbk, 256, 0, h->stream>>>(h->ptr<double>(h->off.T), dims[0], h->I0p, I1, rest, 0, ld0,
                                                  h->ptr<float>(h->off.T32hi), h->ptr<float>(h->off.T32lo));
    CKH(h, cudaGetLastError());
    split_tf32_kernel<<<nbk, 256, 0, h->stream>>>(h->ptr<double>(h->off.T), dims[0], h->I0p, I1, rest, 1, ld1,
                                                  h->ptr<float>(h->off.T1hi), h->ptr<float>(h->off.T1lo));
    CKH(h, cudaGetLastError());
  }
  if (h->i8) {  // per-mode INT8 digits of T with per-row scales (fixed for the handle's life)
    int64_t stv[kMaxModes];
    int dv[kMaxModes];
    stv[0] = 1;
    stv[1] = h->I0p;
    for (int m = 2; m < ndims; ++m) stv[m] = stv[m - 1] * dims[m - 1];
    for (int m = 0; m < ndims; ++m) dv[m] = (int)dims[m];
    int64_t* st_d = h->ptr<int64_t>(h->off.i8st);
    int* dims_d = h->ptr<int>(h->off.i8dims);
    CKH(h, cudaMemcpyAsync(st_d, stv, 8 * ndims, cudaMemcpyHostToDevice, h->stream));
    CKH(h, cudaMemcpyAsync(dims_d, dv, 4 * ndims, cudaMemcpyHostToDevice, h->stream));
    for (int n = 0; n < ndims; ++n) {
      const I8Plan q = make_i8_plan(ndims, dims, n, h->C, *ki);
      int* eT = h->ptr<int>(h->off.i8eT[n]);
      int* eS = h->ptr<int>(h->off.parts);  // scratch: slab exponents of this mode
      const int q0 = (n == 0) ? 1 : 0;
      slab_exp_t_kernel<<<(int)cdiv(q.Jp * q.InP, 256), 256, 0, h->stream>>>(
          h->ptr<double>(h->off.T), ndims, st_d, dims_d, n, q0, (int)q.In, (int)q.InP, (int)q.Iq0, q.Jp, eS);
      row_ref_exp_kernel<<<(int)q.InP, 256, 0, h->stream>>>(eS, (int)q.InP, q.Jp, eT, h->ptr<int8_t>(h->off.i8dS[n]));
      slice_t_i8_kernel<<<(int)cdiv(q.Jp * q.InP * q.KP, 256), 256, 0, h->stream>>>(
          h->ptr<double>(h->off.T), ndims, st_d, dims_d, n, q0, (int)q.In, (int)q.InP, (int)q.Iq0, (int)q.KP, q.Jp,
          eS, h->ptr<int8_t>(h->off.i8B[n]));
      CKH(h, cudaGetLastError());
    }
    CKH(h, cudaStreamSynchronize(h->stream));  // stv / dv are host temporaries
  }
  jkcals_status st = replan(h);
  if (st != JKCALS_OK) return st;
  return JKCALS_OK;
}

// the live block of local submodel `sub`, or -1
static int block_of(jkcals_t h, int sub) {
  for (int k = 0; k < h->K; ++k)
    if (h->h_blk2sub[k] == sub) return k;
  return -1;
}

jkcals_status jkcals_set_init(jkcals_t h, const double* const* P) {
  if (!h || !P) return JKCALS_E_ARG;
  DeviceGuard dg(h->device);
  for (int m = 0; m < h->nmodels; ++m)
    for (int n = 0; n < h->N; ++n) {
      const double* Pm = P[m * h->N + n];
      if (!Pm) return fail(h, JKCALS_E_ARG, "P[%d] is NULL", m * h->N + n);
      for (int64_t e = 0; e < h->dims[n] * h->ranks[m]; ++e)
        if (!std::isfinite(Pm[e])) return fail(h, JKCALS_E_NONFINITE, "P[%d] has a non-finite entry", m * h->N + n);
    }
  // full reset of the fused layout (undo any compaction): one block per owned slot
  std::vector<int> b2s;
  for (int q = 0; q < h->nsub; ++q)
    if (h->h_id[q] >= 0) b2s.push_back(q);
  bool relayout = (b2s != h->h_blk2sub) || (h->cur != 0);
  h->cur = 0;
  jkcals_status st = set_blocks(h, b2s);
  if (st != JKCALS_OK) return st;
  h->h_stored.assign(h->nsub, 0);
  for (int n = 0; n < h->N; ++n) {
    const int I = (int)h->dims[n];
    // reference store = [P_n(model 0) | P_n(model 1) | ...], column-major I x sum_m R_m; kept for
    // the alignment (Alg. 2 aligns every submodel to P)
    double* stage = h->ptr<double>(h->off.pref[n]);
    int64_t c0 = 0;
    for (int m = 0; m < h->nmodels; ++m) {
      CKH(h, cudaMemcpyAsync(stage + (int64_t)I * c0, P[m * h->N + n], sizeof(double) * I * h->ranks[m],
                             cudaMemcpyHostToDevice, h->stream));
      c0 += h->ranks[m];
    }
    CKH(h, cudaMemsetAsync(h->U(n), 0, sizeof(double) * I * h->ldu, h->stream));
    const int64_t tot = (int64_t)I * h->K * h->R;
    init_blocks_kernel<<<(int)cdiv(tot, 256), 256, 0, h->stream>>>(
        stage, I, h->R, h->K, h->ldu, h->U(n), n == 0 ? 1 : 0, h->ptr<int>(h->off.blk2sub),
        h->ptr<int>(h->off.blkcol), h->ptr<int>(h->off.subR), h->ptr<int>(h->off.subRc),
        h->ptr<int64_t>(h->off.pglob), (int)h->d);
    CKH(h, cudaGetLastError());
  }
  st = compute_grams(h);
  if (st != JKCALS_OK) return st;
  reset_state_kernel<<<(int)cdiv(h->nsub, 256), 256, 0, h->stream>>>(
      h->nsub, h->ptr<double>(h->off.fit), h->ptr<double>(h->off.fit_prev), h->ptr<double>(h->off.err),
      h->ptr<int>(h->off.iters), h->ptr<int>(h->off.flags), h->ptr<int>(h->off.active));
  CKH(h, cudaGetLastError());
  for (int q = 0; q < h->nsub; ++q)  // free slots never run
    if (h->h_id[q] < 0) CKH(h, cudaMemsetAsync(h->ptr<int>(h->off.active) + q, 0, sizeof(int), h->stream));
  CKH(h, cudaMemsetAsync(h->ptr<double>(h->off.hist), 0, sizeof(double) * h->nsub * (size_t)h->hist_cap, h->stream));
  if (relayout) {
    st = replan(h);
    if (st != JKCALS_OK) return st;
  }
  CKH(h, cudaStreamSynchronize(h->stream));  // the host P arrays are the copy sources
  h->inited = true;
  h->ran = false;
  h->aligned = false;
  return JKCALS_OK;
}

jkcals_status jkcals_set_init_submodel(jkcals_t h, int64_t p, int mode, const double* U) {
  if (!h || !U || mode < 0 || mode >= h->N || slot_of(h, p) < 0) return JKCALS_E_ARG;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "set_init must come first");
  DeviceGuard dg(h->device);
  const int sub = slot_of(h, p);
  const int blk = block_of(h, sub);
  if (blk < 0) return fail(h, JKCALS_E_STATE, "submodel %lld was compacted out", (long long)p);
  h->aligned = false;
  const int I = (int)h->dims[mode];
  const int R = h->h_subR[sub];
  const int64_t g = h->h_group[sub];
  const int cnt = mode == 0 ? (int)group_rows(h, g) : 0;
  const int rows = I - cnt;
  for (int64_t e = 0; e < (int64_t)rows * R; ++e)
    if (!std::isfinite(U[e])) return fail(h, JKCALS_E_NONFINITE, "non-finite init");
  double* stage = h->ptr<double>(h->off.stage);
  CKH(h, cudaMemcpyAsync(stage, U, sizeof(double) * rows * R, cudaMemcpyHostToDevice, h->stream));
  set_block_kernel<<<(int)cdiv((int64_t)I * R, 256), 256, 0, h->stream>>>(stage, I, R, h->ldu, h->h_blkcol[blk],
                                                                         mode == 0 ? g * h->d : -1, cnt, h->U(mode));
  CKH(h, cudaGetLastError());
  jkcals_status st = compute_grams(h);
  if (st != JKCALS_OK) return st;
  CKH(h, cudaStreamSynchronize(h->stream));
  return JKCALS_OK;
}

jkcals_status jkcals_set_init_all(jkcals_t h, int mode, const double* U) {
  if (!h || !U || mode < 0 || mode >= h->N) return JKCALS_E_ARG;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "set_init must come first");
  DeviceGuard dg(h->device);
  // packed like jkcals_get_all_factors: the owned slots in slot order, each rows_q x R_q
  const int I = (int)h->dims[mode];
  std::vector<int> subs;
  int64_t total = 0;
  for (int q = 0; q < h->nsub; ++q)
    if (h->h_id[q] >= 0) {
      if (block_of(h, q) < 0) return fail(h, JKCALS_E_STATE, "submodel %lld was compacted out", (long long)h->h_id[q]);
      subs.push_back(q);
      total += (int64_t)(I - (mode == 0 ? group_rows(h, h->h_group[q]) : 0)) * h->h_subR[q];
    }
  for (int64_t e = 0; e < total; ++e)
    if (!std::isfinite(U[e])) return fail(h, JKCALS_E_NONFINITE, "non-finite init");
  if (total > h->off.stage_cap) return fail(h, JKCALS_E_OOM, "internal: staging buffer too small");
  h->aligned = false;
  double* stage = h->ptr<double>(h->off.stage);
  CKH(h, cudaMemcpyAsync(stage, U, sizeof(double) * total, cudaMemcpyHostToDevice, h->stream));
  int64_t o = 0;
  for (int q : subs) {
    const int R = h->h_subR[q];
    const int cnt = mode == 0 ? (int)group_rows(h, h->h_group[q]) : 0;
    set_block_kernel<<<(int)cdiv((int64_t)I * R, 256), 256, 0, h->stream>>>(
        stage + o, I, R, h->ldu, h->h_blkcol[block_of(h, q)], mode == 0 ? h->h_group[q] * h->d : -1, cnt, h->U(mode));
    CKH(h, cudaGetLastError());
    o += (int64_t)(I - cnt) * R;
  }
  jkcals_status st = compute_grams(h);
  if (st != JKCALS_OK) return st;
  CKH(h, cudaStreamSynchronize(h->stream));  // U is the copy source
  return JKCALS_OK;
}

// ------------------------------------------------------------ resident whole-iterate path
// Shared-memory layout of one resident CTA for cluster size cs and Cp fused columns per group
// (fills the offsets / pitches of `a`); returns the dynamic bytes.
static size_t res_layout(const jkcals_s* h, int cs, int Cp, int kpc, ResArgs* a) {
  const int N = h->N, last = N - 1, R = h->R;
  // T strides: mode 0 contiguous, every other stride = 4 mod 16 doubles (conflict-free DMMA
  // fragment loads of 4 k x 8 rows, resident.cuh)
  int64_t pitch = 1;
  for (int m = 0; m < N; ++m) {
    a->pitch[m] = (int)pitch;
    pitch = pitch * h->dims[m];
    pitch = rup(pitch - 4, 16) + 4;
  }
  const int slab = (int)cdiv(h->dims[last], cs);
  const int Cpi = res_cpitch(Cp);
  a->Cpi = Cpi;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = (size_t)rup((int64_t)(off + bytes), 16);
    return (int)o;
  };
  a->o_T = take((size_t)slab * a->pitch[last] * 8);
  for (int m = 0; m < N; ++m) a->o_U[m] = take((size_t)h->dims[m] * Cpi * 8);
  size_t mbytes = 0;
  int64_t maxI = 0;
  for (int n = 0; n < N; ++n) {
    const int rows = n == last ? slab : (int)h->dims[n];
    const int KG = kResWarps / res_tgroups(rows);
    mbytes = std::max(mbytes, (size_t)KG * rows * Cpi * 8);
    maxI = std::max<int64_t>(maxI, h->dims[n]);
  }
  a->o_M = take(mbytes);
  a->o_E = take((size_t)cdiv(kpc, cs) * 2 * maxI * (R | 1) * 8);  // per owned slot
  a->o_G = take((size_t)cdiv(kpc, cs) * N * R * R * 8);
  a->o_X = take((size_t)kpc * 4);
  a->o_S = take(sizeof(ResScr));
  return off;
}

// choose the cluster size / grouping (or decide the standard path); sets h->res
static void res_plan(jkcals_t h) {
  h->res.dirty = false;
  h->res.on = false;
  h->res.warp = false;
  // "0": never; "1": the cluster kernel whenever it fits; "2": the warp kernel whenever it fits;
  // unset: the warp kernel for tiny tensors, the cluster kernel where r02 measured it faster
  const int mode = resident_mode();
  if (mode == 0 || h->tf32 || h->i8 || h->mixed || h->R > 8 || h->K < 1) return;
  if (mode == 2 || mode < 0) {  // tiny tensors: T in one CTA's shared memory, a warp per submodel
    int dv[kMaxModes];
    for (int m = 0; m < h->N; ++m) dv[m] = (int)h->dims[m];
    const size_t wsm = ((size_t)((h->P + 1) & ~1) + (size_t)kWrWarps * wr_warp_doubles(h->N, dv, h->R)) * 8;
    // (r02: tiny 10x8x6 -- 480 entries; the MTTKRP is lanes-over-rows FMA, so only for small J)
    if (h->P <= 4096 && wsm <= 200 * 1024 && warp_resident_kernel(2, h->N)) {
      h->res.on = true;
      h->res.warp = true;
      h->res.smem = wsm;
      h->res.rclass = h->R <= 2 ? 2 : h->R <= 4 ? 4 : 8;
      cudaFuncSetAttribute(warp_resident_kernel(h->res.rclass, h->N), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)wsm);
      return;
    }
    if (mode == 2) return;
  }
  double work = (double)h->C * (double)h->P;
  if (mode < 0 && work > (double)(1 << 27)) return;  // large problems: the streamed path is efficient
  const int N = h->N, last = N - 1;
  for (int m = 0; m < N; ++m)
    if (h->dims[m] > 4096) return;
  const ResFn fn = resident_kernel(h->R);
  double best = 1e300;
  for (int cs : {1, 2, 4, 8, 16}) {
    const int slab = (int)cdiv(h->dims[last], cs);
    if ((int64_t)(cs - 1) * slab >= h->dims[last]) continue;  // every CTA holds a non-empty slab
    // size with one submodel per group, then regroup by how many clusters of this size fit at
    // once (groups are independent: clusters need not all be resident, but a second wave doubles time)
    ResArgs a = {};
    int kpc = 1;
    int Cp = (int)rup((int64_t)kpc * h->R, 8);
    size_t smem = res_layout(h, cs, Cp, kpc, &a);
    if (smem > 200 * 1024) continue;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(226 * 1024)) != cudaSuccess ||
        (cs > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs * std::max(1, h->ki->nsm / cs));
    cfg.blockDim = dim3(kResThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int qmax = 0;
    if (cudaOccupancyMaxActiveClusters(&qmax, fn, &cfg) != cudaSuccess || qmax < 1) {
      cudaGetLastError();
      continue;
    }
    const int Q0 = std::min(h->K, qmax);
    kpc = (int)cdiv(h->K, Q0);
    Cp = (int)rup((int64_t)kpc * h->R, 8);
    if (Cp > kResMaxCp || cdiv(kpc, cs) > kResMaxOwn) continue;
    smem = res_layout(h, cs, Cp, kpc, &a);
    if (smem > 226 * 1024) continue;
    // per-CTA MTTKRP work ~ slab x Cp; a cluster adds DSMEM gathers and barriers
    const double cost = (double)slab * Cp * (double)(h->P / h->dims[last]) / 1e4 + (cs > 1 ? 2.0 : 0.0) +
                        0.5 * (double)cdiv(kpc, cs);
    // automatic use only where r02 measured a win over the streamed path: groups of <= 8 fused
    // columns over a multi-CTA cluster (syn50 R1-R2: 33-37 vs 39-43 us per sweep); tiny was even
    // (18.8 vs 18.6) and wider groups slower (syn50 R3-R5) -- JKCALS_RESIDENT=1 forces it
    if (mode < 0 && (Cp > 8 || cs < 2)) continue;
    if (cost < best) {
      best = cost;
      h->res.on = true;
      h->res.cs = cs;
      h->res.kpc = kpc;
      h->res.Q = (int)cdiv(h->K, kpc);
      h->res.Cp = Cp;
      h->res.slab = slab;
      h->res.smem = smem;
      h->res.rclass = h->R <= 2 ? 2 : h->R <= 4 ? 4 : 8;
      h->res.a = a;
    }
  }
  if (h->res.on)
    cudaFuncSetAttribute(resident_kernel(h->res.rclass), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)h->res.smem);
}

static jkcals_status wr_launch(jkcals_t h, int max_iters) {
  WrArgs a = {};
  a.N = h->N;
  a.R = h->R;
  a.d = (int)h->d;
  a.hist_cap = h->hist_cap;
  a.max_iters = max_iters;
  a.nsub = h->nsub;
  a.K = h->K;
  for (int m = 0; m < h->N; ++m) {
    a.dims[m] = (int)h->dims[m];
    a.U[m] = h->U(m);
  }
  a.gst[0] = 1;
  a.gst[1] = h->I0p;
  for (int m = 2; m < h->N; ++m) a.gst[m] = a.gst[m - 1] * h->dims[m - 1];
  a.ldu = h->ldu;
  a.Pel = (int)h->P;
  a.warp_doubles = wr_warp_doubles(h->N, a.dims, h->R);
  a.T = h->ptr<double>(h->off.T);
  a.blk2sub = h->ptr<int>(h->off.blk2sub);
  a.pglob = h->ptr<int64_t>(h->off.pglob);
  a.gram = h->ptr<double>(h->off.gram);
  a.lambda = h->ptr<double>(h->off.lambda);
  a.normT2p = h->ptr<double>(h->off.normT2p);
  a.fit = h->ptr<double>(h->off.fit);
  a.fit_prev = h->ptr<double>(h->off.fit_prev);
  a.err = h->ptr<double>(h->off.err);
  a.iters = h->ptr<int>(h->off.iters);
  a.flags = h->ptr<int>(h->off.flags);
  a.active = h->ptr<int>(h->off.active);
  a.hist = h->ptr<double>(h->off.hist);
  a.tol = reinterpret_cast<const double*>(h->ws + h->off.misc + 8);
  a.sweeps_out = reinterpret_cast<int*>(h->ws + h->off.misc + 24);
  CKH(h, cudaMemsetAsync(a.sweeps_out, 0, sizeof(int), h->stream));
  if (h->instrument) CKH(h, cudaEventRecord(h->ev[0], h->stream));
  warp_resident_kernel(h->res.rclass, h->N)<<<(unsigned)cdiv(h->K, kWrWarps), kWrWarps * 32, h->res.smem, h->stream>>>(a);
  CKH(h, cudaGetLastError());
  if (h->instrument) {
    CKH(h, cudaEventRecord(h->ev[1], h->stream));
    CKH(h, cudaEventSynchronize(h->ev[1]));
    float ms = 0;
    CKH(h, cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
    h->t_mttkrp[0] += ms;
    h->launches += 1;
  }
  CKH(h, cudaMemcpyAsync(h->pinned_count, a.sweeps_out, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  return JKCALS_OK;
}

static jkcals_status res_launch(jkcals_t h, int max_iters) {
  if (h->res.warp) return wr_launch(h, max_iters);
  ResArgs a = h->res.a;
  a.N = h->N;
  a.R = h->R;
  a.cs = h->res.cs;
  a.kpc = h->res.kpc;
  a.Cp = h->res.Cp;
  a.Cpi = res_cpitch(h->res.Cp);
  a.slab = h->res.slab;
  a.d = (int)h->d;
  a.hist_cap = h->hist_cap;
  a.max_iters = max_iters;
  a.nsub = h->nsub;
  a.K = h->K;
  for (int m = 0; m < h->N; ++m) {
    a.dims[m] = (int)h->dims[m];
    a.U[m] = h->U(m);
  }
  a.gst[0] = 1;
  a.gst[1] = h->I0p;
  for (int m = 2; m < h->N; ++m) a.gst[m] = a.gst[m - 1] * h->dims[m - 1];
  a.ldu = h->ldu;
  a.T = h->ptr<double>(h->off.T);
  a.blk2sub = h->ptr<int>(h->off.blk2sub);
  a.pglob = h->ptr<int64_t>(h->off.pglob);
  a.gram = h->ptr<double>(h->off.gram);
  a.lambda = h->ptr<double>(h->off.lambda);
  a.normT2p = h->ptr<double>(h->off.normT2p);
  a.fit = h->ptr<double>(h->off.fit);
  a.fit_prev = h->ptr<double>(h->off.fit_prev);
  a.err = h->ptr<double>(h->off.err);
  a.iters = h->ptr<int>(h->off.iters);
  a.flags = h->ptr<int>(h->off.flags);
  a.active = h->ptr<int>(h->off.active);
  a.hist = h->ptr<double>(h->off.hist);
  a.tol = reinterpret_cast<const double*>(h->ws + h->off.misc + 8);
  a.sweeps_out = reinterpret_cast<int*>(h->ws + h->off.misc + 24);
#ifdef JK_RES_PROF
  a.prof = reinterpret_cast<long long*>(h->ws + h->off.misc + 64);  // 8 counters (dev builds)
#endif
  CKH(h, cudaMemsetAsync(a.sweeps_out, 0, sizeof(int), h->stream));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = h->res.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(h->res.Q * h->res.cs);
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = h->res.smem;
  cfg.stream = h->stream;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (h->instrument) CKH(h, cudaEventRecord(h->ev[0], h->stream));
  CKH(h, cudaLaunchKernelEx(&cfg, resident_kernel(h->res.rclass), a));
  if (h->instrument) {
    CKH(h, cudaEventRecord(h->ev[1], h->stream));
    CKH(h, cudaEventSynchronize(h->ev[1]));
    float ms = 0;
    CKH(h, cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
    h->t_mttkrp[0] += ms;  // the whole launch (MTTKRP and updates are fused)
    h->launches += 1;
  }
  CKH(h, cudaMemcpyAsync(h->pinned_count, a.sweeps_out, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  return JKCALS_OK;
}

jkcals_status jkcals_iterate(jkcals_t h, int max_iters, double tol, int* sweeps_done) {
  NvtxRange nv("jkcals_iterate");
  if (!h || max_iters < 0) return JKCALS_E_ARG;
  if (sweeps_done) *sweeps_done = 0;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "iterate before set_init");
  DeviceGuard dg(h->device);
  h->aligned = false;
  if (h->tf32 && (tol > 0.0) != h->f64last) {  // switch the last mode's MTTKRP kernel: re-capture
    h->f64last = tol > 0.0;
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    if (h->gexec_tol) cudaGraphExecDestroy(h->gexec_tol);
    h->gexec = h->gexec_tol = nullptr;
    h->graph_ok = false;
  }
  h->tol_host = tol;
  CKH(h, cudaMemcpyAsync(h->ws + h->off.misc + 8, &h->tol_host, sizeof(double), cudaMemcpyHostToDevice, h->stream));
  if (h->res.dirty) res_plan(h);
  if (h->res.on && max_iters > 0 && h->K > 0) {  // one launch runs every sweep (device-side stop)
    jkcals_status st = res_launch(h, max_iters);
    if (st != JKCALS_OK) return st;
    CKH(h, cudaStreamSynchronize(h->stream));
    if (sweeps_done) *sweeps_done = *h->pinned_count;
    h->ran = true;
    return JKCALS_OK;
  }
  int it = 0;
  if (tol > 0.0 && !h->instrument) {
    jkcals_status st = ensure_tol_graph(h);
    if (st != JKCALS_OK) return st;
  }
  while (tol > 0.0 && !h->instrument && h->gexec_tol && it < max_iters && h->K > 0) {
    // device-side trigger: one graph launch runs sweeps until compaction is due or the budget ends
    const int cs = (64 + h->R - 1) / h->R;  // compact once >= 64 fused columns have converged
    int* pin = h->pinned_count;
    pin[0] = 0;                                  // misc+24: sweeps run by this launch
    pin[1] = 0;
    pin[2] = max_iters - it;                     // misc+32: sweep budget
    pin[3] = std::max(0, h->K - cs);             // misc+36: continue while active > this
    CKH(h, cudaMemcpyAsync(h->ws + h->off.misc + 24, pin, 4 * sizeof(int), cudaMemcpyHostToDevice, h->stream));
    CKH(h, cudaGraphLaunch(h->gexec_tol, h->stream));
    CKH(h, cudaMemcpyAsync(pin, h->ws + h->off.misc + 16, 4 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CKH(h, cudaStreamSynchronize(h->stream));
    const int nact = pin[0], ran = pin[2];
    it += ran;
    if (nact == 0 || (int64_t)(h->K - nact) * h->R >= 64) {
      jkcals_status st2 = compact(h);
      if (st2 != JKCALS_OK) return st2;
      st2 = ensure_tol_graph(h);
      if (st2 != JKCALS_OK) return st2;
    }
  }
  for (; it < max_iters && h->K > 0; ++it) {
    if (h->instrument) {
      jkcals_status st = enqueue_sweep(h, true);
      if (st != JKCALS_OK) return st;
      CKH(h, cudaEventSynchronize(h->ev[4 * (h->N - 1) + 2]));
      for (int n = 0; n < h->N; ++n) {
        float a = 0, b = 0;
        CKH(h, cudaEventElapsedTime(&a, h->ev[4 * n + 0], h->ev[4 * n + 1]));
        CKH(h, cudaEventElapsedTime(&b, h->ev[4 * n + 1], h->ev[4 * n + 2]));
        h->t_mttkrp[n] += a;
        h->t_epi[n] += b;
      }
      h->launches += h->N;
    } else {
      jkcals_status st = ensure_graph(h);
      if (st != JKCALS_OK) return st;
      CKH(h, cudaGraphLaunch(h->gexec, h->stream));
    }
    if (tol > 0.0) {
      CKH(h, cudaMemcpyAsync(h->pinned_count, h->ws + h->off.misc + 16, sizeof(int), cudaMemcpyDeviceToHost,
                             h->stream));
      CKH(h, cudaStreamSynchronize(h->stream));
      const int nact = *h->pinned_count;
      const int nconv = h->K - nact;
      if (nact == 0 || (int64_t)nconv * h->R >= 64) {
        jkcals_status st = compact(h);
        if (st != JKCALS_OK) return st;
      }
    }
  }
  CKH(h, cudaStreamSynchronize(h->stream));
  if (sweeps_done) *sweeps_done = it;
  h->ran = true;
  return JKCALS_OK;
}

static jkcals_status locate_slot(jkcals_t h, int sub, int mode, const double** src, int64_t* ld) {
  const int R = h->h_subR[sub];
  if (h->h_stored[sub]) {
    int64_t o = 0;
    for (int n = 0; n < mode; ++n) o += h->dims[n] * R;
    *src = h->ptr<double>(h->off.Ures) + (int64_t)sub * sum_dims(h) * h->R + o;
    *ld = R;
    return JKCALS_OK;
  }
  const int k = block_of(h, sub);
  if (k < 0) return fail(h, JKCALS_E_STATE, "slot %d holds no submodel", sub);
  *src = h->U(mode) + h->h_blkcol[k];
  *ld = h->ldu;
  return JKCALS_OK;
}

static jkcals_status locate(jkcals_t h, int64_t p, int mode, const double** src, int64_t* ld, int* sub_out) {
  const int sub = slot_of(h, p);
  *sub_out = sub;
  if (sub < 0) return fail(h, JKCALS_E_ARG, "submodel %lld is not on this handle", (long long)p);
  return locate_slot(h, sub, mode, src, ld);
}

jkcals_status jkcals_get_factors(jkcals_t h, int64_t p, int mode, double* U, double* lambda) {
  if (!h || !U || mode < 0 || mode >= h->N || slot_of(h, p) < 0) return JKCALS_E_ARG;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "no model yet");
  DeviceGuard dg(h->device);
  const double* src = nullptr;
  int64_t ld;
  int sub;
  jkcals_status st = locate(h, p, mode, &src, &ld, &sub);
  if (st != JKCALS_OK) return st;
  const int I = (int)h->dims[mode];
  const int R = h->h_subR[sub];
  const int cnt = mode == 0 ? (int)group_rows(h, h->h_group[sub]) : 0;
  const int rows = I - cnt;
  double* stage = h->ptr<double>(h->off.stage);
  extract_kernel<<<(int)cdiv((int64_t)rows * R, 256), 256, 0, h->stream>>>(
      src, ld, I, R, mode == 0 ? h->h_group[sub] * h->d : -1, cnt, stage);
  CKH(h, cudaGetLastError());
  CKH(h, cudaMemcpyAsync(U, stage, sizeof(double) * rows * R, cudaMemcpyDeviceToHost, h->stream));
  if (lambda)
    CKH(h, cudaMemcpyAsync(lambda, h->ptr<double>(h->off.lambda) + (int64_t)sub * h->R, sizeof(double) * R,
                           cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  return JKCALS_OK;
}

static jkcals_status build_src_table(jkcals_t h, int mode, const std::vector<int>& subs);

jkcals_status jkcals_get_all_factors(jkcals_t h, int mode, double* U, double* lambda) {
  if (!h || !U || mode < 0 || mode >= h->N) return JKCALS_E_ARG;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "no model yet");
  DeviceGuard dg(h->device);
  std::vector<int> subs;  // owned slots, in slot order
  for (int q = 0; q < h->nsub; ++q)
    if (h->h_id[q] >= 0) subs.push_back(q);
  const int ns = (int)subs.size();
  if (ns == 0) return JKCALS_OK;
  jkcals_status st = build_src_table(h, mode, subs);
  if (st != JKCALS_OK) return st;
  const int I = (int)h->dims[mode];
  // packed output: the j-th owned slot's rows x R block at dstoff[j]; per-listed rank / row start
  std::vector<int64_t> dst(ns), pg(ns);
  std::vector<int> rk(ns);
  int64_t total = 0;
  for (int j = 0; j < ns; ++j) {
    const int q = subs[j];
    dst[j] = total;
    rk[j] = h->h_subR[q];
    pg[j] = h->h_group[q] * h->d;
    const int rows = I - (mode == 0 ? (int)group_rows(h, h->h_group[q]) : 0);
    total += (int64_t)rows * h->h_subR[q];
  }
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.dstoff), dst.data(), 8 * ns, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.srcpg), pg.data(), 8 * ns, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.map), rk.data(), 4 * ns, cudaMemcpyHostToDevice, h->stream));
  double* stage = h->ptr<double>(h->off.stage);
  const int per = (int)std::min<int64_t>(cdiv((int64_t)I * h->R, 256), 64);
  extract_all_kernel<<<dim3(per, (unsigned)std::min(ns, 65535)), 256, 0, h->stream>>>(
      reinterpret_cast<const double*>(h->ws), h->ptr<int64_t>(h->off.srcoff), h->ptr<int64_t>(h->off.srcld),
      h->ptr<int>(h->off.map), h->ptr<int64_t>(h->off.dstoff), ns, I, mode == 0 ? 1 : 0,
      h->ptr<int64_t>(h->off.srcpg), (int)h->d, stage);
  CKH(h, cudaGetLastError());
  CKH(h, cudaMemcpyAsync(U, stage, sizeof(double) * total, cudaMemcpyDeviceToHost, h->stream));
  if (lambda) {  // packed the same way: R_q values per submodel
    std::vector<double> lam((size_t)h->nsub * h->R);
    CKH(h, cudaMemcpyAsync(lam.data(), h->ptr<double>(h->off.lambda), sizeof(double) * lam.size(),
                           cudaMemcpyDeviceToHost, h->stream));
    CKH(h, cudaStreamSynchronize(h->stream));
    int64_t o = 0;
    for (int q : subs)
      for (int r = 0; r < h->h_subR[q]; ++r) lambda[o++] = lam[(size_t)q * h->R + r];
  }
  CKH(h, cudaStreamSynchronize(h->stream));
  return JKCALS_OK;
}

jkcals_status jkcals_get_block(jkcals_t h, int64_t p, int mode, double* U) {
  if (!h || !U || mode < 0 || mode >= h->N || slot_of(h, p) < 0) return JKCALS_E_ARG;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "no model yet");
  DeviceGuard dg(h->device);
  const double* src = nullptr;
  int64_t ld;
  int sub;
  jkcals_status st = locate(h, p, mode, &src, &ld, &sub);
  if (st != JKCALS_OK) return st;
  const int I = (int)h->dims[mode];
  const int R = h->h_subR[sub];
  double* stage = h->ptr<double>(h->off.stage);
  extract_kernel<<<(int)cdiv((int64_t)I * R, 256), 256, 0, h->stream>>>(src, ld, I, R, -1, 0, stage);
  CKH(h, cudaGetLastError());
  CKH(h, cudaMemcpyAsync(U, stage, sizeof(double) * I * R, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  return JKCALS_OK;
}

jkcals_status jkcals_get_status(jkcals_t h, double* fit, double* err, int* iters, int* flags) {
  if (!h) return JKCALS_E_ARG;
  DeviceGuard dg(h->device);
  const size_t n = h->nsub;
  if (fit) CKH(h, cudaMemcpyAsync(fit, h->ptr<double>(h->off.fit), 8 * n, cudaMemcpyDeviceToHost, h->stream));
  if (err) CKH(h, cudaMemcpyAsync(err, h->ptr<double>(h->off.err), 8 * n, cudaMemcpyDeviceToHost, h->stream));
  if (iters) CKH(h, cudaMemcpyAsync(iters, h->ptr<int>(h->off.iters), 4 * n, cudaMemcpyDeviceToHost, h->stream));
  if (flags) CKH(h, cudaMemcpyAsync(flags, h->ptr<int>(h->off.flags), 4 * n, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  return JKCALS_OK;
}

jkcals_status jkcals_get_history(jkcals_t h, int64_t p, double* err, int cap, int* count) {
  if (!h || !err || cap < 0 || slot_of(h, p) < 0) return JKCALS_E_ARG;
  DeviceGuard dg(h->device);
  const int sub = slot_of(h, p);
  int it = 0;
  CKH(h, cudaMemcpyAsync(&it, h->ptr<int>(h->off.iters) + sub, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  std::vector<double> ring(h->hist_cap);
  CKH(h, cudaMemcpyAsync(ring.data(), h->ptr<double>(h->off.hist) + (int64_t)sub * h->hist_cap,
                         sizeof(double) * h->hist_cap, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  int avail = std::min(it, h->hist_cap);
  int nout = std::min(avail, cap);
  // oldest first among the last `nout`
  for (int q = 0; q < nout; ++q) {
    int sweep = it - nout + q;  // 0-based sweep index
    err[q] = ring[sweep % h->hist_cap];
  }
  if (count) *count = nout;
  return JKCALS_OK;
}

// device table locating the mode-`mode` blocks of the listed local submodels (live
// multi-factor or result store), in list order
static jkcals_status build_src_table(jkcals_t h, int mode, const std::vector<int>& subs) {
  const int ns = (int)subs.size();
  std::vector<int64_t> off(ns), ld(ns);
  for (int q = 0; q < ns; ++q) {
    const double* src = nullptr;
    int64_t l = 0;
    jkcals_status st = locate_slot(h, subs[q], mode, &src, &l);
    if (st != JKCALS_OK) return st;
    off[q] = src - reinterpret_cast<const double*>(h->ws);
    ld[q] = l;
  }
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.srcoff), off.data(), 8 * ns, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.srcld), ld.data(), 8 * ns, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));  // off/ld are host temporaries
  return JKCALS_OK;
}

// per-element moments of model `model`'s local submodels; returns their count in *g
static jkcals_status moments(jkcals_t h, int model, int mode, double* mean_d, double* m2_d, int* g) {
  std::vector<int> subs;
  for (int q = 0; q < h->nsub; ++q)
    if (h->h_model[q] == model) subs.push_back(q);
  *g = (int)subs.size();
  if (subs.empty()) return JKCALS_OK;
  jkcals_status st = build_src_table(h, mode, subs);
  if (st != JKCALS_OK) return st;
  const int I = (int)h->dims[mode], R = h->ranks[model];
  moments_kernel<<<(int)cdiv((int64_t)I * R * 32, 256), 256, 0, h->stream>>>(
      reinterpret_cast<const double*>(h->ws), h->ptr<int64_t>(h->off.srcoff), h->ptr<int64_t>(h->off.srcld),
      (int)subs.size(), I, R, mean_d, m2_d);
  CKH(h, cudaGetLastError());
  CKH(h, cudaStreamSynchronize(h->stream));
  return JKCALS_OK;
}

jkcals_status jkcals_get_model_moments(jkcals_t h, int model, int mode, double* count, double* mean, double* m2) {
  if (!h || !mean || !m2 || mode < 1 || mode >= h->N || model < 0 || model >= h->nmodels) return JKCALS_E_ARG;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "no model yet");
  DeviceGuard dg(h->device);
  const int64_t IR = h->dims[mode] * h->ranks[model];
  double* stage = h->ptr<double>(h->off.stage);
  int g = 0;
  jkcals_status st = moments(h, model, mode, stage, stage + IR, &g);
  if (st != JKCALS_OK) return st;
  if (g == 0) {
    for (int64_t e = 0; e < IR; ++e) mean[e] = m2[e] = 0.0;
  } else {
    CKH(h, cudaMemcpyAsync(mean, stage, 8 * IR, cudaMemcpyDeviceToHost, h->stream));
    CKH(h, cudaMemcpyAsync(m2, stage + IR, 8 * IR, cudaMemcpyDeviceToHost, h->stream));
    CKH(h, cudaStreamSynchronize(h->stream));
  }
  if (count)
    for (int64_t e = 0; e < IR; ++e) count[e] = (double)g;
  return JKCALS_OK;
}

jkcals_status jkcals_get_model_stats(jkcals_t h, int model, int mode, double* mean, double* std_out) {
  if (!h || !mean || !std_out || mode < 1 || mode >= h->N || model < 0 || model >= h->nmodels) return JKCALS_E_ARG;
  const int64_t IR = h->dims[mode] * h->ranks[model];
  std::vector<double> m2(IR), cnt(IR);
  jkcals_status st = jkcals_get_model_moments(h, model, mode, cnt.data(), mean, m2.data());
  if (st != JKCALS_OK) return st;
  const double g = IR > 0 ? cnt[0] : 0.0;
  if (g < 2) return fail(h, JKCALS_E_ARG, "jackknife statistics need >= 2 submodels of the model");
  for (int64_t e = 0; e < IR; ++e) std_out[e] = std::sqrt(((g - 1.0) / g) * m2[e]);
  return JKCALS_OK;
}

// ---------------------------------------------------------------- alignment (NEXT #3)
jkcals_status jkcals_align(jkcals_t h) {
  if (!h) return JKCALS_E_ARG;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "no model yet");
  for (int m = 0; m < h->nmodels; ++m)
    if (h->ranks[m] > kAlignRMax) return fail(h, JKCALS_E_SHAPE, "alignment supports rank <= %d", kAlignRMax);
  DeviceGuard dg(h->device);
  std::vector<int64_t> off((size_t)h->nsub * h->N), ld((size_t)h->nsub * h->N);
  for (int q = 0; q < h->nsub; ++q)
    for (int n = 0; n < h->N; ++n) {
      const double* src = nullptr;
      int64_t l = 0;
      if (h->h_id[q] < 0) {  // free slot: nothing to align (R = 0 there)
        off[(size_t)q * h->N + n] = 0;
        ld[(size_t)q * h->N + n] = 0;
        continue;
      }
      jkcals_status st = locate_slot(h, q, n, &src, &l);
      if (st != JKCALS_OK) return st;
      off[(size_t)q * h->N + n] = src - reinterpret_cast<const double*>(h->ws);
      ld[(size_t)q * h->N + n] = l;
    }
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.asrc), off.data(), 8 * off.size(), cudaMemcpyHostToDevice,
                         h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.asld), ld.data(), 8 * ld.size(), cudaMemcpyHostToDevice, h->stream));
  AlignArgs a = {};
  a.base = reinterpret_cast<const double*>(h->ws);
  a.asrc = h->ptr<int64_t>(h->off.asrc);
  a.asld = h->ptr<int64_t>(h->off.asld);
  a.lambda = h->ptr<double>(h->off.lambda);
  a.subR = h->ptr<int>(h->off.subR);
  a.subRc = h->ptr<int>(h->off.subRc);
  for (int n = 0; n < h->N; ++n) {
    a.pref[n] = h->ptr<double>(h->off.pref[n]);
    a.dims[n] = h->dims[n];
  }
  a.N = h->N;
  a.Rs = h->R;
  a.sumI = sum_dims(h);
  a.aln = h->ptr<double>(h->off.aln);
  a.perm = h->ptr<int>(h->off.aperm);
  a.sign = h->ptr<int>(h->off.asign);
  a.cong = h->ptr<double>(h->off.acong);
  align_kernel<<<h->nsub, kAlignThreads, 0, h->stream>>>(a);
  CKH(h, cudaGetLastError());
  CKH(h, cudaStreamSynchronize(h->stream));  // off/ld are host temporaries
  h->aligned = true;
  return JKCALS_OK;
}

jkcals_status jkcals_get_alignment(jkcals_t h, int64_t p, int* perm, int* sign, double* congruence) {
  if (!h || slot_of(h, p) < 0) return JKCALS_E_ARG;
  if (!h->aligned) return fail(h, JKCALS_E_STATE, "jkcals_align has not run on the current factors");
  DeviceGuard dg(h->device);
  const int sub = slot_of(h, p), R = h->h_subR[sub];
  if (perm)
    CKH(h, cudaMemcpyAsync(perm, h->ptr<int>(h->off.aperm) + (int64_t)sub * h->R, 4 * R, cudaMemcpyDeviceToHost,
                           h->stream));
  if (congruence)
    CKH(h, cudaMemcpyAsync(congruence, h->ptr<double>(h->off.acong) + (int64_t)sub * h->R, 8 * R,
                           cudaMemcpyDeviceToHost, h->stream));
  if (sign)
    for (int n = 0; n < h->N; ++n)
      CKH(h, cudaMemcpyAsync(sign + (int64_t)n * R, h->ptr<int>(h->off.asign) + ((int64_t)sub * h->N + n) * h->R,
                             4 * R, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  return JKCALS_OK;
}

// aligned block of local submodel `sub`, mode n: row-major I_n x R_sub
static const double* aligned_block(jkcals_t h, int sub, int mode) {
  int64_t o = 0;
  for (int n = 0; n < mode; ++n) o += h->dims[n] * h->h_subR[sub];
  return h->ptr<double>(h->off.aln) + (int64_t)sub * sum_dims(h) * h->R + o;
}

jkcals_status jkcals_get_aligned_factors(jkcals_t h, int64_t p, int mode, double* U) {
  if (!h || !U || mode < 0 || mode >= h->N || slot_of(h, p) < 0) return JKCALS_E_ARG;
  if (!h->aligned) return fail(h, JKCALS_E_STATE, "jkcals_align has not run on the current factors");
  DeviceGuard dg(h->device);
  const int sub = slot_of(h, p), R = h->h_subR[sub];
  const int I = (int)h->dims[mode];
  const int cnt = mode == 0 ? (int)group_rows(h, h->h_group[sub]) : 0;
  double* stage = h->ptr<double>(h->off.stage);
  extract_kernel<<<(int)cdiv((int64_t)(I - cnt) * R, 256), 256, 0, h->stream>>>(
      aligned_block(h, sub, mode), R, I, R, mode == 0 ? h->h_group[sub] * h->d : -1, cnt, stage);
  CKH(h, cudaGetLastError());
  CKH(h, cudaMemcpyAsync(U, stage, sizeof(double) * (I - cnt) * R, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  return JKCALS_OK;
}

jkcals_status jkcals_get_aligned_moments(jkcals_t h, int model, int mode, double* count, double* mean, double* m2) {
  if (!h || !count || !mean || !m2 || mode < 0 || mode >= h->N || model < 0 || model >= h->nmodels)
    return JKCALS_E_ARG;
  if (!h->aligned) return fail(h, JKCALS_E_STATE, "jkcals_align has not run on the current factors");
  DeviceGuard dg(h->device);
  std::vector<int64_t> off, ld, pg;
  for (int q = 0; q < h->nsub; ++q)
    if (h->h_model[q] == model) {
      off.push_back(aligned_block(h, q, mode) - reinterpret_cast<const double*>(h->ws));
      ld.push_back(h->h_subR[q]);
      pg.push_back(h->h_group[q] * h->d);
    }
  const int I = (int)h->dims[mode], R = h->ranks[model];
  const int64_t IR = (int64_t)I * R;
  const int ns = (int)off.size();
  if (ns == 0) {
    for (int64_t e = 0; e < IR; ++e) count[e] = mean[e] = m2[e] = 0.0;
    return JKCALS_OK;
  }
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.srcoff), off.data(), 8 * ns, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.srcld), ld.data(), 8 * ns, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.srcpg), pg.data(), 8 * ns, cudaMemcpyHostToDevice, h->stream));
  double* stage = h->ptr<double>(h->off.stage);
  moments_present_kernel<<<(int)cdiv(IR, 128), 128, 0, h->stream>>>(
      reinterpret_cast<const double*>(h->ws), h->ptr<int64_t>(h->off.srcoff), h->ptr<int64_t>(h->off.srcld),
      h->ptr<int64_t>(h->off.srcpg), mode == 0 ? 1 : 0, (int)h->d, ns, I, R, stage, stage + IR, stage + 2 * IR);
  CKH(h, cudaGetLastError());
  CKH(h, cudaMemcpyAsync(count, stage, 8 * IR, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaMemcpyAsync(mean, stage + IR, 8 * IR, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaMemcpyAsync(m2, stage + 2 * IR, 8 * IR, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  return JKCALS_OK;
}

jkcals_status jkcals_get_aligned_stats(jkcals_t h, int model, int mode, double* mean, double* std_out) {
  if (!h || !mean || !std_out || mode < 0 || mode >= h->N || model < 0 || model >= h->nmodels)
    return JKCALS_E_ARG;
  const int64_t IR = h->dims[mode] * h->ranks[model];
  std::vector<double> cnt(IR), m2(IR);
  jkcals_status st = jkcals_get_aligned_moments(h, model, mode, cnt.data(), mean, m2.data());
  if (st != JKCALS_OK) return st;
  for (int64_t e = 0; e < IR; ++e) {
    const double g = cnt[e];
    std_out[e] = g >= 2.0 ? std::sqrt(((g - 1.0) / g) * m2[e]) : 0.0;
  }
  return JKCALS_OK;
}

jkcals_status jkcals_get_local_moments(jkcals_t h, int mode, double* count, double* mean, double* m2) {
  if (h && h->nmodels != 1) return fail(h, JKCALS_E_ARG, "pooled handle: use jkcals_get_model_moments");
  return jkcals_get_model_moments(h, 0, mode, count, mean, m2);
}

jkcals_status jkcals_merge_moments(int nparts, int64_t n, const double* counts, const double* means,
                                   const double* m2s, double* count, double* mean, double* m2) {
  if (nparts < 1 || n < 0 || !counts || !means || !m2s || !count || !mean || !m2) return JKCALS_E_ARG;
  for (int64_t e = 0; e < n; ++e) {
    double na = 0.0, ma = 0.0, sa = 0.0;
    for (int k = 0; k < nparts; ++k) {
      const double nb = counts[(int64_t)k * n + e];
      if (!(nb > 0.0)) continue;
      const double mb = means[(int64_t)k * n + e], sb = m2s[(int64_t)k * n + e];
      if (na == 0.0) {
        na = nb;
        ma = mb;
        sa = sb;
        continue;
      }
      const double nn = na + nb, d = mb - ma, wb = nb / nn;
      ma = ma + d * wb;
      sa = sa + sb + d * d * na * wb;
      na = nn;
    }
    count[e] = na;
    mean[e] = ma;
    m2[e] = sa;
  }
  return JKCALS_OK;
}

jkcals_status jkcals_get_jackknife_stats(jkcals_t h, int mode, double* mean, double* std_out) {
  if (h && h->nmodels != 1) return fail(h, JKCALS_E_ARG, "pooled handle: use jkcals_get_model_stats");
  return jkcals_get_model_stats(h, 0, mode, mean, std_out);
}

// ---------------------------------------------------------------- slots and migration (NEXT #4)
int jkcals_num_slots(jkcals_t h) { return h ? h->nsub : 0; }

jkcals_status jkcals_get_ids(jkcals_t h, int64_t* ids) {
  if (!h || !ids) return JKCALS_E_ARG;
  for (int q = 0; q < h->nsub; ++q) ids[q] = h->h_id[q];
  return JKCALS_OK;
}

enum { kStHdr = 16 };
static const double kStMagic = 1245397825.0;  // "JKCA"

static size_t state_doubles(const jkcals_s* h, int R) {
  return kStHdr + (size_t)R + (size_t)h->N * R * R + (size_t)h->hist_cap + (size_t)sum_dims(h) * R;
}

size_t jkcals_state_bytes(jkcals_t h, int64_t p) {
  if (!h) return 0;
  const int sub = slot_of(h, p);
  if (sub < 0) return 0;
  return 8 * state_doubles(h, h->h_subR[sub]);
}

jkcals_status jkcals_export_submodel(jkcals_t h, int64_t p, void* buf, size_t bytes) {
  if (!h || !buf) return JKCALS_E_ARG;
  const int sub = slot_of(h, p);
  if (sub < 0) return JKCALS_E_ARG;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "no model yet");
  const int R = h->h_subR[sub], N = h->N;
  if (bytes < 8 * state_doubles(h, R)) return fail(h, JKCALS_E_ARG, "state buffer too small");
  const int blk = block_of(h, sub);
  if (blk < 0) return fail(h, JKCALS_E_STATE, "submodel %lld is not live (converged and stored)", (long long)p);
  DeviceGuard dg(h->device);
  double* b = static_cast<double*>(buf);
  int it = 0, fl = 0, ac = 0;
  double fit = 0, fitp = 0, err = 0, nt2 = 0;
  CKH(h, cudaMemcpyAsync(&it, h->ptr<int>(h->off.iters) + sub, 4, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaMemcpyAsync(&fl, h->ptr<int>(h->off.flags) + sub, 4, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaMemcpyAsync(&ac, h->ptr<int>(h->off.active) + sub, 4, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaMemcpyAsync(&fit, h->ptr<double>(h->off.fit) + sub, 8, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaMemcpyAsync(&fitp, h->ptr<double>(h->off.fit_prev) + sub, 8, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaMemcpyAsync(&err, h->ptr<double>(h->off.err) + sub, 8, cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaMemcpyAsync(&nt2, h->ptr<double>(h->off.normT2p) + sub, 8, cudaMemcpyDeviceToHost, h->stream));
  double* o = b + kStHdr;
  CKH(h, cudaMemcpyAsync(o, h->ptr<double>(h->off.lambda) + (int64_t)sub * h->R, 8 * R, cudaMemcpyDeviceToHost,
                         h->stream));
  o += R;
  for (int n = 0; n < N; ++n, o += R * R)
    CKH(h, cudaMemcpyAsync(o, h->ptr<double>(h->off.gram) + ((int64_t)n * h->nsub + sub) * h->R * h->R, 8 * R * R,
                           cudaMemcpyDeviceToHost, h->stream));
  CKH(h, cudaMemcpyAsync(o, h->ptr<double>(h->off.hist) + (int64_t)sub * h->hist_cap, 8 * h->hist_cap,
                         cudaMemcpyDeviceToHost, h->stream));
  o += h->hist_cap;
  double* stage = h->ptr<double>(h->off.stage);
  for (int n = 0; n < N; ++n) {  // full blocks (mode 0 keeps its zero rows), column-major
    const int I = (int)h->dims[n];
    extract_kernel<<<(int)cdiv((int64_t)I * R, 256), 256, 0, h->stream>>>(h->U(n) + h->h_blkcol[blk], h->ldu, I, R,
                                                                         -1, 0, stage);
    CKH(h, cudaGetLastError());
    CKH(h, cudaMemcpyAsync(o, stage, 8 * (size_t)I * R, cudaMemcpyDeviceToHost, h->stream));
    CKH(h, cudaStreamSynchronize(h->stream));  // stage is reused by the next mode
    o += (int64_t)I * R;
  }
  CKH(h, cudaStreamSynchronize(h->stream));
  const double hdr[kStHdr] = {kStMagic, (double)p, (double)R, (double)h->h_model[sub], (double)h->h_group[sub],
                              (double)it, (double)fl, (double)ac, fit, fitp, err, nt2, (double)h->hist_cap,
                              (double)N, 0.0, 0.0};
  std::memcpy(b, hdr, sizeof hdr);
  // the submodel leaves this handle: drop its block and free the slot
  std::vector<int> keep;
  for (int k = 0; k < h->K; ++k)
    if (h->h_blk2sub[k] != sub) keep.push_back(h->h_blk2sub[k]);
  jkcals_status st = relayout(h, keep);
  if (st != JKCALS_OK) return st;
  h->h_id[sub] = -1;
  h->h_model[sub] = -1;
  h->h_subR[sub] = 0;
  const int zero = 0;
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.subR) + sub, &zero, 4, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.active) + sub, &zero, 4, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaStreamSynchronize(h->stream));
  h->aligned = false;
  return JKCALS_OK;
}

jkcals_status jkcals_import_submodel(jkcals_t h, const void* buf, size_t bytes) {
  if (!h || !buf || bytes < 8 * kStHdr) return JKCALS_E_ARG;
  if (!h->inited) return fail(h, JKCALS_E_STATE, "set_init must come first");
  const double* b = static_cast<const double*>(buf);
  if (b[0] != kStMagic) return fail(h, JKCALS_E_ARG, "not a submodel state");
  const int64_t id = (int64_t)b[1];
  const int R = (int)b[2], model = (int)b[3];
  const int64_t group = (int64_t)b[4];
  if ((int)b[12] != h->hist_cap || (int)b[13] != h->N) return fail(h, JKCALS_E_ARG, "state from another problem");
  if (model < 0 || model >= h->nmodels || h->ranks[model] != R || group < 0 || group >= h->ngroups ||
      id != model * h->ngroups + group)
    return fail(h, JKCALS_E_ARG, "state does not match this pool");
  if (bytes < 8 * state_doubles(h, R)) return fail(h, JKCALS_E_ARG, "state buffer truncated");
  if (slot_of(h, id) >= 0) return fail(h, JKCALS_E_ARG, "submodel %lld is already here", (long long)id);
  if (R > h->R || h->C + R > h->ldu) return fail(h, JKCALS_E_OOM, "no column room for the submodel");
  int sub = -1;
  for (int q = 0; q < h->nsub && sub < 0; ++q)
    if (h->h_id[q] < 0) sub = q;
  if (sub < 0) return fail(h, JKCALS_E_OOM, "no free slot (create with spare slots)");
  DeviceGuard dg(h->device);
  int rc = 0;
  for (int m = 0; m < model; ++m) rc += h->ranks[m];
  h->h_id[sub] = id;
  h->h_model[sub] = model;
  h->h_group[sub] = group;
  h->h_subR[sub] = R;
  h->h_subRc[sub] = rc;
  h->h_stored[sub] = 0;
  const int64_t pg = group * h->d;
  const int it = (int)b[5], fl = (int)b[6], ac = (int)b[7];
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.subR) + sub, &h->h_subR[sub], 4, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.subRc) + sub, &h->h_subRc[sub], 4, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int64_t>(h->off.pglob) + sub, &pg, 8, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.iters) + sub, &it, 4, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.flags) + sub, &fl, 4, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<int>(h->off.active) + sub, &ac, 4, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<double>(h->off.fit) + sub, b + 8, 8, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<double>(h->off.fit_prev) + sub, b + 9, 8, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<double>(h->off.err) + sub, b + 10, 8, cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<double>(h->off.normT2p) + sub, b + 11, 8, cudaMemcpyHostToDevice, h->stream));
  const double* o = b + kStHdr;
  CKH(h, cudaMemcpyAsync(h->ptr<double>(h->off.lambda) + (int64_t)sub * h->R, o, 8 * R, cudaMemcpyHostToDevice,
                         h->stream));
  o += R;
  for (int n = 0; n < h->N; ++n, o += R * R)
    CKH(h, cudaMemcpyAsync(h->ptr<double>(h->off.gram) + ((int64_t)n * h->nsub + sub) * h->R * h->R, o, 8 * R * R,
                           cudaMemcpyHostToDevice, h->stream));
  CKH(h, cudaMemcpyAsync(h->ptr<double>(h->off.hist) + (int64_t)sub * h->hist_cap, o, 8 * h->hist_cap,
                         cudaMemcpyHostToDevice, h->stream));
  o += h->hist_cap;
  // append its block at the end of the live layout
  std::vector<int> b2s = h->h_blk2sub;
  b2s.push_back(sub);
  jkcals_status st = set_blocks(h, b2s);
  if (st != JKCALS_OK) return st;
  const int col = h->h_blkcol[h->K - 1];
  double* stage = h->ptr<double>(h->off.stage);
  for (int n = 0; n < h->N; ++n) {
    const int I = (int)h->dims[n];
    CKH(h, cudaMemcpyAsync(stage, o, 8 * (size_t)I * R, cudaMemcpyHostToDevice, h->stream));
    set_block_kernel<<<(int)cdiv((int64_t)I * R, 256), 256, 0, h->stream>>>(stage, I, R, h->ldu, col, -1, 0,
                                                                           h->U(n));
    CKH(h, cudaGetLastError());
    CKH(h, cudaStreamSynchronize(h->stream));  // stage is reused by the next mode
    o += (int64_t)I * R;
  }
  h->aligned = false;
  return replan(h);
}

jkcals_status jkcals_set_instrument(jkcals_t h, int on) {
  if (!h) return JKCALS_E_ARG;
  h->instrument = on != 0;
  return JKCALS_OK;
}

jkcals_status jkcals_get_kernel_times(jkcals_t h, double* mttkrp_ms, double* epilogue_ms, int64_t* launches) {
  if (!h) return JKCALS_E_ARG;
  for (int n = 0; n < h->N; ++n) {
    if (mttkrp_ms) mttkrp_ms[n] = h->t_mttkrp[n];
    if (epilogue_ms) epilogue_ms[n] = h->t_epi[n];
    h->t_mttkrp[n] = h->t_epi[n] = 0.0;
  }
  if (launches) *launches = h->launches;
  h->launches = 0;
  return JKCALS_OK;
}

double jkcals_sweep_flops(jkcals_t h) {
  if (!h) return 0.0;
  return 2.0 * (double)h->C * (double)h->P * (double)h->N;
}

int jkcals_launches_per_sweep(jkcals_t h) {
  if (!h) return 0;
  int n_red = 0;
  for (int n = 0; n < h->N; ++n) n_red += h->red_on[n] ? 1 : 0;
  return 2 * h->N + n_red + (h->i8 ? 2 * h->N : 0);  // (+ the two U_q0-digit kernels per mode)
}

#ifdef JK_RES_PROF
int jkcals_dev_res_prof(jkcals_t h, long long* out) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpy(out, h->ws + h->off.misc + 64, 64, cudaMemcpyDeviceToHost);
}
#endif

const char* jkcals_last_error(jkcals_t h) { return h ? h->err.c_str() : "null handle"; }

void jkcals_destroy(jkcals_t h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->gexec_tol) cudaGraphExecDestroy(h->gexec_tol);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  if (h->pinned_count) cudaFreeHost(h->pinned_count);
  if (h->cap) cudaStreamDestroy(h->cap);
  delete h;
}

// ---------------------------------------------------------------- stand-alone ops
size_t jkcals_mttkrp_scratch_bytes(int ndims, const int64_t* dims, int n, int64_t C, int device) {
  if (!valid_dims(ndims, dims, 1) || n < 0 || n >= ndims || C < 1) return 0;
  KernelInfo* ki = kernel_info(device, nullptr);
  if (!ki) return 0;
  int64_t P = 1;
  for (int k = 0; k < ndims; ++k) P *= dims[k];
  int64_t parts;
  int tiles;
  plan_bounds(mode_geo(ndims, dims, n), n, C, *ki, &parts, &tiles);
  // + staged copies: T with an even mode-0 pitch, every U_m with pitch round_up(C, 128)
  int64_t sumI = 0;
  for (int k = 0; k < ndims; ++k) sumI += dims[k];
  const int64_t ldp = rup(C, 128);
  return (size_t)rup(parts * 8, kAlign) + (size_t)rup(plan_table_bytes(tiles, ki->nsm * 8), kAlign) +
         (size_t)rup(rup(dims[0], 2) * (P / dims[0]) * 8, kAlign) + (size_t)ndims * kAlign +
         (size_t)sumI * ldp * 8 + kAlign;
}

jkcals_status jkcals_mttkrp(int ndims, const int64_t* dims, int n, const double* T, const double* const* U, int64_t C,
                            int64_t ldu, double* M, int64_t ldm, void* scratch, size_t scratch_bytes, void* stream) {
  if (!valid_dims(ndims, dims, 1) || n < 0 || n >= ndims || !T || !U || !M || C < 1 || ldu < C || ldm < C ||
      (ldu % 2) != 0 || (C % 2 == 1 && ldu < C + 1))
    return JKCALS_E_ARG;
  int dev = 0;
  cudaGetDevice(&dev);
  KernelInfo* ki = kernel_info(dev, nullptr);
  if (!ki) return JKCALS_E_CUDA;
  if (scratch_bytes < jkcals_mttkrp_scratch_bytes(ndims, dims, n, C, dev)) return JKCALS_E_OOM;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t P = 1;
  for (int k = 0; k < ndims; ++k) P *= dims[k];
  ModePlan p = make_plan(mode_geo(ndims, dims, n), n, C, *ki);
  uintptr_t base = (reinterpret_cast<uintptr_t>(scratch) + kAlign - 1) & ~(uintptr_t)(kAlign - 1);
  TileInfo* ti = reinterpret_cast<TileInfo*>(base);
  base += rup(plan_table_bytes(p.ntiles, p.G), kAlign);
  double* parts = reinterpret_cast<double*>(base);
  base += rup(plan_parts_doubles(p) * 8, kAlign);
  // stage T (even mode-0 pitch) and U (pitch round_up(C,128), zero padding) for the TMA views
  const int64_t I0p = rup(dims[0], 2), J0 = P / dims[0], ldp = rup(C, 128);
  double* Tp = reinterpret_cast<double*>(base);
  base += rup(I0p * J0 * 8, kAlign);
  if (cudaMemsetAsync(Tp, 0, I0p * J0 * 8, s) != cudaSuccess ||
      cudaMemcpy2DAsync(Tp, I0p * 8, T, dims[0] * 8, dims[0] * 8, J0, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return JKCALS_E_CUDA;
  double* Up[kMaxModes];
  for (int m = 0; m < ndims; ++m) {
    Up[m] = reinterpret_cast<double*>(base);
    base += rup(dims[m] * ldp * 8, kAlign);
    if (m == n) continue;
    if (cudaMemsetAsync(Up[m], 0, dims[m] * ldp * 8, s) != cudaSuccess ||
        cudaMemcpy2DAsync(Up[m], ldp * 8, U[m], ldu * 8, C * 8, dims[m], cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return JKCALS_E_CUDA;
  }
  std::vector<char> table = pack_plan(p);
  if (cudaMemcpyAsync(ti, table.data(), table.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return JKCALS_E_CUDA;
  MttkrpView v = make_mview(ndims, dims, n, Up, p.KB);
  CUtensorMap tmT, tmU;
  const int q0 = (n == 0) ? 1 : 0;
  if (!make_tmap_T(&tmT, Tp, ndims, dims, I0p, n, p.BN, bnp_of(p.NT), p.KB) ||
      !make_tmap_U(&tmU, Up[q0], dims[q0], ldp, p.BM + 4, p.KB))
    return JKCALS_E_CUDA;
  MttkrpGeom g;
  g.C = (int)C;
  g.ldu = ldp;
  g.nMt = p.nMt;
  g.nNt = p.nNt;
  g.KT = p.KT;
  g.units = p.units;
  g.G = p.G;
  ki->fn[p.KV][p.WV][p.KM][p.ST4][p.NT - 1]<<<p.G, (kWMs[p.WV] + 1) * 32, p.smem, s>>>(tmT, tmU, v, g, ti, parts);
  if (cudaGetLastError() != cudaSuccess) return JKCALS_E_CUDA;
  int64_t tot = dims[n] * C;
  reduce_parts_kernel<<<(int)cdiv(tot, 256), 256, 0, s>>>(parts, ti, (int)dims[n], (int)C, p.BN, p.nMt, M, ldm,
                                                          p.BM);
  if (cudaGetLastError() != cudaSuccess) return JKCALS_E_CUDA;
  // tinfo staging is pageable-host -> device: make sure the copy has consumed it
  if (cudaStreamSynchronize(s) != cudaSuccess) return JKCALS_E_CUDA;
  return JKCALS_OK;
}

// ---------------------------------------------------------------- EXPERIMENTAL: INT8-sliced MTTKRP
namespace {
struct I8Scratch {
  TileInfo* ti;
  double* parts;
  int8_t *A, *B;
  int *eT, *eU, *dims_d, *eS;
  int8_t* dS;
  int64_t* st_d;
  double* Up[kMaxModes];
  size_t total;
};
I8Scratch i8_layout(uintptr_t base0, int ndims, const int64_t* dims, const I8Plan& q) {
  I8Scratch x;
  uintptr_t base = (base0 + kAlign - 1) & ~(uintptr_t)(kAlign - 1);
  const uintptr_t start = base;
  auto take = [&](size_t bytes) {
    uintptr_t o = base;
    base += rup((int64_t)bytes, kAlign);
    return o;
  };
  x.ti = reinterpret_cast<TileInfo*>(take(plan_table_bytes(q.p.ntiles, q.p.G)));
  x.parts = reinterpret_cast<double*>(take((size_t)(q.p.G + q.p.ntiles) * q.p.BN * 128 * 8));
  x.A = reinterpret_cast<int8_t*>(take((size_t)kI8S * q.CP * q.KP));
  x.B = reinterpret_cast<int8_t*>(take((size_t)kI8S * q.Jp * q.InP * q.KP));
  x.eT = reinterpret_cast<int*>(take((size_t)q.InP * 4));
  x.eS = reinterpret_cast<int*>(take((size_t)q.Jp * q.InP * 4));
  x.dS = reinterpret_cast<int8_t*>(take((size_t)q.Jp * q.InP));
  x.eU = reinterpret_cast<int*>(take((size_t)q.CP * 4));
  x.dims_d = reinterpret_cast<int*>(take(kMaxModes * 4));
  x.st_d = reinterpret_cast<int64_t*>(take(kMaxModes * 8));
  for (int m = 0; m < ndims; ++m) x.Up[m] = reinterpret_cast<double*>(take((size_t)dims[m] * q.CP * 8));
  x.total = (size_t)(base - start) + kAlign;
  return x;
}
}  // namespace

size_t jkcals_mttkrp_i8_scratch_bytes(int ndims, const int64_t* dims, int n, int64_t C, int device) {
  if (!valid_dims(ndims, dims, 1) || n < 0 || n >= ndims || C < 1) return 0;
  KernelInfo* ki = kernel_info(device, nullptr);
  if (!ki) return 0;
  const I8Plan q = make_i8_plan(ndims, dims, n, C, *ki);
  return i8_layout(0, ndims, dims, q).total;
}

jkcals_status jkcals_mttkrp_i8(int ndims, const int64_t* dims, int n, const double* T, const double* const* U,
                               int64_t C, int64_t ldu, double* M, int64_t ldm, void* scratch, size_t scratch_bytes,
                               void* stream) {
  if (!valid_dims(ndims, dims, 1) || n < 0 || n >= ndims || !T || !U || !M || C < 1 || ldu < C || ldm < C ||
      !i8_k_ok(ndims, dims))
    return JKCALS_E_ARG;
  int dev = 0;
  cudaGetDevice(&dev);
  KernelInfo* ki = kernel_info(dev, nullptr);
  if (!ki) return JKCALS_E_CUDA;
  if (scratch_bytes < jkcals_mttkrp_i8_scratch_bytes(ndims, dims, n, C, dev)) return JKCALS_E_OOM;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const I8Plan q = make_i8_plan(ndims, dims, n, C, *ki);
  I8Scratch x = i8_layout(reinterpret_cast<uintptr_t>(scratch), ndims, dims, q);
  const int q0 = (n == 0) ? 1 : 0;
  int64_t st[kMaxModes];
  int dd[kMaxModes];
  int64_t P = 1;
  for (int m = 0; m < ndims; ++m) {
    st[m] = P;
    dd[m] = (int)dims[m];
    P *= dims[m];
  }
  if (cudaMemcpyAsync(x.st_d, st, 8 * ndims, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(x.dims_d, dd, 4 * ndims, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return JKCALS_E_CUDA;
  for (int m = 0; m < ndims; ++m) {
    if (m == n) continue;
    if (cudaMemsetAsync(x.Up[m], 0, dims[m] * q.CP * 8, s) != cudaSuccess ||
        cudaMemcpy2DAsync(x.Up[m], q.CP * 8, U[m], ldu * 8, C * 8, dims[m], cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return JKCALS_E_CUDA;
  }
  // operands: T digits per mode-n row scale, U_q0 digits per column scale
  slab_exp_t_kernel<<<(int)cdiv(q.Jp * q.InP, 256), 256, 0, s>>>(T, ndims, x.st_d, x.dims_d, n, q0, (int)q.In,
                                                                (int)q.InP, (int)q.Iq0, q.Jp, x.eS);
  row_ref_exp_kernel<<<(int)q.InP, 256, 0, s>>>(x.eS, (int)q.InP, q.Jp, x.eT, x.dS);
  slice_t_i8_kernel<<<(int)cdiv(q.Jp * q.InP * q.KP, 256), 256, 0, s>>>(T, ndims, x.st_d, x.dims_d, n, q0, (int)q.In,
                                                                        (int)q.InP, (int)q.Iq0, (int)q.KP, q.Jp,
                                                                        x.eS, x.B);
  col_exp_u_kernel<<<(int)cdiv(q.CP, 32), 256, 0, s>>>(x.Up[q0], q.CP, (int)q.Iq0, (int)C, (int)q.CP, x.eU);
  slice_u_i8_kernel<<<(int)cdiv(q.CP * q.KP, 256), 256, 0, s>>>(x.Up[q0], q.CP, (int)q.Iq0, (int)C, (int)q.CP,
                                                                (int)q.KP, x.eU, x.A);
  if (cudaGetLastError() != cudaSuccess) return JKCALS_E_CUDA;
  std::vector<char> table = pack_plan(q.p);
  if (cudaMemcpyAsync(x.ti, table.data(), table.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return JKCALS_E_CUDA;
  CUtensorMap tmA, tmB;
  if (!make_tmap_i8(&tmA, x.A, q.KP, q.CP, 128, q.variant == 2 ? 4 : kI8S) ||
      !make_tmap_i8(&tmB, x.B, q.KP, q.Jp * q.InP, kI8N))
    return JKCALS_E_CUDA;
  I8Geom g;
  g.nMt = q.nMt;
  g.nNt = q.nNt;
  g.Jp = (int)q.Jp;
  g.KS = (int)(q.KP / kI8K);
  g.Kq = (int)q.Iq0;
  g.units = q.p.units;
  g.InP = (int)q.InP;
  g.nslow = ndims - 2;
  int sl = 0;
  for (int m = 0; m < ndims; ++m) {
    if (m == n || m == q0) continue;
    g.sdim[sl] = (int)dims[m];
    g.Us[sl] = x.Up[m];
    ++sl;
  }
  for (; sl < kMaxModes - 2; ++sl) {
    g.sdim[sl] = 1;
    g.Us[sl] = nullptr;
  }
  g.ldu = q.CP;
  g.eT = x.eT;
  g.dS = x.dS;
  g.eU = x.eU;
#ifdef JKCALS_DEV_PROBES  // timing-probe builds only: 1 = drain skipped, 2 = one product per K32 step
  g.probe = tuning().i8_probe;
#endif
  if (launch_i8(q, tmA, tmB, g, x.ti, x.parts, s) != cudaSuccess) return JKCALS_E_CUDA;
  const int64_t tot = q.In * C;
  reduce_parts_kernel<<<(int)cdiv(tot, 256), 256, 0, s>>>(x.parts, x.ti, (int)q.In, (int)C, q.p.BN, q.nMt, M, ldm);
  if (cudaGetLastError() != cudaSuccess) return JKCALS_E_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return JKCALS_E_CUDA;
  return JKCALS_OK;
}

jkcals_status jkcals_krp(int ndims, const int64_t* dims, int n, const double* const* U, int64_t C, int64_t ldu,
                         double* K, int64_t ldk, void* stream) {
  if (!valid_dims(ndims, dims, 1) || n < 0 || n >= ndims || !U || !K || C < 1 || ldu < C || ldk < C)
    return JKCALS_E_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t P = 1;
  for (int k = 0; k < ndims; ++k) P *= dims[k];
  ModeView v;
  v.N = ndims;
  v.n = n;
  v.nrest = ndims - 1;
  v.In = (int)dims[n];
  v.J = (int)(P / dims[n]);
  v.L = 1;
  v.LIn = 0;
  int q = 0;
  for (int m = 0; m < ndims; ++m) {
    if (m == n) continue;
    v.rdim[q] = (int)dims[m];
    v.U[q] = U[m];
    ++q;
  }
  for (; q < kMaxModes - 1; ++q) {
    v.rdim[q] = 1;
    v.U[q] = nullptr;
  }
  dim3 grid((unsigned)cdiv(v.J, kKrpRows), (unsigned)cdiv(cdiv(C, 4), 256));
  krp_gen_kernel<<<grid, 256, 0, s>>>(v, (int)C, ldu, K, ldk);
  return cudaGetLastError() == cudaSuccess ? JKCALS_OK : JKCALS_E_CUDA;
}

}  // extern "C"
