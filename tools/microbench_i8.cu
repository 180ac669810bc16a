// De-risking the next-round INT8-sliced FP64 MTTKRP: tcgen05.mma kind::i8 on
// sm_100a -- (1) a correctness check of one M128 x N x K64 int8 MMA pair with K-major SWIZZLE_64B
// operands (the layout the FP32 path already uses, with 64 int8 k-values per 64-byte row) against
// a CPU product, (2) the sustained MMA rate per SM for N = 64 / 128 / 256 from one CTA per SM
// issuing a long chain, operands resident in shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbi8 tools/microbench_i8.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(512u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)4u << 61);
}
// SWIZZLE_32B variant (32-byte rows = 32 int8 k-values; next-round k-tiles of 32 waste less
// padding on I_q0 = 200 than 64): layout type 6, SBO = 8 rows x 32 B = 256 B
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(256u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)6u << 61);
}
__host__ __device__ inline uint32_t sw32_off(int row, int k) {
  const int ch = k >> 4;
  return (uint32_t)(row >> 3) * 256u + (uint32_t)(row & 7) * 32u + (uint32_t)((ch ^ ((row & 7) >> 2)) & 1) * 16u +
         (uint32_t)(k & 15);
}

template <int N>
__global__ void i8_sw32_check(const int8_t* A, const int8_t* B, int* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;              // 128 x 32 int8, SW32
  uint8_t* sb = sm + 128 * 32;   // N x 32 int8, SW32
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * 32; e += blockDim.x) sa[sw32_off(e / 32, e % 32)] = (uint8_t)A[e];
  for (int e = tid; e < N * 32; e += blockDim.x) sb[sw32_off(e / 32, e % 32)] = (uint8_t)B[e];
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 0) {
    if (lane == 0) {
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                   "l"(desc_sw32(smem_u32(sa))), "l"(desc_sw32(smem_u32(sb))),
                   "r"((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24)));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    }
    __syncwarp();
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp < 4) {
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int q = 0; q < 16; ++q) D[(warp * 32 + lane) * N + c + q] = (int)r[q];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

// kind::i8: D s32 (2 << 4), A s8 (1 << 7), B s8 (1 << 10), K-major both, N >> 3, M >> 4
__device__ __forceinline__ uint32_t idesc_i8(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
               "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}
// byte offset of (row, k) in a K-major SWIZZLE_64B tile of 64-byte rows (8-row groups of 512 B)
__host__ __device__ inline uint32_t sw64_off(int row, int k) {
  const int ch = k >> 4;
  return (uint32_t)(row >> 3) * 512u + (uint32_t)(row & 7) * 64u + (uint32_t)((ch ^ ((row & 7) >> 1)) & 3) * 16u +
         (uint32_t)(k & 15);
}

template <int N>
__global__ void i8_kernel(const int8_t* A, const int8_t* B, int* D, int reps, long long* clk) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;               // 128 x 64 int8, SW64
  uint8_t* sb = sm + 128 * 64;    // N x 64 int8, SW64
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 128 * 64; e += blockDim.x) sa[sw64_off(e / 64, e % 64)] = (uint8_t)A[e];
  for (int e = tid; e < N * 64; e += blockDim.x) sb[sw64_off(e / 64, e % 64)] = (uint8_t)B[e];
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t idesc = idesc_i8(N);
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    long long t0 = clock64();
    if (lane == 0) {
      for (int r = 0; r < reps; ++r)
        for (int kk = 0; kk < 2; ++kk)  // 2 x K32 = the 64-byte row
          mma_i8(tmem, desc_sw64(a0 + kk * 32), desc_sw64(b0 + kk * 32), idesc, (r | kk) ? 1u : 0u);
      commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane == 0) clk[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp < 4 && blockIdx.x == 0) {  // D rows = TMEM lanes (32 per warp), N int32 columns
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int q = 0; q < 16; ++q) D[(warp * 32 + lane) * N + c + q] = (int)r[q];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

template <int N>
void run(int sms) {
  int8_t hA[128 * 64], hB[N * 64];
  for (int i = 0; i < 128 * 64; ++i) hA[i] = (int8_t)((i * 37 % 129) - 64);
  for (int i = 0; i < N * 64; ++i) hB[i] = (int8_t)((i * 53 % 127) - 63);
  int8_t *dA, *dB;
  int* dD;
  long long* dclk;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dD, 128 * N * 4);
  cudaMalloc(&dclk, sms * 8);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  const int smem = 128 * 64 + N * 64 + 1024;
  cudaFuncSetAttribute(i8_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // correctness: reps = 1 -> D = A B^T over K = 64
  i8_kernel<N><<<1, 128, smem>>>(dA, dB, dD, 1, dclk);
  static int hD[128 * 256];
  cudaError_t e = cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      int s = 0;
      for (int k = 0; k < 64; ++k) s += hA[m * 64 + k] * hB[n * 64 + k];
      if (s != hD[m * N + n]) ++bad;
    }
  // rate: one CTA per SM, 4096 x 2 MMAs each
  const int reps = 4096;
  i8_kernel<N><<<sms, 128, smem>>>(dA, dB, dD, reps, dclk);
  e = cudaDeviceSynchronize();
  long long hclk[256];
  cudaMemcpy(hclk, dclk, sms * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = hclk[i] > mx ? hclk[i] : mx;
  const double macs = 2.0 * reps * 128.0 * N * 32.0;
  printf("kind::i8 M128 N%-3d K32: layout check %s (%s); %.0f MAC/clk/SM -> %.2f POPS at 1.965 GHz x %d SMs\n", N,
         bad ? "MISMATCH" : "ok", cudaGetErrorString(e), macs / mx, 2.0 * macs / mx * 1.965e9 * sms / 1e15, sms);
}

int sw32_check() {
  const int N = 64;
  static int8_t hA[128 * 32], hB[N * 32];
  for (int i = 0; i < 128 * 32; ++i) hA[i] = (int8_t)((i * 37 % 129) - 64);
  for (int i = 0; i < N * 32; ++i) hB[i] = (int8_t)((i * 53 % 127) - 63);
  int8_t *dA, *dB;
  int* dD;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  i8_sw32_check<N><<<1, 128, 128 * 32 + N * 32 + 1024>>>(dA, dB, dD);
  static int hD[128 * N];
  cudaError_t e = cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      int s = 0;
      for (int k = 0; k < 32; ++k) s += hA[m * 32 + k] * hB[n * 32 + k];
      if (s != hD[m * N + n]) ++bad;
    }
  printf("kind::i8 SWIZZLE_32B (K32 rows) M128 N64: layout check %s (%s)\n", bad ? "MISMATCH" : "ok", cudaGetErrorString(e));
  return bad;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  sw32_check();
  run<64>(sms);
  run<128>(sms);
  run<256>(sms);
  return 0;
}
