// Does the DMMA (FP64 tensor) path share its throughput with DFMA on sm_100a? Even warps run
// m16n8k8 f64 MMAs, odd warps run DFMA chains; compare the combined FLOP rate with each alone.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbmix tools/microbench_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma_body(double* out, int iters) {
  double acc[8][4] = {};
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-4, a2 = a0 + 2e-4, a3 = a0 + 3e-4;
  double b0 = 1.0 + 1e-9 * threadIdx.x, b1 = b0 + 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void dfma_body(double* out, int iters) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = i;
  double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma(double* out, int it) { dmma_body(out, it); }
__global__ void k_dfma(double* out, int it) { dfma_body(out, it); }
__global__ void k_mix(double* out, int it_mma, int it_fma) {
  if ((threadIdx.x >> 5) & 1) dfma_body(out, it_fma);
  else dmma_body(out, it_mma);
}

template <class F>
float tm(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 2 * 512);
  const int blocks = sms * 2, threads = 512;  // 16 warps per CTA
  const double warps = blocks * 16.0;
  const int itm = 4000, itf = 16000;
  const double fl_mma = 8.0 * 16 * 8 * 8 * 2;      // per warp-iteration (8 MMAs m16n8k8)
  const double fl_fma = 32.0 * 16 * 2;             // per warp-iteration (16 DFMA x 32 lanes)
  float t1 = tm([&] { k_dmma<<<blocks, threads>>>(out, itm); });
  printf("DMMA only : %.2f TFLOP/s\n", warps * itm * fl_mma / (t1 * 1e-3) / 1e12);
  float t2 = tm([&] { k_dfma<<<blocks, threads>>>(out, itf); });
  printf("DFMA only : %.2f TFLOP/s\n", warps * itf * fl_fma / (t2 * 1e-3) / 1e12);
  float t3 = tm([&] { k_mix<<<blocks, threads>>>(out, itm, itf); });
  const double fl = warps / 2 * itm * fl_mma + warps / 2 * itf * fl_fma;
  printf("mixed     : %.2f TFLOP/s combined (half the warps each; %.3f ms)\n", fl / (t3 * 1e-3) / 1e12, t3);
  return 0;
}
