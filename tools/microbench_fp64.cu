// FP64 pipe microbenchmark for sm_100a: DMMA (mma.sync f64) shapes vs DFMA.
// Purpose: decide the MTTKRP inner product instruction (SURVEY §7 hard part 1).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_fp64.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_k4(double* out, int iters) {
  double acc[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-4, b0 = 1.0 + 1e-9 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a0), "d"(a1), "d"(b0));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_k8(double* out, int iters) {
  double acc[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1e-4, a2 = a0 + 2e-4, a3 = a0 + 3e-4;
  double b0 = 1.0 + 1e-9 * threadIdx.x, b1 = b0 + 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_k16(double* out, int iters) {
  double acc[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i * 1e-4;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = i;
  double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// fragment-layout check for m16n8k4: D = A(16x4,row) * B(4x8,col)
__global__ void layout_k4(const double* A, const double* B, double* D) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a0 = A[g * 4 + t], a1 = A[(g + 8) * 4 + t];
  double b0 = B[t * 8 + g];
  double d0 = 0, d1 = 0, d2 = 0, d3 = 0;
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};\n"
               : "+d"(d0), "+d"(d1), "+d"(d2), "+d"(d3) : "d"(a0), "d"(a1), "d"(b0));
  D[g * 8 + 2 * t] = d0; D[g * 8 + 2 * t + 1] = d1;
  D[(g + 8) * 8 + 2 * t] = d2; D[(g + 8) * 8 + 2 * t + 1] = d3;
}

template <typename F>
double time_it(F f, int reps = 5) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; CK(cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024));
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      int blocks = sms * bps, threads = 32 * wpb;
      double warps = (double)blocks * wpb;
      double ms;
      ms = time_it([&] { dmma_k4<8><<<blocks, threads>>>(out, iters); });
      printf("DMMA m16n8k4  acc=8  wpb=%2d bps=%d : %.2f TFLOP/s\n", wpb, bps, warps * iters * 8 * 16 * 8 * 4 * 2 / (ms * 1e-3) / 1e12);
      ms = time_it([&] { dmma_k8<8><<<blocks, threads>>>(out, iters / 2); });
      printf("DMMA m16n8k8  acc=8  wpb=%2d bps=%d : %.2f TFLOP/s\n", wpb, bps, warps * (iters / 2) * 8 * 16 * 8 * 8 * 2 / (ms * 1e-3) / 1e12);
      ms = time_it([&] { dmma_k16<8><<<blocks, threads>>>(out, iters / 4); });
      printf("DMMA m16n8k16 acc=8  wpb=%2d bps=%d : %.2f TFLOP/s\n", wpb, bps, warps * (iters / 4) * 8 * 16 * 8 * 16 * 2 / (ms * 1e-3) / 1e12);
      ms = time_it([&] { dfma_loop<16><<<blocks, threads>>>(out, iters * 4); });
      printf("DFMA          acc=16 wpb=%2d bps=%d : %.2f TFLOP/s\n", wpb, bps, warps * 32.0 * iters * 4 * 16 * 2 / (ms * 1e-3) / 1e12);
    }
  }
  // small accumulator count: single-warp DMMA latency-boundness
  {
    int blocks = sms, threads = 128; double warps = blocks * 4.0;
    double ms = time_it([&] { dmma_k4<1><<<blocks, threads>>>(out, iters * 4); });
    printf("DMMA m16n8k4  acc=1 (dependent chain) wpb=4: %.2f TFLOP/s  (latency ~%.1f cyc @1.9GHz)\n",
           warps * iters * 4 * 1024 / (ms * 1e-3) / 1e12, ms * 1e-3 * 1.9e9 / (iters * 4));
  }
  // layout check
  double hA[64], hB[32], hD[128], *dA, *dB, *dD;
  for (int i = 0; i < 64; ++i) hA[i] = (i * 7 % 13) - 6;
  for (int i = 0; i < 32; ++i) hB[i] = (i * 5 % 11) - 5;
  CK(cudaMalloc(&dA, 512)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dD, 1024));
  cudaMemcpy(dA, hA, 512, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  layout_k4<<<1, 32>>>(dA, dB, dD); CK(cudaMemcpy(hD, dD, 1024, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < 16; ++m) for (int n = 0; n < 8; ++n) {
    double s = 0; for (int k = 0; k < 4; ++k) s += hA[m * 4 + k] * hB[k * 8 + n];
    if (s != hD[m * 8 + n]) ++bad;
  }
  printf("m16n8k4 layout check: %s\n", bad ? "MISMATCH" : "ok");
  return 0;
}
