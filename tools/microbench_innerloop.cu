// Inner-loop microbenchmark: the MTTKRP k-tile body (A from smem x scale, B from smem,
// 2 x NT DMMA.8x8x4 per k4 step) with no global loads and optional __syncthreads per tile.
// Isolates the DMMA issue efficiency of the loop structure from the data movement.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int NT, bool SYNC, int BK>
__global__ void __launch_bounds__(256, 2) body(double* out, int tiles) {
  __shared__ double As[BK][132];
  __shared__ double Bs[BK][68];
  __shared__ double Ss[128];
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gid = lane >> 2, tig = lane & 3;
  for (int e = tid; e < BK * 132; e += 256) (&As[0][0])[e] = 1e-3 * (e % 7);
  for (int e = tid; e < BK * 68; e += 256) (&Bs[0][0])[e] = 1e-3 * (e % 5);
  if (tid < 128) Ss[tid] = 1.0;
  __syncthreads();
  double acc[2][NT][2] = {};
  for (int t = 0; t < tiles; ++t) {
    if (SYNC) __syncthreads();
    double s0 = Ss[warp * 16 + gid], s1 = Ss[warp * 16 + gid + 8];
    double a[BK / 4][2];
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      a[kk][0] = As[kk * 4 + tig][warp * 16 + gid] * s0;
      a[kk][1] = As[kk * 4 + tig][warp * 16 + gid + 8] * s1;
    }
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
#pragma unroll
      for (int ni = 0; ni < NT; ++ni) {
        double b = Bs[kk * 4 + tig][ni * 8 + gid];
        dmma(acc[0][ni][0], acc[0][ni][1], a[kk][0], b);
        dmma(acc[1][ni][0], acc[1][ni][1], a[kk][1], b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int ni = 0; ni < NT; ++ni) s += acc[0][ni][0] + acc[0][ni][1] + acc[1][ni][0] + acc[1][ni][1];
  out[blockIdx.x * 256 + tid] = s;
}

template <int NT, bool SYNC, int BK>
void run(double* out, int sms, int cps) {
  int tiles = 4000 * 16 / BK;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  body<NT, SYNC, BK><<<sms * cps, 256>>>(out, 10);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  body<NT, SYNC, BK><<<sms * cps, 256>>>(out, tiles);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double flops = 2.0 * (double)sms * cps * 8 * 16 * NT * 8 * BK * tiles;
  printf("NT=%d sync=%d BK=%d ctas/sm=%d: %.2f TFLOP/s\n", NT, SYNC, BK, cps, flops / (ms * 1e-3) / 1e12);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 4 * 256);
  for (int cps : {1, 2}) {
    run<7, false, 16>(out, sms, cps);
    run<7, true, 16>(out, sms, cps);
    run<8, false, 16>(out, sms, cps);
    run<8, true, 16>(out, sms, cps);
    run<4, false, 16>(out, sms, cps);

  }
  return 0;
}
