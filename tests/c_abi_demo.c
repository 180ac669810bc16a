/*
 * c_abi_demo.c -- drives the JK-CALS hot path through the plain C ABI (include/jkcals.h) with
 * no Python in the loop: the boundary is usable from C as declared.
 *
 *   c_abi_demo <in.bin> <out.bin> <sweeps>
 *
 * in.bin  : int64 N, int64 dims[N], int64 R, then T (prod(dims) doubles, column-major, Eq. 3)
 *           and P_0..P_{N-1} (dims[n] x R doubles each, column-major).
 * out.bin : for every submodel p = 0..dims[0]-1 and mode n: its factor in the get_factors layout
 *           ((dims[0]-1) x R for mode 0, dims[n] x R otherwise, column-major), then lambda (R).
 * Exit code 0 on success; any jkcals error prints jkcals_last_error and exits 1.
 */
#include <cuda_runtime_api.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "jkcals.h"

#define CHECK(x)                                                                     \
  do {                                                                               \
    jkcals_status s_ = (x);                                                          \
    if (s_ != JKCALS_OK) {                                                           \
      fprintf(stderr, "%s -> %d: %s\n", #x, (int)s_, h ? jkcals_last_error(h) : ""); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

static int read_all(FILE* f, void* p, size_t n) { return fread(p, 1, n, f) == n; }

int main(int argc, char** argv) {
  if (argc != 4) {
    fprintf(stderr, "usage: %s in.bin out.bin sweeps\n", argv[0]);
    return 2;
  }
  jkcals_t h = NULL;
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 2;
  int64_t N = 0, R = 0, dims[JKCALS_MAX_MODES];
  if (!read_all(f, &N, 8) || N < 3 || N > JKCALS_MAX_MODES || !read_all(f, dims, 8 * (size_t)N) ||
      !read_all(f, &R, 8))
    return 2;
  int64_t P = 1;
  for (int n = 0; n < N; ++n) P *= dims[n];
  double* T = malloc(8 * (size_t)P);
  double* Pm[JKCALS_MAX_MODES];
  if (!T || !read_all(f, T, 8 * (size_t)P)) return 2;
  for (int n = 0; n < N; ++n) {
    Pm[n] = malloc(8 * (size_t)(dims[n] * R));
    if (!Pm[n] || !read_all(f, Pm[n], 8 * (size_t)(dims[n] * R))) return 2;
  }
  fclose(f);

  /* the caller owns the device workspace (here a plain cudaMalloc) and the stream (default) */
  const int hist = atoi(argv[3]);
  size_t bytes = jkcals_workspace_bytes((int)N, dims, (int)R, dims[0], JKCALS_FP64, hist, 0);
  if (bytes == 0) return 3;
  void* ws = NULL;
  if (cudaMalloc(&ws, bytes) != cudaSuccess) return 3;
  CHECK(jkcals_create(&h, (int)N, dims, (int)R, 0, dims[0], T, 0, JKCALS_FP64, 0, NULL, ws, bytes, hist));
  CHECK(jkcals_set_init(h, (const double* const*)Pm));
  int done = 0;
  CHECK(jkcals_iterate(h, hist, 0.0, &done));
  if (done != hist) return 4;

  FILE* o = fopen(argv[2], "wb");
  if (!o) return 2;
  int64_t maxI = 0;
  for (int n = 0; n < N; ++n) maxI = dims[n] > maxI ? dims[n] : maxI;
  double* U = malloc(8 * (size_t)(maxI * R));
  double* lam = malloc(8 * (size_t)R);
  for (int64_t p = 0; p < dims[0]; ++p) {
    for (int n = 0; n < N; ++n) {
      const int64_t rows = n == 0 ? dims[0] - 1 : dims[n];
      CHECK(jkcals_get_factors(h, p, n, U, n == N - 1 ? lam : NULL));
      fwrite(U, 8, (size_t)(rows * R), o);
    }
    fwrite(lam, 8, (size_t)R, o);
  }
  fclose(o);
  jkcals_destroy(h);
  cudaFree(ws);
  printf("c_abi_demo ok: %lld submodels, %d sweeps\n", (long long)dims[0], done);
  return 0;
}
