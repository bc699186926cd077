// Latency of dependent fp64 ops on one warp (cycles per op): DFMA, DADD, div, sqrt, shfl.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed, int iters) {
  double a = seed + threadIdx.x * 1e-9, b = 1.0000001, c = 1e-12;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
  // div chain
  double d = a;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { d = 1.5 / d; d = 1.5 / d; d = 1.5 / d; d = 1.5 / d; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0);
  // sqrt chain
  double s = d + 2.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { s = sqrt(s) + 1.0; s = sqrt(s) + 1.0; s = sqrt(s) + 1.0; s = sqrt(s) + 1.0; }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0);
  // shfl chain (double)
  double h = s;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    h = __shfl_sync(0xffffffffu, h, (threadIdx.x + 1) & 31); h = __shfl_sync(0xffffffffu, h, (threadIdx.x + 1) & 31);
    h = __shfl_sync(0xffffffffu, h, (threadIdx.x + 1) & 31); h = __shfl_sync(0xffffffffu, h, (threadIdx.x + 1) & 31);
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0);
  // syncthreads (8 warps)
  t0 = clock64();
  for (int i = 0; i < iters; ++i) { __syncthreads(); __syncthreads(); __syncthreads(); __syncthreads(); }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0);
  out[threadIdx.x] = a + d + s + h;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 8 * 8);
  int iters = 1000;
  for (int threads : {32, 256}) {
    k<<<1, threads>>>(out, cyc, 1.0, iters); cudaDeviceSynchronize();
    k<<<1, threads>>>(out, cyc, 1.0, iters); cudaDeviceSynchronize();
    const char* names[] = {"dfma", "ddiv", "dsqrt+add", "shfl.f64", "syncthreads"};
    printf("threads=%d:", threads);
    for (int i = 0; i < 5; ++i) printf(" %s %.1f", names[i], cyc[i] / (4.0 * iters));
    printf(" cycles/op\n");
  }
  return 0;
}
