// L2 read bandwidth: every CTA streams an L2-resident buffer (LDG.128 .cg,
// 4 independent loads per thread per iteration) many times; aggregate bytes/s
// for buffers below and above the 126 MB L2.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double2* __restrict__ x, long long n2, int reps, double* out) {
  double a = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (int r = 0; r < reps; ++r) {
    long long i = t0;
    for (; i + 3 * stride < n2; i += 4 * stride) {
      double2 v0 = __ldcg(x + i), v1 = __ldcg(x + i + stride), v2 = __ldcg(x + i + 2 * stride),
              v3 = __ldcg(x + i + 3 * stride);
      a += (v0.x + v1.y) + (v2.x + v3.y);
    }
    for (; i < n2; i += stride) a += __ldcg(x + i).x;
  }
  if (a == 1234.5) out[0] = a;
}
int main() {
  for (long long mb : {16LL, 32LL, 64LL, 96LL, 1024LL}) {
    long long n2 = mb * 1024 * 1024 / 16;
    double2* x; double* out;
    cudaMalloc(&x, n2 * 16); cudaMalloc(&out, 8);
    cudaMemset(x, 0, n2 * 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = mb <= 96 ? 40 : 4;
    for (int bps : {4, 8}) {
      rd<<<148 * bps, 512>>>(x, n2, 1, out);
      cudaEventRecord(e0); rd<<<148 * bps, 512>>>(x, n2, reps, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("buffer %4lld MB, %d CTAs/SM x 512 thr: %.1f GB/s\n", mb, bps, (double)n2 * 16 * reps / ms / 1e6);
    }
    cudaFree(x); cudaFree(out);
  }
  return 0;
}
