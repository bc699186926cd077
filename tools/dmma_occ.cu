// DMMA m8n8k4 throughput vs resident warps per SM, 32 independent accumulators per warp
// (the GEMM's 64x32 warp tile), plus the same with 2 smem fragment loads per 4 DMMAs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, int iters, int use_smem) {
  __shared__ double sm[1024];
  double a = threadIdx.x * 1e-3, b = 0.5;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  double c[32][2];
#pragma unroll
  for (int q = 0; q < 32; ++q) { c[q][0] = 0; c[q][1] = 0; }
  for (int it = 0; it < iters; ++it) {
    double af[8], bf[4];
    if (use_smem) {
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = sm[(it * 8 + i * 33 + threadIdx.x) & 1023];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = sm[(it * 4 + j * 65 + threadIdx.x * 3) & 1023];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = a + i;
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = b + j;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i * 4 + j][0]), "+d"(c[i * 4 + j][1]) : "d"(af[i]), "d"(bf[j]));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 32; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out; cudaMalloc(&out, 148 * 16 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2000;
  for (int use_smem = 0; use_smem < 2; ++use_smem)
    for (int wps : {2, 4, 8, 12, 16, 24, 32}) {
      int threads = 128, blocks = 148 * wps / 4;
      k<<<blocks, threads>>>(out, 10, use_smem);
      cudaEventRecord(e0); k<<<blocks, threads>>>(out, iters, use_smem); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = 2.0 * 256 * 32 * (double)iters * (blocks * threads / 32);
      printf("smem=%d warps/SM=%2d: %.2f TFLOP/s\n", use_smem, wps, fl / ms / 1e9);
    }
  return 0;
}
