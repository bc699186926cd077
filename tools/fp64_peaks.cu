// Microbenchmark: fp64 DFMA vs DMMA (mma.sync m8n8k4 f64) throughput, and
// L2 random row-gather bandwidth. Used once to pick the Gram/GEMM design.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 0.5;
  double c[8][4];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; c[k][2] = 0; c[k][3] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// each warp gathers rows of width W doubles at random row indices
__global__ void gather_kernel(const double* __restrict__ X, const int* __restrict__ idx, int nidx, int W,
                              double* out) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  double2 acc = make_double2(0, 0);
  for (int e = warp; e < nidx; e += nw) {
    const double2* row = reinterpret_cast<const double2*>(X + (size_t)idx[e] * W);
    for (int c = lane; c < W / 2; c += 32) { double2 v = __ldg(row + c); acc.x += v.x; acc.y += v.y; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}

int main() {
  double* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 4, threads = 512, iters = 4096;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 64 * iters * (double)blocks * threads;
    if (rep) printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * (blocks * threads / 32);
    if (rep) printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0); dmma16_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 4 * 8 * (double)iters * (blocks * threads / 32);
    if (rep) printf("DMMA m16n8k4: %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
  }
  // gather: X of n rows x W doubles, 5M random indices
  int n = 50000, nidx = 5000000;
  int Ws[] = {16, 64, 110, 660};
  int* hidx = (int*)malloc(nidx * 4);
  uint64_t s = 12345;
  for (int i = 0; i < nidx; ++i) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; hidx[i] = (s >> 33) % n; }
  int* didx; cudaMalloc(&didx, nidx * 4); cudaMemcpy(didx, hidx, nidx * 4, cudaMemcpyHostToDevice);
  for (int W : Ws) {
    double* X; cudaMalloc(&X, (size_t)n * W * 8); cudaMemset(X, 0, (size_t)n * W * 8);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0); gather_kernel<<<148 * 16, 256>>>(X, didx, nidx, W, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("gather W=%d: %.1f GB/s of row bytes (%.3f ms)\n", W, (double)nidx * W * 8 / ms / 1e6, ms);
    cudaFree(X);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
