// Cost of a cooperative-groups grid barrier on B200 vs CTA count.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
// flag-based barrier: each CTA bumps its own counter slot; CTA 0 waits then releases
__global__ void k2(int iters, volatile unsigned* arrive, volatile unsigned* release) {
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd((unsigned*)arrive, 1u);
      if (blockIdx.x == 0) {
        while (*arrive < (unsigned)(gridDim.x * i)) {}
        __threadfence();
        *release = i;
      } else {
        while (*release < (unsigned)i) {}
      }
      __threadfence();
    }
    __syncthreads();
  }
}
// single-counter barrier: every CTA's thread 0 adds (release) and polls the same word (acquire)
__global__ void k3(int iters, unsigned* ctr) {
  for (int i = 1; i <= iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned v;
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
      const unsigned target = gridDim.x * (unsigned)i;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      } while (v < target);
    }
    __syncthreads();
  }
}
int main() {
  int* out; cudaMalloc(&out, 4);
  unsigned* flags; cudaMalloc(&flags, 64); 
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int G : {1, 16, 74, 148, 296}) {
    for (int threads : {256}) {
      int iters = 2000;
      void* args[] = {&iters, &out};
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaLaunchCooperativeKernel((void*)k, G, threads, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k, G, threads, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      cudaMemset(flags, 0, 64);
      void* args2[] = {&iters, &flags, &flags + 0};
      unsigned* rel = flags + 8;
      void* args3[] = {&iters, (void*)&flags, (void*)&rel};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k2, G, threads, args3, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms2; cudaEventElapsedTime(&ms2, a, b);
      cudaMemset(flags, 0, 64);
      unsigned* ctr = flags + 4;
      void* args4[] = {&iters, (void*)&ctr};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k3, G, threads, args4, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms3; cudaEventElapsedTime(&ms3, a, b);
      printf("G=%d threads=%d: cg grid.sync %.3f us, flag barrier %.3f us, single counter (red.release + ld.acquire) %.3f us  (%s)\n", G, threads, ms * 1000 / iters, ms2 * 1000 / iters, ms3 * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
      (void)args2;
    }
  }
  return 0;
}
