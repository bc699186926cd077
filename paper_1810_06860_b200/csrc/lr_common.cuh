// Shared helpers for the sm_100a kernels of the lowrank B200 library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/lowrank_b200.h"

namespace lr {

void set_error(const char* fmt, ...);
int sm_count();

#define LR_CHECK_CUDA(call)                                                            \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::lr::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
      return LR_ERR_CUDA;                                                              \
    }                                                                                  \
  } while (0)

// Every kernel launch is followed by LR_CHECK_LAUNCH(), which also counts it
// (lr_launch_count(): the bench's "gpu_launches" claim).
void count_launches(long long n);

#define LR_CHECK_LAUNCH_N(nlaunch)                                                      \
  do {                                                                                  \
    ::lr::count_launches(nlaunch);                                                      \
    cudaError_t _e = cudaGetLastError();                                                \
    if (_e != cudaSuccess) {                                                            \
      ::lr::set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e));  \
      return LR_ERR_CUDA;                                                               \
    }                                                                                   \
  } while (0)

#define LR_CHECK_LAUNCH()                                                               \
  do {                                                                                  \
    ::lr::count_launches(1);                                                            \
    cudaError_t _e = cudaGetLastError();                                                \
    if (_e != cudaSuccess) {                                                            \
      ::lr::set_error("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e));  \
      return LR_ERR_CUDA;                                                               \
    }                                                                                   \
  } while (0)

#define LR_REQUIRE(cond, ...)        \
  do {                               \
    if (!(cond)) {                   \
      ::lr::set_error(__VA_ARGS__);  \
      return LR_ERR_ARG;             \
    }                                \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// integer tuning knob from the environment, clamped to [lo, hi] (default when unset)
int env_int_clamped(const char* name, int dflt, int lo, int hi);

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order block reduction (sum). Result valid in thread 0.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (l < THREADS / 32) ? sh[l] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}
template <int THREADS>
__device__ __forceinline__ double block_max(double v, double* sh) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (l < THREADS / 32) ? sh[l] : 0.0;
    r = warp_max(r);
  }
  __syncthreads();
  return r;
}

// Streaming loads that do not allocate in L1 (the CSR index / value / M / Y
// streams of the sparse kernels): L1 keeps the gathered dense rows, whose
// Zipf-hot part it can serve.
__device__ __forceinline__ int ld_stream(const int* p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
// Y (read-write in the same kernel): plain load without L1 allocation
__device__ __forceinline__ double ld_stream_rw(const double* p) {
  double v;
  asm("ld.global.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Non-contracted arithmetic where the reference's numpy expression has no FMA.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

}  // namespace lr
