// Latency of cluster.sync() (16 and 8 CTAs, 512 threads) and of a DSMEM remote load.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(512) ksync(long long* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[1024];
  buf[threadIdx.x] = threadIdx.x;
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  // dependent remote loads (pointer chase across ranks)
  double acc = 0.0;
  int idx = threadIdx.x & 1023;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double* rb = cl.map_shared_rank(buf, (cl.block_rank() + 1 + i) % cl.num_blocks());
    acc += rb[idx];
    idx = ((int)acc + i) & 1023;
  }
  long long t3 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) {
    out[0] = (t1 - t0) / iters;
    out[1] = (t3 - t2) / iters;
    out[2] = (long long)acc;
  }
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 64);
  cudaFuncSetAttribute(ksync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, ksync, out, 2000);
    cudaDeviceSynchronize();
    printf("cluster %2d: %s cluster.sync %lld cycles, dependent DSMEM load+add %lld cycles\n", cs,
           cudaGetErrorString(e), out[0], out[1]);
  }
  return 0;
}
