// CSR -> CSC of a fixed pattern on the device: the transpose index of
// SparseMatrix._transpose_index (sparse.py:129-139 in the reference: stable
// argsort of the column indices, CSC offsets = cumsum(bincount), CSC rows =
// coo_rows[perm]).  Integer work, bit-exact with the host's stable argsort.
//
// Stability comes from the CSR order itself: inside a column the entries must
// keep increasing row order, i.e. CSR order.  Rows are cut into B contiguous
// blocks; per block a column histogram c_b[j] (atomics on ints: order-free,
// deterministic counts); a column-wise exclusive scan over blocks turns c_b[j]
// into the number of column-j entries in earlier blocks; the CSC offsets are
// the exclusive scan of the column totals; finally each block walks its rows
// IN ORDER (one row per step, the row's entries in parallel -- they have
// distinct columns) and hands out positions t_ptr[j] + c_b[j]++.
// HBM-bound: a few passes over nnz int32 plus the B x n counter table.
#include "lr_common.cuh"

namespace lr {

constexpr int TP_THREADS = 256;

static int tp_blocks(int m, int n) {
  // B row blocks: ~1000 CTAs keep every SM busy while each walks its rows in
  // order (one row-latency chain per CTA); the counter table stays <= 256 Mi ints
  long long B = (long long)m / 32 + 1;
  if (B > 512) B = 512;
  const long long cap = (256LL << 20) / (n > 0 ? n : 1);
  if (B > cap) B = cap;
  if (B < 1) B = 1;
  return (int)B;
}

__global__ void tp_hist_kernel(const int* __restrict__ ptr, const int* __restrict__ idx, int m, int n, int B,
                               int* __restrict__ cnt) {
  const int b = blockIdx.x;
  const long long r0 = (long long)m * b / B, r1 = (long long)m * (b + 1) / B;
  const int e0 = ptr[r0], e1 = ptr[r1];
  int* cb = cnt + (long long)b * n;
  for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(cb + idx[e], 1);
}

// per column j: c_b[j] <- sum_{b' < b} c_b'[j]; tot[j] = sum_b c_b[j]
__global__ void tp_colscan_kernel(int* __restrict__ cnt, int n, int B, int* __restrict__ tot) {
  constexpr int U = 16;  // loads in flight per thread (the walk down a column is latency-bound)
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    int run = 0;
    int b = 0;
    for (; b + U <= B; b += U) {
      int c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = cnt[(long long)(b + u) * n + j];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        cnt[(long long)(b + u) * n + j] = run;
        run += c[u];
      }
    }
    for (; b < B; ++b) {
      const long long o = (long long)b * n + j;
      const int c = cnt[o];
      cnt[o] = run;
      run += c;
    }
    tot[j] = run;
  }
}

// t_ptr = exclusive scan of tot (n + 1 entries), one CTA
__global__ void __launch_bounds__(1024) tp_ptrscan_kernel(const int* __restrict__ tot, int n, int* __restrict__ t_ptr) {
  __shared__ int part[1024];
  const int tid = threadIdx.x;
  const int per = (n + 1023) / 1024;
  const int lo = tid * per, hi = min(n, lo + per);
  int s = 0;
  for (int j = lo; j < hi; ++j) s += tot[j];
  part[tid] = s;
  __syncthreads();
  // Hillis-Steele inclusive scan of the 1024 partials
  for (int o = 1; o < 1024; o <<= 1) {
    const int v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int run = tid ? part[tid - 1] : 0;
  for (int j = lo; j < hi; ++j) {
    t_ptr[j] = run;
    run += tot[j];
  }
  if (tid == 1023) t_ptr[n] = part[1023];
}

__global__ void __launch_bounds__(TP_THREADS) tp_scatter_kernel(const int* __restrict__ ptr, const int* __restrict__ idx,
                                                              int m, int n, int B, int* __restrict__ cnt,
                                                              const int* __restrict__ t_ptr, int* __restrict__ t_idx,
                                                              int* __restrict__ perm, int* __restrict__ inv_perm) {
  const int b = blockIdx.x;
  const int r0 = (int)((long long)m * b / B), r1 = (int)((long long)m * (b + 1) / B);
  int* cb = cnt + (long long)b * n;
  for (int i = r0; i < r1; ++i) {
    const int e0 = ptr[i], e1 = ptr[i + 1];
    for (int e = e0 + threadIdx.x; e < e1; e += TP_THREADS) {
      const int j = idx[e];
      const int pos = t_ptr[j] + cb[j];  // columns within a row are distinct: no race
      cb[j] += 1;
      t_idx[pos] = i;
      perm[pos] = e;
      inv_perm[e] = pos;
    }
    __syncthreads();  // the next row sees this row's cursor bumps
  }
}

}  // namespace lr

using namespace lr;

extern "C" {

long long lr_csr_transpose_workspace_ints(int m, int n) {
  return (long long)tp_blocks(m, n) * n + n + 64;
}

int lr_csr_transpose_i32(int m, int n, long long nnz, const int* ptr, const int* idx, int* t_ptr, int* t_idx,
                         int* perm, int* inv_perm, int* work, long long work_ints, void* stream) {
  LR_REQUIRE(m >= 1 && n >= 1 && nnz >= 0, "csr_transpose: bad shape %dx%d nnz=%lld", m, n, nnz);
  LR_REQUIRE(nnz < (1LL << 31), "csr_transpose: nnz %lld exceeds int32 indexing", nnz);
  const int B = tp_blocks(m, n);
  LR_REQUIRE(work_ints >= (long long)B * n + n, "csr_transpose: workspace too small");
  cudaStream_t s = as_stream(stream);
  int* cnt = work;
  int* tot = work + (long long)B * n;
  LR_CHECK_CUDA(cudaMemsetAsync(cnt, 0, (size_t)B * n * sizeof(int), s));
  if (nnz > 0) {
    tp_hist_kernel<<<B, TP_THREADS, 0, s>>>(ptr, idx, m, n, B, cnt);
    LR_CHECK_LAUNCH();
  }
  int cblocks = (n + 255) / 256;
  if (cblocks > sm_count() * 8) cblocks = sm_count() * 8;
  tp_colscan_kernel<<<cblocks, 256, 0, s>>>(cnt, n, B, tot);
  LR_CHECK_LAUNCH();
  tp_ptrscan_kernel<<<1, 1024, 0, s>>>(tot, n, t_ptr);
  LR_CHECK_LAUNCH();
  if (nnz > 0) {
    tp_scatter_kernel<<<B, TP_THREADS, 0, s>>>(ptr, idx, m, n, B, cnt, t_ptr, t_idx, perm, inv_perm);
    LR_CHECK_LAUNCH();
  }
  return LR_OK;
}

}  // extern "C"
