// Coordinate triples -> CSR on the device: ObservationSet's validation and
// SparseMatrix.from_coo (reference sparse.py:84-104 and :259-328: bounds,
// duplicate cells rejected, lexsort by (row, col), indptr = cumsum(bincount)).
// Integer work, bit-exact with the host lexsort: with distinct cells the
// sorted order is unique, so the build may bucket rows with atomics (order
// inside a row is then arbitrary) and sort every row segment by column.
//
//   1. coo_hist   : bounds check, per-row counts of the selected entries
//                   (entries whose split tag equals `tag`, or all)
//   2. coo_scan   : indptr = exclusive scan of the counts (one CTA)
//   3. coo_bucket : each entry takes a slot of its row (atomic row cursor)
//   4. coo_rowsort: one CTA per row sorts its (column, source) pairs by column
//                   (bitonic, in shared memory up to 4096 entries, in place in
//                   global memory beyond) and records the first duplicate
//                   cell in CSR order (atomicMin of the slot)
//   5. coo_emit   : int32 column indices, values gathered in CSR order
// HBM-bound apart from the row sorts (log^2 of the row length per entry).
#include "lr_common.cuh"

namespace lr {

constexpr int kCooThreads = 256;
constexpr int kRowSortSmem = 4096;  // entries sorted in shared memory (32 KB)

__global__ void coo_hist_kernel(const long long* __restrict__ rows, const long long* __restrict__ cols,
                                const unsigned char* __restrict__ split, int tag, long long count, int m, int n,
                                int* __restrict__ row_cnt, int* __restrict__ flags) {
  int bad = 0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x) {
    if (split && (int)split[e] != tag) continue;
    const long long i = rows[e], j = cols[e];
    if (i < 0 || i >= m || j < 0 || j >= n) {
      bad |= (i < 0 || i >= m) ? 1 : 4;  // 1: a row out of range, 4: a column
      continue;
    }
    atomicAdd(row_cnt + i, 1);
  }
  if (bad) atomicOr(flags, bad);
}

// ptr[0..m] = exclusive scan of cnt[0..m-1]; one CTA of 1024 threads
__global__ void __launch_bounds__(1024) coo_scan_kernel(const int* __restrict__ cnt, int m, int* __restrict__ ptr) {
  __shared__ long long part[1024];
  const int tid = threadIdx.x;
  const int per = (m + 1023) / 1024;
  const int lo = min(m, tid * per), hi = min(m, lo + per);
  long long s = 0;
  for (int i = lo; i < hi; ++i) s += cnt[i];
  part[tid] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const long long v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  long long run = tid ? part[tid - 1] : 0;
  for (int i = lo; i < hi; ++i) {
    ptr[i] = (int)run;
    run += cnt[i];
  }
  if (tid == 1023) ptr[m] = (int)part[1023];
}

__global__ void coo_bucket_kernel(const long long* __restrict__ rows, const long long* __restrict__ cols,
                                  const unsigned char* __restrict__ split, int tag, long long count,
                                  const int* __restrict__ ptr, int* __restrict__ cursor, int* __restrict__ tcol,
                                  int* __restrict__ tsrc) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x) {
    if (split && (int)split[e] != tag) continue;
    const int i = (int)rows[e];
    const int pos = ptr[i] + atomicAdd(cursor + i, 1);
    tcol[pos] = (int)cols[e];
    tsrc[pos] = (int)e;
  }
}

// bitonic sort of len (column, source) pairs by column, padded to a power of
// two with +inf columns; col/src point to shared or global memory
__device__ void bitonic_pairs(int* col, int* src, int len, int P) {
  for (int t = len + threadIdx.x; t < P; t += blockDim.x) col[t] = 0x7fffffff;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int t = threadIdx.x; t < P; t += blockDim.x) {
        const int u = t ^ jj;
        if (u > t) {
          const bool up = (t & k) == 0;
          const int a = col[t], b = col[u];
          if ((a > b) == up) {
            col[t] = b;
            col[u] = a;
            const int sa = src[t];
            src[t] = src[u];
            src[u] = sa;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(kCooThreads) coo_rowsort_kernel(const int* __restrict__ ptr, int m,
                                                                  int* __restrict__ tcol, int* __restrict__ tsrc,
                                                                  int* __restrict__ gcol, int* __restrict__ gsrc,
                                                                  int* __restrict__ first_dup) {
  __shared__ int scol[kRowSortSmem];
  __shared__ int ssrc[kRowSortSmem];
  for (int i = blockIdx.x; i < m; i += gridDim.x) {
    const int b = ptr[i], len = ptr[i + 1] - b;
    if (len <= 0) continue;
    if (len > 1) {
      int P = 1;
      while (P < len) P <<= 1;
      if (P <= kRowSortSmem) {
        for (int t = threadIdx.x; t < len; t += kCooThreads) {
          scol[t] = tcol[b + t];
          ssrc[t] = tsrc[b + t];
        }
        __syncthreads();
        bitonic_pairs(scol, ssrc, len, P);
        for (int t = threadIdx.x; t < len; t += kCooThreads) {
          tcol[b + t] = scol[t];
          tsrc[b + t] = ssrc[t];
        }
      } else {  // long row: the same network in global scratch, rows at 2 * offset (P < 2 len: disjoint)
        int* gc = gcol + 2LL * b;
        int* gs = gsrc + 2LL * b;
        for (int t = threadIdx.x; t < len; t += kCooThreads) {
          gc[t] = tcol[b + t];
          gs[t] = tsrc[b + t];
        }
        __syncthreads();
        bitonic_pairs(gc, gs, len, P);
        for (int t = threadIdx.x; t < len; t += kCooThreads) {
          tcol[b + t] = gc[t];
          tsrc[b + t] = gs[t];
        }
      }
      __syncthreads();
      for (int t = threadIdx.x; t + 1 < len; t += kCooThreads)
        if (tcol[b + t] == tcol[b + t + 1]) atomicMin(first_dup, b + t);
      __syncthreads();
    }
  }
}

__global__ void coo_emit_kernel(const int* __restrict__ tsrc, long long nnz, const double* __restrict__ vals,
                                double* __restrict__ out_vals, int* __restrict__ flags) {
  int nonfin = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < nnz;
       p += (long long)gridDim.x * blockDim.x) {
    const double v = vals[tsrc[p]];
    out_vals[p] = v;
    nonfin |= !isfinite(v);
  }
  if (nonfin) atomicOr(flags, 2);
}

static int coo_grid(long long count) {
  long long b = (count + kCooThreads - 1) / kCooThreads;
  const long long cap = (long long)sm_count() * 16;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace lr

using namespace lr;

extern "C" {

long long lr_coo_to_csr_workspace_ints(int m, long long count) {
  // row counts + cursors (2m), flags + first duplicate (64), long-row scratch (2 x 2 count)
  return 2LL * m + 64 + 4 * count;
}

int lr_coo_to_csr_i32(int m, int n, long long count, const long long* rows, const long long* cols,
                      const unsigned char* split, int tag, const double* vals, int* ptr, int* col_out, int* src_out,
                      double* vals_out, int* work, long long work_ints, int* status_host, void* stream) {
  LR_REQUIRE(m >= 1 && n >= 1 && count >= 0, "coo_to_csr: bad shape %dx%d count=%lld", m, n, count);
  LR_REQUIRE(count < (1LL << 31), "coo_to_csr: %lld entries exceed int32 indexing", count);
  LR_REQUIRE(work_ints >= lr_coo_to_csr_workspace_ints(m, count), "coo_to_csr: workspace too small");
  cudaStream_t s = as_stream(stream);
  int* row_cnt = work;
  int* cursor = work + m;
  int* flags = work + 2LL * m;          // [0] error bits, [1] first duplicate slot
  int* gcol = flags + 64;
  int* gsrc = gcol + 2 * count;
  LR_CHECK_CUDA(cudaMemsetAsync(work, 0, (2LL * m + 64) * sizeof(int), s));
  LR_CHECK_CUDA(cudaMemsetAsync(flags + 1, 0x7f, sizeof(int), s));  // first duplicate = 0x7f7f7f7f (none)
  const int grid = coo_grid(count);
  if (count > 0) {
    coo_hist_kernel<<<grid, kCooThreads, 0, s>>>(rows, cols, split, tag, count, m, n, row_cnt, flags);
    LR_CHECK_LAUNCH();
  }
  coo_scan_kernel<<<1, 1024, 0, s>>>(row_cnt, m, ptr);
  LR_CHECK_LAUNCH();
  int h[2] = {0, 0};
  int nnz = 0;
  LR_CHECK_CUDA(cudaMemcpyAsync(h, flags, sizeof(int), cudaMemcpyDeviceToHost, s));
  LR_CHECK_CUDA(cudaMemcpyAsync(&nnz, ptr + m, sizeof(int), cudaMemcpyDeviceToHost, s));
  LR_CHECK_CUDA(cudaStreamSynchronize(s));
  if (h[0] & 5) {
    status_host[0] = (h[0] & 1) ? 1 : 3;  // 1: a row out of range, 3: a column out of range
    status_host[1] = -1;
    status_host[2] = 0;
    return LR_OK;
  }
  if (nnz > 0) {
    coo_bucket_kernel<<<grid, kCooThreads, 0, s>>>(rows, cols, split, tag, count, ptr, cursor, col_out, src_out);
    LR_CHECK_LAUNCH();
    int rb = m < sm_count() * 16 ? m : sm_count() * 16;
    coo_rowsort_kernel<<<rb, kCooThreads, 0, s>>>(ptr, m, col_out, src_out, gcol, gsrc, flags + 1);
    LR_CHECK_LAUNCH();
    if (vals_out) {
      coo_emit_kernel<<<coo_grid(nnz), kCooThreads, 0, s>>>(src_out, nnz, vals, vals_out, flags);
      LR_CHECK_LAUNCH();
    }
  }
  LR_CHECK_CUDA(cudaMemcpyAsync(h, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  LR_CHECK_CUDA(cudaStreamSynchronize(s));
  status_host[0] = (h[0] & 2) ? 2 : 0;                  // 2: non-finite value
  status_host[1] = (h[1] == 0x7f7f7f7f) ? -1 : h[1];    // first duplicate slot in CSR order, or -1
  status_host[2] = nnz;
  return LR_OK;
}

}  // extern "C"
