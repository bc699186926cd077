// Blocked upper Cholesky (A = R^T R) and triangular inverse R^{-1} for the
// W x W Grams of CholeskyQR2 / shifted CholeskyQR3 -- the GPU replacement for
// the Householder QR of `orth` (linalg.py:101-124; survey K3).  Diagonal
// 64x64 blocks are factored and inverted in shared memory by one CTA; panel
// and trailing updates are DMMA GEMMs (lr_gemm.cu).  A device flag makes the
// remaining work a no-op after a non-positive pivot; the host reads `info`.
#include "lr_common.cuh"

namespace lr {

constexpr int CH_NB = 64;
constexpr int CH_THREADS = 256;
constexpr int kDiagSmem = 2 * CH_NB * (CH_NB + 1) * sizeof(double);

__global__ void add_diag_kernel(double* A, long long lda, int n, double shift) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    A[(long long)i * lda + i] += shift;
}

// Factor the jb x jb diagonal block at (J,J) in place (upper R), zero its
// strict lower part, write inv(R_JJ) to Dinv (jb x jb, ld CH_NB).
__global__ void __launch_bounds__(CH_THREADS) chol_diag_kernel(double* A, long long lda, int J, int jb,
                                                             double* Dinv, int* info) {
  if (*info != 0) return;
  // 16 x 16 threads, each owns a 4 x 4 tile (rows 4ty.., cols 4tx..) of the
  // 64 x 64 block; indices >= jb are padded with the identity (decoupled).
  extern __shared__ double ch_smem[];
  double(*a)[CH_NB + 1] = reinterpret_cast<double(*)[CH_NB + 1]>(ch_smem);
  double(*x)[CH_NB + 1] = reinterpret_cast<double(*)[CH_NB + 1]>(ch_smem + CH_NB * (CH_NB + 1));
  __shared__ double rowbuf[CH_NB];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int i0 = 4 * ty, c0 = 4 * tx;
#pragma unroll
  for (int di = 0; di < 4; ++di)
#pragma unroll
    for (int dc = 0; dc < 4; ++dc) {
      const int i = i0 + di, c = c0 + dc;
      double v;
      if (i < jb && c < jb)
        v = (c >= i) ? A[(long long)(J + i) * lda + J + c] : 0.0;
      else
        v = (i == c) ? 1.0 : 0.0;
      a[i][c] = v;
      x[i][c] = (i == c) ? 1.0 : 0.0;
    }
  __syncthreads();
  for (int j = 0; j < CH_NB; ++j) {
    const double d = a[j][j];
    if (!(d > 0.0)) {  // uniform: every thread read the same value
      if (tid == 0) *info = J + j + 1;
      return;
    }
    const double r = sqrt(d);
    if (ty == (j >> 2)) {  // owners of row j: finalize it (nobody else touches row j now)
#pragma unroll
      for (int dc = 0; dc < 4; ++dc) {
        const int c = c0 + dc;
        if (c >= j) {
          const double v = (c == j) ? r : a[j][c] / r;
          a[j][c] = v;
          rowbuf[c] = v;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int di = 0; di < 4; ++di)
#pragma unroll
      for (int dc = 0; dc < 4; ++dc) {
        const int i = i0 + di, c = c0 + dc;
        if (i > j && c >= i) a[i][c] = fma(-rowbuf[i], rowbuf[c], a[i][c]);
      }
    __syncthreads();
  }
  // R^{-1} by right-looking back substitution: X = I; for i = n-1..0:
  // X[i,:] /= R_ii; X[r,:] -= R_ri X[i,:] (r < i)
  for (int i = CH_NB - 1; i >= 0; --i) {
    const double rii = a[i][i];
    if (ty == (i >> 2)) {
#pragma unroll
      for (int dc = 0; dc < 4; ++dc) {
        const int c = c0 + dc;
        if (c >= i) {
          const double v = x[i][c] / rii;
          x[i][c] = v;
          rowbuf[c] = v;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int di = 0; di < 4; ++di)
#pragma unroll
      for (int dc = 0; dc < 4; ++dc) {
        const int rr = i0 + di, c = c0 + dc;
        if (rr < i && c >= i) x[rr][c] = fma(-a[rr][i], rowbuf[c], x[rr][c]);
      }
    __syncthreads();
  }
#pragma unroll
  for (int di = 0; di < 4; ++di)
#pragma unroll
    for (int dc = 0; dc < 4; ++dc) {
      const int i = i0 + di, c = c0 + dc;
      if (i < jb && c < jb) {
        A[(long long)(J + i) * lda + J + c] = a[i][c];
        Dinv[i * CH_NB + c] = x[i][c];
      }
    }
}

__global__ void zero_lower_kernel(double* A, long long lda, int n) {
  const long long total = (long long)n * n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int i = (int)(t / n), c = (int)(t % n);
    if (c < i) A[(long long)i * lda + c] = 0.0;
  }
}

// X[I:I+ib, :] block row set from Dinv for the diagonal, zeros to the left
__global__ void inv_place_diag_kernel(double* X, long long ldx, int n, int I, int ib, const double* Dinv) {
  const long long total = (long long)ib * n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int i = (int)(t / n), c = (int)(t % n);
    if (c < I)
      X[(long long)(I + i) * ldx + c] = 0.0;
    else if (c < I + ib)
      X[(long long)(I + i) * ldx + c] = Dinv[i * CH_NB + (c - I)];
  }
}

}  // namespace lr

using namespace lr;

extern "C" {

long long lr_potrf_workspace_doubles(int n) {
  // Dinv blocks + panel temp + gemm split workspace (none: transA gemms here are tiny-K)
  long long nblk = (n + CH_NB - 1) / CH_NB;
  return nblk * CH_NB * CH_NB + (long long)CH_NB * n + 64;
}

int lr_potrf_inv_f64(int n, double* A, long long lda, double shift, double* Rinv, long long ldr,
                     double* work, int* info_host, void* stream) {
  LR_REQUIRE(n >= 1 && lda >= n && ldr >= n, "potrf: bad shape");
  cudaStream_t s = as_stream(stream);
  const long long nblk = (n + CH_NB - 1) / CH_NB;
  double* Dinv = work;
  double* T = work + nblk * CH_NB * CH_NB;  // CH_NB x n
  int* info = reinterpret_cast<int*>(T + (long long)CH_NB * n);
  LR_CHECK_CUDA(cudaMemsetAsync(info, 0, sizeof(int), s));
  static bool attr_set = false;
  if (!attr_set) {
    LR_CHECK_CUDA(cudaFuncSetAttribute(chol_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kDiagSmem));
    attr_set = true;
  }
  if (shift != 0.0) {
    add_diag_kernel<<<(n + 255) / 256, 256, 0, s>>>(A, lda, n, shift);
    LR_CHECK_LAUNCH();
  }
  for (int J = 0, b = 0; J < n; J += CH_NB, ++b) {
    const int jb = n - J < CH_NB ? n - J : CH_NB;
    double* Db = Dinv + (long long)b * CH_NB * CH_NB;
    chol_diag_kernel<<<1, CH_THREADS, kDiagSmem, s>>>(A, lda, J, jb, Db, info);
    LR_CHECK_LAUNCH();
    const int rest = n - J - jb;
    if (rest > 0) {
      // R[J, J+jb:] = inv(R_JJ)^T A[J, J+jb:]
      int st = lr_gemm_f64(1, jb, rest, jb, 1.0, Db, CH_NB, A + (long long)J * lda + J + jb, lda, 0.0,
                           T, rest, 0, nullptr, 0, stream);
      if (st) return st;
      st = lr_copy2d_f64(T, rest, A + (long long)J * lda + J + jb, lda, jb, rest, 0, stream);
      if (st) return st;
      // trailing: A[J+jb:, J+jb:] -= R_panel^T R_panel  (upper, exactly symmetric)
      const double* P = A + (long long)J * lda + J + jb;
      st = lr_gemm_f64(1, rest, rest, jb, -1.0, P, lda, P, lda, 1.0,
                       A + (long long)(J + jb) * lda + J + jb, lda, LR_GEMM_SYRK_UPPER, nullptr, 0,
                       stream);
      if (st) return st;
    }
  }
  zero_lower_kernel<<<(int)((1LL * n * n + 255) / 256 > 1184 ? 1184 : (1LL * n * n + 255) / 256), 256, 0,
                      s>>>(A, lda, n);
  LR_CHECK_LAUNCH();
  // R^{-1} by block back substitution: X[I,:] = inv(R_II) (E_I - R[I,>I] X[>I,:])
  if (Rinv) {
    for (long long b = nblk - 1; b >= 0; --b) {
      const int I = (int)b * CH_NB;
      const int ib = n - I < CH_NB ? n - I : CH_NB;
      const double* Db = Dinv + b * CH_NB * CH_NB;
      inv_place_diag_kernel<<<(ib * n + 255) / 256 > 1184 ? 1184 : (ib * n + 255) / 256, 256, 0, s>>>(
          Rinv, ldr, n, I, ib, Db);
      LR_CHECK_LAUNCH();
      const int rest = n - I - ib;
      if (rest > 0) {
        // T = R[I, I+ib:] * X[I+ib:, I+ib:]   (X upper)
        int st = lr_gemm_f64(0, ib, rest, rest, 1.0, A + (long long)I * lda + I + ib, lda,
                             Rinv + (long long)(I + ib) * ldr + I + ib, ldr, 0.0, T, rest,
                             LR_GEMM_B_UPPER, nullptr, 0, stream);
        if (st) return st;
        // X[I, I+ib:] = -inv(R_II) T
        st = lr_gemm_f64(0, ib, rest, ib, -1.0, Db, CH_NB, T, rest, 0.0,
                         Rinv + (long long)I * ldr + I + ib, ldr, 0, nullptr, 0, stream);
        if (st) return st;
      }
    }
  }
  if (info_host) {
    LR_CHECK_CUDA(cudaMemcpyAsync(info_host, info, sizeof(int), cudaMemcpyDeviceToHost, s));
    LR_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  return LR_OK;
}

}  // extern "C"
