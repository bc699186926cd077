// Symmetric eigendecomposition by parallel Jacobi, the GPU replacement for
// LAPACK dsyevd behind `sym_eig` (linalg.py:153-169; survey K5).
//
//   n <= kSmallN : one CTA, matrix and eigenvectors in shared memory, cyclic
//                  round-robin (circle-method) ordering, all n/2 rotations of
//                  a round applied at once as independent 2x2 blocks.
//   n >  kSmallN : two-level block Jacobi, blocks of kB = 16 indices.  Each
//                  round pairs the 2P blocks; one CTA per pair diagonalizes
//                  its 32x32 subproblem in shared memory (the same in-smem
//                  solver), then every 32x32 tile of A is rotated on both
//                  sides and V on the right by the pair rotations (DMMA-free
//                  small products in shared memory).
// Rotation test (relative accuracy, Demmel-Veselic): rotate (p,q) iff
// |a_pq| > tol * sqrt(|a_pp a_qq|); a sweep with no rotation ends the
// iteration.  Eigenvalues come out ascending with their vectors reordered.
// Latency-bound: reported as time and share of the step.
#include "lr_common.cuh"

namespace lr {

constexpr int kSmallN = 96;
constexpr int kSmallThreads = 512;
constexpr int kB = 32;        // block size of the two-level scheme
constexpr int kSub = 2 * kB;  // subproblem size
constexpr int kSubThreads = 512;
constexpr int kInnerSweeps = 1;
constexpr double kJacobiTol = 1e-15;
// rotations below this fraction of max|a_ii| are rounding noise: skipping them
// keeps singular (rank-deficient) Grams from rotating forever; it perturbs
// eigenvalues by O(1e-34) relative to the largest.
constexpr double kNoiseFloor = 4e-16;
constexpr int kPairSmem = 2 * kSub * (kSub + 1) * (int)sizeof(double);
constexpr int kApplySmem = 3 * kSub * (kSub + 1) * (int)sizeof(double);

// circle-method pairing: players 0..N-1 (N even), round r in [0, N-1)
__device__ __forceinline__ void circle_pair(int N, int r, int k, int& p, int& q) {
  if (k == 0) {
    p = N - 1;
    q = r;
  } else {
    p = (r + k) % (N - 1);
    q = (r - k + (N - 1)) % (N - 1);
  }
  if (p > q) {
    int t = p;
    p = q;
    q = t;
  }
}

// One CTA runs cyclic parallel Jacobi on a (n x n, ld lda) in shared memory,
// accumulating rotations into v (n x n, ld ldv, shared or global).
// rot: shared scratch of >= 2*(N/2) doubles, idx: >= N ints, flag: shared int.
// Returns sweeps performed (> max_sweeps means not converged); *any_rot tells
// whether the first sweep rotated anything.
__device__ int jacobi_block_solve(double* a, int lda, double* v, int ldv, int n, int max_sweeps,
                                  double tol, double floor, double* rot, int* idx, int* flag, int* any_rot) {
  const int N = (n + 1) & ~1;
  const int half = N / 2;
  const int tid = threadIdx.x, nt = blockDim.x;
  int sweep = 0;
  *any_rot = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < N - 1; ++r) {
      for (int k = tid; k < half; k += nt) {
        int p, q;
        circle_pair(N, r, k, p, q);
        idx[2 * k] = p;
        idx[2 * k + 1] = q;
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double app = a[p * lda + p], aqq = a[q * lda + q], apq = a[p * lda + q];
          if (fabs(apq) > floor && fabs(apq) > tol * sqrt(fabs(app) * fabs(aqq))) {
            const double tau = (aqq - app) / (2.0 * apq);
            const double t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            *flag = 1;
          }
        }
        rot[2 * k] = c;
        rot[2 * k + 1] = s;
      }
      __syncthreads();
      // A <- J^T A J on disjoint 2x2 blocks (k1 rows, k2 cols)
      for (int e = tid; e < half * half; e += nt) {
        const int k1 = e / half, k2 = e - k1 * half;
        const int p1 = idx[2 * k1], q1 = idx[2 * k1 + 1];
        const int p2 = idx[2 * k2], q2 = idx[2 * k2 + 1];
        const double c1 = rot[2 * k1], s1 = rot[2 * k1 + 1];
        const double c2 = rot[2 * k2], s2 = rot[2 * k2 + 1];
        if (s1 == 0.0 && s2 == 0.0) continue;
        const bool vq1 = q1 < n, vq2 = q2 < n;
        if (k1 == k2) {
          // the rotated pair itself: closed form, off-diagonal exactly zero
          const double app = a[p1 * lda + p1], aqq = a[q1 * lda + q1], apq = a[p1 * lda + q1];
          const double t = s1 / c1;
          a[p1 * lda + p1] = app - t * apq;
          a[q1 * lda + q1] = aqq + t * apq;
          a[p1 * lda + q1] = 0.0;
          a[q1 * lda + p1] = 0.0;
          continue;
        }
        const double a11 = a[p1 * lda + p2];
        const double a12 = vq2 ? a[p1 * lda + q2] : 0.0;
        const double a21 = vq1 ? a[q1 * lda + p2] : 0.0;
        const double a22 = (vq1 && vq2) ? a[q1 * lda + q2] : 0.0;
        const double m11 = c2 * a11 - s2 * a12, m12 = s2 * a11 + c2 * a12;
        const double m21 = c2 * a21 - s2 * a22, m22 = s2 * a21 + c2 * a22;
        a[p1 * lda + p2] = c1 * m11 - s1 * m21;
        if (vq2) a[p1 * lda + q2] = c1 * m12 - s1 * m22;
        if (vq1) a[q1 * lda + p2] = s1 * m11 + c1 * m21;
        if (vq1 && vq2) a[q1 * lda + q2] = s1 * m12 + c1 * m22;
      }
      // V <- V J
      for (int e = tid; e < n * half; e += nt) {
        const int i = e / half, k = e - i * half;
        const double s = rot[2 * k + 1];
        if (s == 0.0) continue;
        const double c = rot[2 * k];
        const int p = idx[2 * k], q = idx[2 * k + 1];
        const double vp = v[i * ldv + p], vq = v[i * ldv + q];
        v[i * ldv + p] = c * vp - s * vq;
        v[i * ldv + q] = s * vp + c * vq;
      }
      __syncthreads();
    }
    const int rotated = *flag;
    if (sweep == 0) *any_rot = rotated;
    __syncthreads();
    if (!rotated) break;
  }
  return sweep + 1;
}

// ------------------------------------------------------------ small path
__global__ void __launch_bounds__(kSmallThreads) jacobi_small_kernel(const double* __restrict__ A, long long lda,
                                                                   int n, double* d_unsorted, double* Vout,
                                                                   long long ldv, int max_sweeps, int* sweeps_out) {
  extern __shared__ double sm[];
  const int LD = n + 1;
  double* a = sm;
  double* v = a + n * LD;
  double* rot = v + n * LD;
  int* idx = reinterpret_cast<int*>(rot + n + 2);
  __shared__ int flag, any;
  const int tid = threadIdx.x;
  for (int e = tid; e < n * n; e += blockDim.x) {
    int i = e / n, c = e - i * n;
    a[i * LD + c] = A[(long long)i * lda + c];
    v[i * LD + c] = (i == c) ? 1.0 : 0.0;
  }
  __shared__ double red[32];
  double dm = 0.0;
  for (int i = tid; i < n; i += blockDim.x) dm = fmax(dm, fabs(a[i * LD + i]));
  dm = block_max<kSmallThreads>(dm, red);
  __shared__ double floor_sh;
  if (tid == 0) floor_sh = kNoiseFloor * dm;
  __syncthreads();
  int sw = jacobi_block_solve(a, LD, v, LD, n, max_sweeps, kJacobiTol, floor_sh, rot, idx, &flag, &any);
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {
    int i = e / n, c = e - i * n;
    Vout[(long long)i * ldv + c] = v[i * LD + c];
  }
  for (int i = tid; i < n; i += blockDim.x) d_unsorted[i] = a[i * LD + i];
  if (tid == 0) *sweeps_out = (flag == 0) ? sw : max_sweeps + 1;
}

// ---------------------------------------------------------- block path
// pair k of round r -> blocks (bI, bJ); gather the 2kB x 2kB subproblem, run
// `inner_sweeps` cyclic sweeps on it, write its rotation Z for the apply
// kernel.  floor_ptr: absolute rotation floor (noise level of the input).
__global__ void __launch_bounds__(kSubThreads) jacobi_pair_solve_kernel(const double* __restrict__ Aw, int N,
                                                                      int nblk, int round, double* Z,
                                                                      int* sweep_flag, int inner_sweeps,
                                                                      const double* floor_ptr) {
  extern __shared__ double ps_smem[];
  double* a = ps_smem;
  double* z = a + kSub * (kSub + 1);
  __shared__ double rot[kSub + 2];
  __shared__ int idx[kSub + 2];
  __shared__ int flag, any;
  const int k = blockIdx.x;
  int bI, bJ;
  circle_pair(nblk, round, k, bI, bJ);
  const int tid = threadIdx.x;
  for (int e = tid; e < kSub * kSub; e += blockDim.x) {
    const int i = e / kSub, c = e - i * kSub;
    const int gi = (i < kB) ? bI * kB + i : bJ * kB + (i - kB);
    const int gc = (c < kB) ? bI * kB + c : bJ * kB + (c - kB);
    a[i * (kSub + 1) + c] = Aw[(long long)gi * N + gc];
    z[i * (kSub + 1) + c] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  jacobi_block_solve(a, kSub + 1, z, kSub + 1, kSub, inner_sweeps, kJacobiTol, *floor_ptr, rot, idx, &flag, &any);
  __syncthreads();
  for (int e = tid; e < kSub * kSub; e += blockDim.x) {
    const int i = e / kSub, c = e - i * kSub;
    Z[(long long)k * kSub * kSub + e] = z[i * (kSub + 1) + c];
  }
  if (tid == 0 && any) atomicOr(sweep_flag, 1);
}

// blocks [0, P*P): tile (k1, k2) of A <- Z1^T A Z2;
// blocks [P*P, P*P + P*ceil(N/kSub)): V[row chunk, cols of pair k] <- V Z_k
__global__ void __launch_bounds__(256) jacobi_apply_kernel(double* Aw, double* Vw, int N, int nblk, int round,
                                                         const double* __restrict__ Z) {
  extern __shared__ double ap_smem[];
  constexpr int L = kSub + 1;
  double* t = ap_smem;
  double* u = t + kSub * L;
  double* z = u + kSub * L;
  const int P = nblk / 2;
  const int tid = threadIdx.x;
  int b = blockIdx.x;
  if (b < P * P) {
    const int k1 = b / P, k2 = b - (b / P) * P;
    int b1I, b1J, b2I, b2J;
    circle_pair(nblk, round, k1, b1I, b1J);
    circle_pair(nblk, round, k2, b2I, b2J);
    for (int e = tid; e < kSub * kSub; e += blockDim.x) {
      const int i = e / kSub, c = e - i * kSub;
      const int gi = (i < kB) ? b1I * kB + i : b1J * kB + (i - kB);
      const int gc = (c < kB) ? b2I * kB + c : b2J * kB + (c - kB);
      t[i * L + c] = Aw[(long long)gi * N + gc];
      z[i * L + c] = Z[(long long)k2 * kSub * kSub + e];
    }
    __syncthreads();
    for (int e = tid; e < kSub * kSub; e += blockDim.x) {  // u = t z2
      const int i = e / kSub, c = e - i * kSub;
      double s = 0.0;
#pragma unroll 8
      for (int q = 0; q < kSub; ++q) s = fma(t[i * L + q], z[q * L + c], s);
      u[i * L + c] = s;
    }
    __syncthreads();
    for (int e = tid; e < kSub * kSub; e += blockDim.x) z[(e / kSub) * L + e % kSub] = Z[(long long)k1 * kSub * kSub + e];
    __syncthreads();
    for (int e = tid; e < kSub * kSub; e += blockDim.x) {  // out = z1^T u
      const int i = e / kSub, c = e - i * kSub;
      double s = 0.0;
#pragma unroll 8
      for (int q = 0; q < kSub; ++q) s = fma(z[q * L + i], u[q * L + c], s);
      const int gi = (i < kB) ? b1I * kB + i : b1J * kB + (i - kB);
      const int gc = (c < kB) ? b2I * kB + c : b2J * kB + (c - kB);
      Aw[(long long)gi * N + gc] = s;
    }
    return;
  }
  b -= P * P;
  const int chunks = (N + kSub - 1) / kSub;
  const int k = b / chunks, r0 = (b - k * chunks) * kSub;
  int bI, bJ;
  circle_pair(nblk, round, k, bI, bJ);
  for (int e = tid; e < kSub * kSub; e += blockDim.x) {
    const int i = e / kSub, c = e - i * kSub;
    const int gc = (c < kB) ? bI * kB + c : bJ * kB + (c - kB);
    t[i * L + c] = (r0 + i < N) ? Vw[(long long)(r0 + i) * N + gc] : 0.0;
    z[i * L + c] = Z[(long long)k * kSub * kSub + e];
  }
  __syncthreads();
  for (int e = tid; e < kSub * kSub; e += blockDim.x) {
    const int i = e / kSub, c = e - i * kSub;
    if (r0 + i >= N) continue;
    double s = 0.0;
#pragma unroll 8
    for (int q = 0; q < kSub; ++q) s = fma(t[i * L + q], z[q * L + c], s);
    const int gc = (c < kB) ? bI * kB + c : bJ * kB + (c - kB);
    Vw[(long long)(r0 + i) * N + gc] = s;
  }
}

// floor = kNoiseFloor * max_i |A_ii| (one block)
__global__ void diag_floor_kernel(const double* A, long long lda, int n, double* floor_out) {
  __shared__ double sh[32];
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(A[(long long)i * lda + i]));
  m = block_max<256>(m, sh);
  if (threadIdx.x == 0) *floor_out = kNoiseFloor * m;
}

__global__ void pad_copy_kernel(const double* __restrict__ A, long long lda, int n, double* Aw, double* Vw,
                                int N) {
  const long long total = (long long)N * N;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / N), c = (int)(t - (long long)i * N);
    Aw[t] = (i < n && c < n) ? A[(long long)i * lda + c] : 0.0;
    Vw[t] = (i == c) ? 1.0 : 0.0;
  }
}

__global__ void diag_extract_kernel(const double* Aw, int N, int n, double* d) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    d[i] = Aw[(long long)i * N + i];
}

// ascending order, ties by index: rank_i = #{d_j < d_i} + #{j < i, d_j == d_i}
__global__ void rank_kernel(const double* d, int n, int* rank) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double di = d[i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const double dj = d[j];
      r += (dj < di) || (dj == di && j < i);
    }
    rank[i] = r;
  }
}

__global__ void permute_out_kernel(const double* d_in, const double* Vin, long long ldvin, int n, const int* rank,
                                   double* d_out, double* Vout, long long ldv) {
  const long long total = (long long)n * n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / n), c = (int)(t - (long long)i * n);
    Vout[(long long)i * ldv + rank[c]] = Vin[(long long)i * ldvin + c];
    if (i == 0) d_out[rank[c]] = d_in[c];
  }
}

static int small_smem(int n) { return (n * (n + 1) * 2 + n + 2) * 8 + (n + 2) * 4 + 64; }

}  // namespace lr

using namespace lr;

extern "C" {

long long lr_syevj_workspace_doubles(int n) {
  if (n <= kSmallN) return (long long)n * n + 2 * n + 64;
  const int nblk0 = (n + kB - 1) / kB;
  const int nblk = (nblk0 + 1) & ~1;
  const long long N = (long long)nblk * kB;
  return 2 * N * N + (long long)(nblk / 2) * kSub * kSub + 2 * n + 66;
}

int lr_syevj_f64(int n, double* A, long long lda, double* d, double* V, long long ldv, int max_sweeps,
                 double* work, int* sweeps_host, void* stream) {
  LR_REQUIRE(n >= 1 && lda >= n && ldv >= n, "syevj: bad shape");
  cudaStream_t s = as_stream(stream);
  if (max_sweeps <= 0) max_sweeps = 40;
  int sweeps = 0;
  if (n <= kSmallN) {
    double* Vtmp = work;
    double* dun = Vtmp + (long long)n * n;
    int* rank = reinterpret_cast<int*>(dun + n);
    int* dsw = rank + n;
    const int smem = small_smem(n);
    static bool attr = false;
    if (!attr) {
      LR_CHECK_CUDA(cudaFuncSetAttribute(jacobi_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         small_smem(kSmallN)));
      attr = true;
    }
    jacobi_small_kernel<<<1, kSmallThreads, smem, s>>>(A, lda, n, dun, Vtmp, n, max_sweeps, dsw);
    LR_CHECK_LAUNCH();
    rank_kernel<<<(n + 127) / 128, 128, 0, s>>>(dun, n, rank);
    LR_CHECK_LAUNCH();
    permute_out_kernel<<<((long long)n * n + 255) / 256, 256, 0, s>>>(dun, Vtmp, n, n, rank, d, V, ldv);
    LR_CHECK_LAUNCH();
    LR_CHECK_CUDA(cudaMemcpyAsync(&sweeps, dsw, sizeof(int), cudaMemcpyDeviceToHost, s));
    LR_CHECK_CUDA(cudaStreamSynchronize(s));
  } else {
    const int nblk0 = (n + kB - 1) / kB;
    const int nblk = (nblk0 + 1) & ~1;
    const int P = nblk / 2;
    const int N = nblk * kB;
    double* Aw = work;
    double* Vw = Aw + (long long)N * N;
    double* Z = Vw + (long long)N * N;
    double* dun = Z + (long long)P * kSub * kSub;
    double* floor_d = dun + n;
    int* rank = reinterpret_cast<int*>(floor_d + 2);
    int* flag = rank + n;
    static bool battr = false;
    if (!battr) {
      LR_CHECK_CUDA(cudaFuncSetAttribute(jacobi_pair_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmem));
      LR_CHECK_CUDA(cudaFuncSetAttribute(jacobi_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kApplySmem));
      battr = true;
    }
    long long tot = (long long)N * N;
    pad_copy_kernel<<<(int)((tot + 255) / 256 > 2048 ? 2048 : (tot + 255) / 256), 256, 0, s>>>(A, lda, n, Aw, Vw, N);
    LR_CHECK_LAUNCH();
    diag_floor_kernel<<<1, 256, 0, s>>>(A, lda, n, floor_d);
    LR_CHECK_LAUNCH();
    const int apply_blocks = P * P + P * ((N + kSub - 1) / kSub);
    int host_flag = 1;
    for (sweeps = 1; sweeps <= max_sweeps; ++sweeps) {
      LR_CHECK_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
      for (int r = 0; r < nblk - 1; ++r) {
        jacobi_pair_solve_kernel<<<P, kSubThreads, kPairSmem, s>>>(Aw, N, nblk, r, Z, flag, kInnerSweeps, floor_d);
        jacobi_apply_kernel<<<apply_blocks, 256, kApplySmem, s>>>(Aw, Vw, N, nblk, r, Z);
      }
      LR_CHECK_LAUNCH_N(2LL * (nblk - 1));
      LR_CHECK_CUDA(cudaMemcpyAsync(&host_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
      LR_CHECK_CUDA(cudaStreamSynchronize(s));
      if (!host_flag) break;
    }
    diag_extract_kernel<<<(n + 255) / 256, 256, 0, s>>>(Aw, N, n, dun);
    rank_kernel<<<(n + 127) / 128, 128, 0, s>>>(dun, n, rank);
    permute_out_kernel<<<(int)(((long long)n * n + 255) / 256 > 4096 ? 4096 : ((long long)n * n + 255) / 256), 256,
                         0, s>>>(dun, Vw, N, n, rank, d, V, ldv);
    LR_CHECK_LAUNCH_N(3);
  }
  if (sweeps_host) *sweeps_host = sweeps;
  if (sweeps > max_sweeps) {
    set_error("symmetric eigensolver did not converge in %d Jacobi sweeps", max_sweeps);
    return LR_ERR_NOCONV;
  }
  return LR_OK;
}

}  // extern "C"
