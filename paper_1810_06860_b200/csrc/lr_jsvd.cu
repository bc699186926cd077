// One-sided (Hestenes) Jacobi sweeps for the dense SVD fallback
// (oracle_svd, /root/reference/pkg/src/lowrank/linalg.py:205-221 -> LAPACK
// dgesdd).  The Gram route alone resolves small singular values only to
// ~sqrt(eps) * s_max; the host preconditions with it (B = A V, columns
// already nearly orthogonal) and these sweeps finish the job: column pairs
// (p, q) are rotated until every pair is orthogonal to tol * |b_p| |b_q|, so
// the column norms are the singular values to ~eps * s_max (absolute, like
// dgesdd) and the rotations accumulate into V.
//
// Layout: the columns of B are the ROWS of Bt (n x m, row-major) and the
// columns of V the rows of Vt (n x n): every pair operation streams two
// contiguous rows.  One launch per round-robin step (circle method over
// N = n rounded up to even; the odd player sits out), one CTA per pair with a
// fixed-order block reduction: deterministic.
#include "lr_common.cuh"

namespace lr {

constexpr int kJsThreads = 256;

__device__ __forceinline__ void pair_of(int k, int s, int N, int& p, int& q) {
  // circle method: player N-1 fixed, the rest rotate by s
  if (k == 0) {
    p = N - 1;
    q = s;
  } else {
    p = (s + k) % (N - 1);
    q = (s - k + (N - 1)) % (N - 1);
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

__global__ void __launch_bounds__(kJsThreads) jacobi_pair_kernel(double* __restrict__ Bt, long long ldb, int m,
                                                                  double* __restrict__ Vt, long long ldv, int n,
                                                                  int N, int s, double tol, double noise2,
                                                                  unsigned long long* __restrict__ off) {
  int p, q;
  pair_of(blockIdx.x, s, N, p, q);
  if (q >= n) return;
  __shared__ double red[32];
  __shared__ double rot[2];
  double* bp = Bt + (long long)p * ldb;
  double* bq = Bt + (long long)q * ldb;
  double a = 0.0, b = 0.0, g = 0.0;
  for (int i = threadIdx.x; i < m; i += kJsThreads) {
    const double x = bp[i], y = bq[i];
    a = fma(x, x, a);
    b = fma(y, y, b);
    g = fma(x, y, g);
  }
  a = block_sum<kJsThreads>(a, red);
  b = block_sum<kJsThreads>(b, red);
  g = block_sum<kJsThreads>(g, red);
  if (threadIdx.x == 0) {
    double c = 1.0, sn = 0.0;
    const double den = sqrt(a) * sqrt(b);
    // two noise-level columns (squared norms below noise2) are not rotated:
    // their mutual angle is rounding noise and need not converge
    const double meas = (den > 0.0 && !(a < noise2 && b < noise2)) ? fabs(g) / den : 0.0;
    if (meas > tol) {
      // rotate so that the new columns are orthogonal (Rutishauser's formulas)
      const double zeta = (b - a) / (2.0 * g);
      const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
      c = 1.0 / sqrt(1.0 + t * t);
      sn = c * t;
      atomicMax(off, (unsigned long long)__double_as_longlong(meas));  // meas >= 0: bit order = value order
    }
    rot[0] = c;
    rot[1] = sn;
  }
  __syncthreads();
  const double c = rot[0], sn = rot[1];
  if (sn == 0.0) return;
  for (int i = threadIdx.x; i < m; i += kJsThreads) {
    const double x = bp[i], y = bq[i];
    bp[i] = c * x - sn * y;
    bq[i] = sn * x + c * y;
  }
  double* vp = Vt + (long long)p * ldv;
  double* vq = Vt + (long long)q * ldv;
  for (int i = threadIdx.x; i < n; i += kJsThreads) {
    const double x = vp[i], y = vq[i];
    vp[i] = c * x - sn * y;
    vq[i] = sn * x + c * y;
  }
}

__global__ void __launch_bounds__(kJsThreads) row_norms_kernel(const double* __restrict__ Bt, long long ldb, int m,
                                                               double* __restrict__ out) {
  __shared__ double red[32];
  const double* b = Bt + (long long)blockIdx.x * ldb;
  // scaled two-pass norm: no overflow / underflow for any finite row
  double mx = 0.0;
  for (int i = threadIdx.x; i < m; i += kJsThreads) mx = fmax(mx, fabs(b[i]));
  mx = block_max<kJsThreads>(mx, red);  // valid in thread 0: broadcast
  __shared__ double bc;
  if (threadIdx.x == 0) bc = mx;
  __syncthreads();
  mx = bc;
  double ss = 0.0;
  if (mx > 0.0) {
    const double inv = 1.0 / mx;
    for (int i = threadIdx.x; i < m; i += kJsThreads) {
      const double x = b[i] * inv;
      ss = fma(x, x, ss);
    }
  }
  ss = block_sum<kJsThreads>(ss, red);
  if (threadIdx.x == 0) out[blockIdx.x] = (mx > 0.0) ? mx * sqrt(ss) : 0.0;
}

}  // namespace lr

using namespace lr;

extern "C" {

int lr_jacobi_sweep_f64(int n, int m, double* Bt, long long ldb, double* Vt, long long ldv, double tol,
                        double noise2, double* off, void* stream) {
  LR_REQUIRE(n >= 1 && m >= 1 && ldb >= m && ldv >= n, "jacobi_sweep: bad dims (n=%d m=%d)", n, m);
  cudaStream_t s = as_stream(stream);
  LR_CHECK_CUDA(cudaMemsetAsync(off, 0, sizeof(double), s));
  if (n == 1) return LR_OK;
  const int N = n + (n & 1);
  for (int step = 0; step < N - 1; ++step) {
    jacobi_pair_kernel<<<N / 2, kJsThreads, 0, s>>>(Bt, ldb, m, Vt, ldv, n, N, step, tol, noise2,
                                                    reinterpret_cast<unsigned long long*>(off));
    LR_CHECK_LAUNCH();
  }
  return LR_OK;
}

int lr_row_norms_f64(const double* Bt, long long ldb, int n, int m, double* out, void* stream) {
  LR_REQUIRE(n >= 0 && m >= 1 && ldb >= m, "row_norms: bad dims (n=%d m=%d)", n, m);
  if (n == 0) return LR_OK;
  row_norms_kernel<<<n, kJsThreads, 0, as_stream(stream)>>>(Bt, ldb, m, out);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

}  // extern "C"
