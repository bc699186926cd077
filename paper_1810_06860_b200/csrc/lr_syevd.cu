// Symmetric eigendecomposition by Householder tridiagonalization, bisection
// and inverse iteration -- the default replacement for LAPACK dsyevd behind
// `sym_eig` / `eig_svd` (linalg.py:153-202; survey K5).
//
//   1. tridiag   : one cooperative kernel; the n x n matrix is row-distributed
//                  over the CTAs' shared memory.  Per column: the owner of row
//                  j builds the reflector (dlarfg convention), one grid barrier
//                  publishes v, every CTA forms its slice of p = tau*A*v, a
//                  second barrier publishes p, every CTA applies the rank-2
//                  update A -= v w^T + w v^T to its rows (w = p - tau/2 (p.v) v).
//   2. bisection : one warp per eigenvalue, 32-way multisection on Sturm counts
//                  (eigenvalue i is the i-th smallest: the output is ascending).
//   3. inverse iteration : one thread per eigenvalue, tridiagonal LU with
//                  partial pivoting (coalesced [row][eigenvalue] scratch).
//   4. clusters  : eigenvalues closer than 1e-8*||T|| are re-orthonormalised
//                  (modified Gram-Schmidt, twice) by one CTA per cluster.
//   5. back-transform : one warp per eigenvector applies H_{n-3} ... H_0.
// Accuracy is LAPACK's: eigenvalues to O(eps*||A||) absolute, eigenvectors to
// O(eps*||A||/gap).  Latency-bound (2 grid barriers per column): reported as
// time and share of the step.
#include <cooperative_groups.h>
#include <cstdlib>

#include "lr_common.cuh"

namespace cg = cooperative_groups;

namespace lr {

constexpr int TD_THREADS = 256;

struct TdParams {
  const double* A;
  long long lda;
  int n, rows_per;
  double* d;     // n
  double* e;     // n (e[i] couples i, i+1)
  double* tau;   // n
  double* Vr;    // n x n: row j holds reflector j at columns j+1..n-1 (v[j+1] = 1)
  double* vbuf;  // 2 x n
  double* pbuf;  // 2 x n
  double* rows_global;  // n x (n+1) working rows when they do not fit shared memory, else null
};

__device__ __forceinline__ void td_barrier(cg::grid_group& grid) {
  if (gridDim.x == 1)
    __syncthreads();
  else
    grid.sync();
}

__global__ void __launch_bounds__(TD_THREADS) tridiag_kernel(TdParams P) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double td_smem[];
  const int n = P.n, tid = threadIdx.x;
  const int r0 = blockIdx.x * P.rows_per;
  const int r1 = min(n, r0 + P.rows_per);
  const int nr = max(0, r1 - r0);
  const int LD = n + 1;
  // my rows: shared memory when they fit, else a global (L2-resident) slab
  double* R = P.rows_global ? P.rows_global + (size_t)r0 * LD : td_smem;
  double* v = P.rows_global ? td_smem : td_smem + (size_t)P.rows_per * LD;  // n
  double* p = v + n;                                                       // n
  __shared__ double red[32];
  __shared__ double sh_tau, sh_k;

  for (int e = tid; e < nr * n; e += TD_THREADS) {
    const int i = e / n, c = e - (e / n) * n;
    R[i * LD + c] = P.A[(long long)(r0 + i) * P.lda + c];
  }
  __syncthreads();

  for (int j = 0; j + 2 < n; ++j) {
    const int par = j & 1;
    double* vg = P.vbuf + par * n;
    double* pg = P.pbuf + par * n;
    const int L = n - j - 1;  // trailing indices j+1 .. n-1
    if (j >= r0 && j < r1) {
      // owner: Householder reflector from x = A[j][j+1:]  (dlarfg)
      const double* row = R + (j - r0) * LD;
      double ss = 0.0;
      for (int c = j + 2 + tid; c < n; c += TD_THREADS) ss = fma(row[c], row[c], ss);
      ss = block_sum<TD_THREADS>(ss, red);
      if (tid == 0) {
        const double alpha = row[j + 1];
        double tau = 0.0, beta = alpha, scal = 0.0;
        if (ss != 0.0) {
          const double nrm = sqrt(alpha * alpha + ss);
          beta = (alpha >= 0.0) ? -nrm : nrm;
          tau = (beta - alpha) / beta;
          scal = 1.0 / (alpha - beta);
        }
        P.d[j] = row[j];
        P.e[j] = beta;
        P.tau[j] = tau;
        sh_tau = scal;  // temporarily the v scale
        sh_k = tau;
      }
      __syncthreads();
      const double scal = sh_tau;
      const double tau = sh_k;
      for (int c = j + 1 + tid; c < n; c += TD_THREADS) {
        const double vc = (c == j + 1) ? 1.0 : (tau == 0.0 ? 0.0 : row[c] * scal);
        vg[c] = vc;
        P.Vr[(long long)j * n + c] = vc;
      }
    }
    td_barrier(grid);
    const double tau = P.tau[j];
    for (int c = j + 1 + tid; c < n; c += TD_THREADS) v[c] = vg[c];
    __syncthreads();
    if (tau != 0.0) {
      // p_r = tau * sum_c A[r][c] v[c] for my rows r >= j+1 (one warp per row)
      const int lane = tid & 31, w = tid >> 5;
      for (int i = w; i < nr; i += TD_THREADS / 32) {
        const int r = r0 + i;
        if (r <= j) continue;
        const double* row = R + i * LD;
        double s = 0.0;
        for (int c = j + 1 + lane; c < n; c += 32) s = fma(row[c], v[c], s);
        s = warp_sum(s);
        if (lane == 0) pg[r] = tau * s;
      }
    }
    td_barrier(grid);
    if (tau != 0.0) {
      for (int c = j + 1 + tid; c < n; c += TD_THREADS) p[c] = pg[c];
      __syncthreads();
      double pv = 0.0;
      for (int c = j + 1 + tid; c < n; c += TD_THREADS) pv = fma(p[c], v[c], pv);
      pv = block_sum<TD_THREADS>(pv, red);
      if (tid == 0) sh_k = 0.5 * tau * pv;
      __syncthreads();
      const double K = sh_k;
      for (int c = j + 1 + tid; c < n; c += TD_THREADS) p[c] = p[c] - K * v[c];  // w
      __syncthreads();
      for (int e = tid; e < nr * L; e += TD_THREADS) {
        const int i = e / L, c = j + 1 + (e - (e / L) * L);
        const int r = r0 + i;
        if (r <= j) continue;
        // symmetric in (r, c): products are exact-commutative, sum order fixed
        const double upd = __dadd_rn(__dmul_rn(v[r], p[c]), __dmul_rn(p[r], v[c]));
        R[i * LD + c] -= upd;
      }
    }
    __syncthreads();
  }
  // last 2x2 block
  for (int r = r0; r < r1; ++r) {
    if (tid != 0) break;
    if (r == n - 2) {
      P.d[n - 2] = R[(r - r0) * LD + n - 2];
      P.e[n - 2] = R[(r - r0) * LD + n - 1];
    }
    if (r == n - 1) P.d[n - 1] = R[(r - r0) * LD + n - 1];
    if (n == 1 && r == 0) P.d[0] = R[0];
  }
}

// Sturm count: number of eigenvalues of T strictly below x
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                           double x, double pivmin) {
  int cnt = 0;
  double q = d[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

__global__ void tri_prep_kernel(const double* d, const double* e, int n, double* e2, double* bounds) {
  // bounds = {lo, hi, pivmin, tnorm}; one block
  __shared__ double red[32];
  double lo = 1e308, hi = -1e308, emax = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double el = i > 0 ? fabs(e[i - 1]) : 0.0;
    const double er = i + 1 < n ? fabs(e[i]) : 0.0;
    lo = fmin(lo, d[i] - el - er);
    hi = fmax(hi, d[i] + el + er);
    if (i + 1 < n) {
      e2[i] = e[i] * e[i];
      emax = fmax(emax, e2[i]);
    }
  }
  lo = -block_max<256>(-lo, red);
  hi = block_max<256>(hi, red);
  emax = block_max<256>(emax, red);
  if (threadIdx.x == 0) {
    const double tnorm = fmax(fabs(lo), fabs(hi));
    const double pad = 2.0 * 2.220446049250313e-16 * tnorm * n + 1e-300;
    bounds[0] = lo - pad;
    bounds[1] = hi + pad;
    bounds[2] = 2.2250738585072014e-308 * fmax(1.0, emax) * 4.0;
    bounds[3] = tnorm;
  }
}

// one warp per eigenvalue index k (k-th smallest)
__global__ void bisect_kernel(const double* __restrict__ d, const double* __restrict__ e2, int n,
                              const double* __restrict__ bounds, double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= n) return;
  double lo = bounds[0], hi = bounds[1];
  const double pivmin = bounds[2];
  // absolute floor: the reduction already perturbs eigenvalues by O(eps*||T||)
  const double abs_floor = 1e-3 * 2.220446049250313e-16 * bounds[3];
  for (int it = 0; it < 40; ++it) {
    const double width = hi - lo;
    if (width <= 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi)) * 2.0 || width <= pivmin ||
        width <= abs_floor)
      break;
    const double x = lo + width * (double)(lane + 1) / 33.0;
    const int c = sturm_count(d, e2, n, x, pivmin);
    // largest x with count <= k is the new lo, smallest with count > k the new hi
    const unsigned le = __ballot_sync(0xffffffffu, c <= k);
    double nlo = lo, nhi = hi;
    if (le) {
      const int l = 31 - __clz(le);  // counts are monotone in lane: highest lane with c <= k
      nlo = __shfl_sync(0xffffffffu, x, l);
    }
    const unsigned gt = ~le;
    if (gt) {
      const int l = __ffs(gt) - 1;
      nhi = __shfl_sync(0xffffffffu, x, l);
    }
    if (nlo == lo && nhi == hi) break;
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) w[k] = 0.5 * (lo + hi);
}

// inverse iteration, one thread per eigenvalue; scratch laid out [i * n + k]
// (coalesced across the warp).  Values that the recurrences carry stay in
// registers; only independent loads touch memory.
__global__ void inviter_kernel(const double* __restrict__ d, const double* __restrict__ e, int n,
                               const double* __restrict__ w, const double* __restrict__ bounds, double* __restrict__ Z,
                               double* __restrict__ U1, double* __restrict__ U2, double* __restrict__ Lm,
                               double* __restrict__ Dg, int* __restrict__ Pv) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double lam = w[k];
  const double tnorm = bounds[3];
  const double tiny = fmax(2.220446049250313e-16 * tnorm, 1e-300);
#define IX(i) ((long long)(i) * n + k)
  // LU with partial pivoting of T - lam I (dlagtf): U = diag Dg, super U1, 2nd super U2
  double a = d[0] - lam;
  double b = n > 1 ? e[0] : 0.0;
  for (int i = 0; i < n - 1; ++i) {
    const double c = e[i];
    const double a_next = d[i + 1] - lam;
    const double b_next = (i + 2 < n) ? e[i + 1] : 0.0;
    if (fabs(a) >= fabs(c)) {
      const double piv = (a == 0.0) ? tiny : a;
      const double l = c / piv;
      Dg[IX(i)] = piv;
      U1[IX(i)] = b;
      U2[IX(i)] = 0.0;
      Lm[IX(i)] = l;
      Pv[IX(i)] = 0;
      a = a_next - l * b;
      b = b_next;
    } else {
      const double l = a / c;
      Dg[IX(i)] = c;
      U1[IX(i)] = a_next;
      U2[IX(i)] = b_next;
      Lm[IX(i)] = l;
      Pv[IX(i)] = 1;
      a = b - l * a_next;
      b = -l * b_next;
    }
  }
  Dg[IX(n - 1)] = (a == 0.0) ? tiny : a;
  unsigned long long s = 0x9E3779B97F4A7C15ULL * (unsigned long long)(k + 1);
  double scale = 1.0;
  for (int it = 0; it < 3; ++it) {
    // forward: z <- L^{-1} P (scale * z); the start vector is generated in pass 0
    double zc;
    if (it == 0) {
      s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
      zc = (double)((s * 2685821657736338717ULL) >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    } else {
      zc = Z[IX(0)] * scale;
    }
#pragma unroll 4
    for (int i = 0; i < n - 1; ++i) {
      double zn;
      if (it == 0) {
        s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
        zn = (double)((s * 2685821657736338717ULL) >> 11) * (2.0 / 9007199254740992.0) - 1.0;
      } else {
        zn = Z[IX(i + 1)] * scale;
      }
      const double l = Lm[IX(i)];
      if (Pv[IX(i)]) {
        Z[IX(i)] = zn;
        zc = zc - l * zn;
      } else {
        Z[IX(i)] = zc;
        zc = zn - l * zc;
      }
    }
    Z[IX(n - 1)] = zc;
    // backward: U x = y, track max |x| for the next scale
    double x1 = 0.0, x2 = 0.0, mx = 0.0;
#pragma unroll 4
    for (int i = n - 1; i >= 0; --i) {
      double dg = Dg[IX(i)];
      if (fabs(dg) < tiny) dg = (dg < 0.0) ? -tiny : tiny;
      const double xi = (Z[IX(i)] - U1[IX(i)] * x1 - U2[IX(i)] * x2) / dg;
      Z[IX(i)] = xi;
      x2 = x1;
      x1 = xi;
      mx = fmax(mx, fabs(xi));
    }
    scale = (mx > 0.0) ? 1.0 / mx : 1.0;
  }
  double ss = 0.0;
#pragma unroll 4
  for (int i = 0; i < n; ++i) {
    const double z = Z[IX(i)] * scale;
    ss = fma(z, z, ss);
  }
  const double inv = scale / sqrt(ss);
#pragma unroll 4
  for (int i = 0; i < n; ++i) Z[IX(i)] *= inv;
#undef IX
}

// modified Gram-Schmidt (twice) over a cluster [k0, k1) of columns of Z (n x n row-major)
__global__ void __launch_bounds__(256) cluster_mgs_kernel(double* Z, int n, const int* clusters) {
  const int k0 = clusters[2 * blockIdx.x], k1 = clusters[2 * blockIdx.x + 1];
  __shared__ double red[32];
  __shared__ double coef;
  for (int pass = 0; pass < 2; ++pass) {
    for (int j = k0; j < k1; ++j) {
      for (int i = k0; i < j; ++i) {
        double s = 0.0;
        for (int r = threadIdx.x; r < n; r += blockDim.x) s = fma(Z[(long long)r * n + i], Z[(long long)r * n + j], s);
        s = block_sum<256>(s, red);
        if (threadIdx.x == 0) coef = s;
        __syncthreads();
        const double c = coef;
        for (int r = threadIdx.x; r < n; r += blockDim.x) Z[(long long)r * n + j] -= c * Z[(long long)r * n + i];
        __syncthreads();
      }
      double s = 0.0;
      for (int r = threadIdx.x; r < n; r += blockDim.x) s = fma(Z[(long long)r * n + j], Z[(long long)r * n + j], s);
      s = block_sum<256>(s, red);
      if (threadIdx.x == 0) coef = 1.0 / sqrt(s);
      __syncthreads();
      const double c = coef;
      for (int r = threadIdx.x; r < n; r += blockDim.x) Z[(long long)r * n + j] *= c;
      __syncthreads();
    }
  }
}

// V[:, k] = H_0 H_1 ... H_{n-3} Z[:, k]; one warp per column, column staged in smem
__global__ void __launch_bounds__(128) backtransform_kernel(const double* __restrict__ Z, const double* __restrict__ Vr,
                                                          const double* __restrict__ tau, int n, double* __restrict__ V,
                                                          long long ldv) {
  extern __shared__ double bt_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int k = blockIdx.x * (blockDim.x >> 5) + wib;
  if (k >= n) return;
  double* x = bt_smem + (size_t)wib * n;
  for (int i = lane; i < n; i += 32) x[i] = Z[(long long)i * n + k];
  __syncwarp();
  for (int j = n - 3; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    const double* v = Vr + (long long)j * n;
    double s = 0.0;
    for (int i = j + 1 + lane; i < n; i += 32) s = fma(v[i], x[i], s);
    s = warp_sum(s) * t;
    for (int i = j + 1 + lane; i < n; i += 32) x[i] = fma(-s, v[i], x[i]);
    __syncwarp();
  }
  for (int i = lane; i < n; i += 32) V[(long long)i * ldv + k] = x[i];
}

struct TdPlan {
  int G, rows_per;
  size_t smem;
  bool global_rows;
};

// one CTA per SM at most (cooperative residency); rows go to shared memory
// when they fit, otherwise to a global slab (n >~ 1300)
static TdPlan td_plan(int n) {
  TdPlan pl;
  const int sms = sm_count();
  int G = n <= 96 ? 1 : (n < sms ? n : sms);
  int rows_per = (n + G - 1) / G;
  G = (n + rows_per - 1) / rows_per;
  size_t smem = ((size_t)rows_per * (n + 1) + 2 * (size_t)n) * sizeof(double);
  pl.global_rows = smem > 200 * 1024;
  if (pl.global_rows) smem = 2 * (size_t)n * sizeof(double);
  pl.G = G;
  pl.rows_per = rows_per;
  pl.smem = smem;
  return pl;
}

}  // namespace lr

using namespace lr;

extern "C" {

long long lr_syevd_workspace_doubles(int n) {
  const long long N = n;
  // d, e, tau, e2, w, bounds | Vr | vbuf, pbuf | Z, U1, U2, Lm, Dg | Pv (ints) | clusters | global rows
  return 6 * N + 8 + N * N + 4 * N + 5 * N * N + N * N / 2 + N + N + 64 + N * (N + 1);
}

int lr_syevd_f64(int n, const double* A, long long lda, double* d_out, double* V, long long ldv, double* work,
                 int* clusters_host, void* stream) {
  LR_REQUIRE(n >= 1 && lda >= n && ldv >= n, "syevd: bad shape");
  cudaStream_t s = as_stream(stream);
  const long long N = n;
  double* d = work;
  double* e = d + N;
  double* tau = e + N;
  double* e2 = tau + N;
  double* w = e2 + N;
  double* bounds = w + N;
  double* Vr = bounds + 8;
  double* vbuf = Vr + N * N;
  double* pbuf = vbuf + 2 * N;
  double* Z = pbuf + 2 * N;
  double* U1 = Z + N * N;
  double* U2 = U1 + N * N;
  double* Lm = U2 + N * N;
  double* Dg = Lm + N * N;
  int* Pv = reinterpret_cast<int*>(Dg + N * N);
  int* clus = reinterpret_cast<int*>(Dg + N * N + N * N / 2 + N);
  if (n == 1) {
    LR_CHECK_CUDA(cudaMemcpyAsync(d_out, A, sizeof(double), cudaMemcpyDeviceToDevice, s));
    int st = lr_fill_f64(V, ldv, 1, 1, 1.0, stream);
    if (clusters_host) *clusters_host = 0;
    return st;
  }
  // 1. tridiagonalize
  TdPlan pl = td_plan(n);
  static bool attr = false;
  if (!attr) {
    LR_CHECK_CUDA(cudaFuncSetAttribute(tridiag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    LR_CHECK_CUDA(cudaFuncSetAttribute(backtransform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  int occ = 0;
  LR_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tridiag_kernel, TD_THREADS, pl.smem));
  LR_REQUIRE((long long)occ * sm_count() >= pl.G, "syevd: cooperative grid %d exceeds residency", pl.G);
  TdParams P;
  P.A = A;
  P.lda = lda;
  P.n = n;
  P.rows_per = pl.rows_per;
  P.d = d;
  P.e = e;
  P.tau = tau;
  P.Vr = Vr;
  P.vbuf = vbuf;
  P.pbuf = pbuf;
  P.rows_global = pl.global_rows ? reinterpret_cast<double*>(clus) + N + 64 : nullptr;
  LR_CHECK_CUDA(cudaMemsetAsync(tau, 0, N * sizeof(double), s));
  static const bool timing = getenv("LR_SYEVD_TIMING") != nullptr;
  cudaEvent_t ev[6];
  if (timing)
    for (int i = 0; i < 6; ++i) {
      cudaEventCreate(&ev[i]);
    }
  if (timing) cudaEventRecord(ev[0], s);
  void* args[] = {&P};
  LR_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)tridiag_kernel, dim3(pl.G), dim3(TD_THREADS), args,
                                            pl.smem, s));
  count_launches(1);
  if (timing) cudaEventRecord(ev[1], s);
  // 2. eigenvalues (ascending) by multisection
  tri_prep_kernel<<<1, 256, 0, s>>>(d, e, n, e2, bounds);
  LR_CHECK_LAUNCH();
  bisect_kernel<<<(n * 32 + 255) / 256, 256, 0, s>>>(d, e2, n, bounds, w);
  LR_CHECK_LAUNCH();
  if (timing) cudaEventRecord(ev[2], s);
  // 3. eigenvectors of T
  inviter_kernel<<<(n + 63) / 64, 64, 0, s>>>(d, e, n, w, bounds, Z, U1, U2, Lm, Dg, Pv);
  LR_CHECK_LAUNCH();
  if (timing) cudaEventRecord(ev[3], s);
  // 4. clusters (host decides from the eigenvalues: one small D2H)
  double* wh = new double[n + 4];
  LR_CHECK_CUDA(cudaMemcpyAsync(wh, w, N * sizeof(double), cudaMemcpyDeviceToHost, s));
  LR_CHECK_CUDA(cudaMemcpyAsync(wh + n, bounds, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
  LR_CHECK_CUDA(cudaStreamSynchronize(s));
  const double ctol = 1e-8 * fmax(wh[n + 3], 1e-300);
  int* ch = new int[2 * n];
  int ncl = 0;
  for (int i = 0; i < n;) {
    int j = i + 1;
    while (j < n && wh[j] - wh[j - 1] <= ctol) ++j;
    if (j - i > 1) {
      ch[2 * ncl] = i;
      ch[2 * ncl + 1] = j;
      ++ncl;
    }
    i = j;
  }
  if (ncl) {
    cudaError_t ce = cudaMemcpyAsync(clus, ch, 2 * ncl * sizeof(int), cudaMemcpyHostToDevice, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) {
      delete[] wh;
      delete[] ch;
      set_error("syevd: cluster upload: %s", cudaGetErrorString(ce));
      return LR_ERR_CUDA;
    }
    cluster_mgs_kernel<<<ncl, 256, 0, s>>>(Z, n, clus);
  }
  delete[] wh;
  delete[] ch;
  if (ncl) LR_CHECK_LAUNCH();
  if (clusters_host) *clusters_host = ncl;
  if (timing) cudaEventRecord(ev[4], s);
  // 5. back-transform and eigenvalues out
  const int wpb = (size_t)n * 4 * sizeof(double) <= 200 * 1024 ? 4 : 1;
  LR_REQUIRE((size_t)n * wpb * sizeof(double) <= 200 * 1024, "syevd: n = %d too large for the back-transform", n);
  backtransform_kernel<<<(n + wpb - 1) / wpb, 32 * wpb, (size_t)wpb * n * sizeof(double), s>>>(Z, Vr, tau, n, V, ldv);
  LR_CHECK_LAUNCH();
  LR_CHECK_CUDA(cudaMemcpyAsync(d_out, w, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (timing) {
    cudaEventRecord(ev[5], s);
    cudaEventSynchronize(ev[5]);
    float t[5];
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    fprintf(stderr, "syevd n=%d G=%d: tridiag %.3f bisect %.3f inviter %.3f clusters(%d) %.3f backtr %.3f ms\n", n,
            pl.G, t[0], t[1], t[2], ncl, t[3], t[4]);
    for (int i = 0; i < 6; ++i) cudaEventDestroy(ev[i]);
  }
  return LR_OK;
}

}  // extern "C"
