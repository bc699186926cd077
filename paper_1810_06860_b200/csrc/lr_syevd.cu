// Symmetric eigendecomposition by Householder tridiagonalization, bisection
// and inverse iteration -- the default replacement for LAPACK dsyevd behind
// `sym_eig` / `eig_svd` (linalg.py:153-202; survey K5).
//
//   1. tridiag   : one cooperative kernel; the n x n matrix is row-distributed
//                  over the CTAs' shared memory.  ONE grid barrier per column:
//                  every CTA publishes its slice of p = tau*A*v and the owner
//                  of row j+1 publishes that row; after the barrier every CTA
//                  forms w = p - tau/2 (p.v) v, applies A -= v w^T + w v^T to
//                  its rows and derives the next reflector (dlarfg convention)
//                  redundantly from the published row -- bit-identical in all
//                  CTAs.  (single CTA, 1024 threads, for n <= 96)
//   2. bisection : one warp per eigenvalue, 32-way multisection on Sturm counts
//                  (eigenvalue i is the i-th smallest: the output is ascending).
//   3. inverse iteration : one thread per eigenvalue, two solves with the
//                  dlagtf-pivoted tridiagonal LU ([row][eigenvalue] scratch).
//   4. clusters  : eigenvalues closer than 1e-8*||T|| are re-orthonormalised
//                  (modified Gram-Schmidt, twice) by one CTA per cluster.
//   5. back-transform : compact WY blocks of 32 reflectors (T factors built in
//                  parallel), applied by one CTA per 8 eigenvector columns with
//                  the block's reflectors staged in shared memory.
// Accuracy is LAPACK's: eigenvalues to O(eps*||A||) absolute, eigenvectors to
// O(eps*||A||/gap).  Latency-bound (one grid barrier per column): reported as
// time and share of the step.
#include <cooperative_groups.h>
#include <cstdlib>

#include "lr_common.cuh"

namespace cg = cooperative_groups;

namespace lr {

constexpr int TD_NMAX_FAST = 2048;  // n up to which the post-barrier loads are one batch per thread
constexpr int kPvSlots = 2 * 512;  // p.v partial slots (2 x G, G <= SM count)
constexpr int TD_PPL = 8;   // p.v partials per lane: G <= 256  // trailing elements per thread loaded in one batch after the column barrier

// 1/x to within an ulp: MUFU.RCP64H seed refined by two Newton steps (x is a
// clamped pivot: never zero, never denormal)
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// 1/sqrt(x) for x > 0: MUFU.RSQ64H seed and two Newton steps
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

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
  double* pvbuf;  // 2 x G per-CTA partials of p.v
  double* rows_global;  // n x (n+1) working rows when they do not fit shared memory, else null
  long long* prof;      // optional per-phase clocks of CTA 0 (LR_SYEVD_TIMING)
};

__device__ __forceinline__ void td_barrier(cg::grid_group& grid) {
  if (gridDim.x == 1)
    __syncthreads();
  else
    grid.sync();
}

// Reflector of x[j+1:] (dlarfg): every CTA computes it redundantly from the
// same data in the same order, so all CTAs hold bit-identical v and tau.
template <int THREADS>
__device__ __forceinline__ void td_reflector(const double* x, int j, int n, double* v, double* red, double* sh,
                                             const TdParams& P, bool record) {
  const int tid = threadIdx.x;
  double ss = 0.0;
  for (int c = j + 2 + tid; c < n; c += THREADS) ss = fma(x[c], x[c], ss);
  ss = block_sum<THREADS>(ss, red);
  if (tid == 0) {
    const double alpha = x[j + 1];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (ss != 0.0) {
      const double x2 = alpha * alpha + ss;
      const double nrm = x2 * fast_rsqrt(x2);
      beta = (alpha >= 0.0) ? -nrm : nrm;
      tau = (beta - alpha) * fast_rcp(beta);
      scal = fast_rcp(alpha - beta);
    }
    sh[0] = tau;
    sh[1] = scal;
    if (record) {
      P.d[j] = x[j];
      P.e[j] = beta;
      P.tau[j] = tau;
    }
  }
  __syncthreads();
  const double tau = sh[0], scal = sh[1];
  for (int c = j + 1 + tid; c < n; c += THREADS) {
    const double vc = (c == j + 1) ? 1.0 : (tau == 0.0 ? 0.0 : x[c] * scal);
    v[c] = vc;
    if (record) P.Vr[(long long)j * n + c] = vc;
  }
  __syncthreads();
}

// One grid barrier per column: before the barrier every CTA publishes its
// slice of p = tau*A*v and the owner of row j+1 publishes that row (state
// after step j-1); after it every CTA forms w, updates its rows, rebuilds
// row j+1 after step j from the published copy with the same rank-2 formula
// and derives the next reflector redundantly.
// SINGLE (one CTA holds every row, n <= 96): p, the row j+1 copy and the
// p.v partial stay in shared memory -- no L2 round trip per column.
template <int THREADS, bool SINGLE = false>
__global__ void __launch_bounds__(THREADS) tridiag_kernel(TdParams P) {
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
  double* w = v + n;                                                       // n
  double* x = w + n;                                                       // n
  double* psh = x + n;                                // n (SINGLE: p in shared memory)
  __shared__ double red[32];
  __shared__ double sh[4];
  const bool rec = blockIdx.x == 0;
  auto ldx = [](const double* q) { return SINGLE ? *q : __ldcg(q); };
  constexpr int EPT = (TD_NMAX_FAST + THREADS - 1) / THREADS;  // 8 at 256 threads, 2 at 1024

  for (int e = tid; e < nr * n; e += THREADS) {
    const int i = e / n, c = e - (e / n) * n;
    R[i * LD + c] = P.A[(long long)(r0 + i) * P.lda + c];
  }
  // row 0 to every CTA, then the first reflector
  if (r0 == 0)
    for (int c = tid; c < n; c += THREADS) P.vbuf[c] = P.A[c];
  td_barrier(grid);
  for (int c = tid; c < n; c += THREADS) x[c] = P.vbuf[c];
  __syncthreads();
  if (n > 2) td_reflector<THREADS>(x, 0, n, v, red, sh, P, rec);

  for (int j = 0; j + 2 < n; ++j) {
    const int par = j & 1;
    double* pg = SINGLE ? psh : P.pbuf + par * n;
    double* rg = SINGLE ? R + (j + 1) * LD : P.vbuf + (1 - par) * n;  // row j+1 (vbuf[0] held row 0)
    const double tau = sh[0];
    long long* prof = (P.prof && blockIdx.x == 0 && tid == 0) ? P.prof : nullptr;
    long long tp[6];
    if (prof) tp[0] = clock64();
    // (a) my slice of p, (b) the owner publishes row j+1
    if (tau != 0.0) {
      const int lane = tid & 31, wp = tid >> 5;
      double wpv = 0.0;  // this warp's share of p.v (rows in order)
      for (int i = wp; i < nr; i += THREADS / 32) {
        const int r = r0 + i;
        if (r <= j) continue;
        const double* row = R + i * LD;
        double s = 0.0;
        for (int c = j + 1 + lane; c < n; c += 32) s = fma(row[c], v[c], s);
        s = warp_sum(s);
        const double pr = tau * s;
        if (lane == 0) pg[r] = pr;
        wpv = fma(pr, v[r], wpv);
      }
      // CTA partial of p.v published with p: the post-barrier phase sums the
      // G partials per warp instead of a block reduction over p
      if (lane == 0) red[wp] = wpv;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int q = 0; q < THREADS / 32; ++q) t += red[q];
        if (SINGLE)
          sh[3] = t;
        else
          P.pvbuf[par * gridDim.x + blockIdx.x] = t;
      }
    }
    if (!SINGLE && j + 1 >= r0 && j + 1 < r1)
      for (int c = j + 1 + tid; c < n; c += THREADS) rg[c] = R[(j + 1 - r0) * LD + c];
    if (prof) tp[1] = clock64();
    td_barrier(grid);
    if (prof) tp[2] = clock64();
    // (c) w = p - (tau/2)(p.v) v  (every CTA, full length); row j+1 copy in
    // the same pass so both vectors cost one L2 round trip
    if (tau != 0.0 && n - (j + 1) <= EPT * THREADS && (int)gridDim.x <= 32 * TD_PPL) {
      // every load of this thread in flight at once (one L2 round trip): its
      // p and row elements and a lane's share of the G partials of p.v,
      // which every warp folds in the same fixed order (bit-identical K in
      // every thread of every CTA, no block reduction)
      const int lane = tid & 31;
      double pcs[EPT], xcs[EPT], pps[TD_PPL];
#pragma unroll
      for (int u = 0; u < EPT; ++u) {
        const int c = j + 1 + tid + u * THREADS;
        pcs[u] = c < n ? ldx(pg + c) : 0.0;
        xcs[u] = c < n ? ldx(rg + c) : 0.0;
      }
      double pv;
      if (SINGLE) {
        pv = sh[3];
      } else {
#pragma unroll
        for (int u = 0; u < TD_PPL; ++u) {
          const int q = lane + 32 * u;
          pps[u] = q < (int)gridDim.x ? __ldcg(P.pvbuf + par * gridDim.x + q) : 0.0;
        }
        pv = 0.0;
#pragma unroll
        for (int u = 0; u < TD_PPL; ++u) pv += pps[u];
        pv = warp_sum(pv);
      }
      const double K = 0.5 * tau * pv;
#pragma unroll
      for (int u = 0; u < EPT; ++u) {
        const int c = j + 1 + tid + u * THREADS;
        if (c < n) {
          x[c] = xcs[u];
          w[c] = pcs[u] - K * v[c];
        }
      }
    } else if (tau != 0.0) {
      double pv = 0.0;
      {
        for (int c = j + 1 + tid; c < n; c += THREADS) {
          const double pc = ldx(pg + c);
          x[c] = ldx(rg + c);
          w[c] = pc;
          pv = fma(pc, v[c], pv);
        }
      }
      pv = block_sum<THREADS>(pv, red);  // valid in thread 0
      if (tid == 0) sh[2] = 0.5 * tau * pv;
      __syncthreads();
      const double K = sh[2];
      for (int c = j + 1 + tid; c < n; c += THREADS) w[c] = w[c] - K * v[c];
    } else {
      for (int c = j + 1 + tid; c < n; c += THREADS) {
        w[c] = 0.0;
        x[c] = ldx(rg + c);
      }
    }
    __syncthreads();
    if (prof) tp[3] = clock64();
    // (d) rank-2 update of my rows; (e) row j+1 after step j from the copy,
    // with this thread's share of the next reflector's ||x[j+3:]||^2
    const int lane = tid & 31, wp = tid >> 5;
    double ssp = 0.0;
    if (tau != 0.0) {
      for (int i = max(0, j + 1 - r0) + wp; i < nr; i += THREADS / 32) {  // warp per row
        const int r = r0 + i;
        const double vr = v[r], wr = w[r];
        double* row = R + i * LD;
        for (int c = j + 1 + lane; c < n; c += 32) row[c] -= __dadd_rn(__dmul_rn(vr, w[c]), __dmul_rn(wr, v[c]));
      }
      for (int c = j + 1 + tid; c < n; c += THREADS) {
        const double xc = x[c] - __dadd_rn(__dmul_rn(v[j + 1], w[c]), __dmul_rn(w[j + 1], v[c]));
        x[c] = xc;
        if (c >= j + 3) ssp = fma(xc, xc, ssp);
      }
    } else {
      for (int c = j + 3 + tid; c < n; c += THREADS) ssp = fma(x[c], x[c], ssp);
    }
    // one barrier closes the update and all-reduces ||x[j+3:]||^2 (every
    // thread folds the warp partials in the same order: bit-identical
    // reflectors in every thread of every CTA, no broadcast round)
    if (THREADS > 256) {  // 32-warp CTA: the block reduction of td_reflector is cheaper than 32-way folds
      __syncthreads();
      if (prof) tp[4] = clock64();
      if (j + 3 < n) {
        td_reflector<THREADS>(x, j + 1, n, v, red, sh, P, rec);
      } else if (rec && tid == 0) {  // j + 1 == n - 2: the last 2 x 2 block
        P.d[n - 2] = x[n - 2];
        P.e[n - 2] = x[n - 1];
        sh[0] = 0.0;
      }
      __syncthreads();
      if (prof) {
        tp[5] = clock64();
        for (int q = 0; q < 5; ++q) prof[q] += tp[q + 1] - tp[q];
      }
      continue;
    }
    ssp = warp_sum(ssp);
    if (lane == 0) red[wp] = ssp;
    __syncthreads();
    if (prof) tp[4] = clock64();
    if (j + 3 < n) {
      double ss = 0.0;
#pragma unroll
      for (int q = 0; q < THREADS / 32; ++q) ss += red[q];
      // dlarfg on x[j+2:] for column j+1, as td_reflector
      const int jr = j + 1;
      const double alpha = x[jr + 1];
      double tau1 = 0.0, beta = alpha, scal = 0.0;
      if (ss != 0.0) {
        // on the column-to-column chain: MUFU seeds + Newton instead of the
        // library sqrt and two divisions
        const double x2 = alpha * alpha + ss;
        const double nrm = x2 * fast_rsqrt(x2);
        beta = (alpha >= 0.0) ? -nrm : nrm;
        tau1 = (beta - alpha) * fast_rcp(beta);
        scal = fast_rcp(alpha - beta);
      }
      if (tid == 0) {
        sh[0] = tau1;
        if (rec) {
          P.d[jr] = x[jr];
          P.e[jr] = beta;
          P.tau[jr] = tau1;
        }
      }
      for (int c = jr + 1 + tid; c < n; c += THREADS) {
        const double vc = (c == jr + 1) ? 1.0 : (tau1 == 0.0 ? 0.0 : x[c] * scal);
        v[c] = vc;
        if (rec) P.Vr[(long long)jr * n + c] = vc;
      }
    } else if (tid == 0) {  // j + 1 == n - 2: the last 2 x 2 block
      if (rec) {
        P.d[n - 2] = x[n - 2];
        P.e[n - 2] = x[n - 1];
      }
      sh[0] = 0.0;
    }
    __syncthreads();
    if (prof) {
      tp[5] = clock64();
      for (int q = 0; q < 5; ++q) prof[q] += tp[q + 1] - tp[q];
    }
  }
  if (n == 2 && rec && tid == 0) {
    P.d[0] = x[0];
    P.e[0] = x[1];
  }
  // d[n-1] from the owner of the last row (after all updates)
  if (tid == 0 && n - 1 >= r0 && n - 1 < r1) P.d[n - 1] = R[(n - 1 - r0) * LD + n - 1];
}

// Sturm count: number of eigenvalues of T strictly below x
// Sturm count (number of eigenvalues of T strictly below x) from the
// leading-minor sequence p_i = det(T_i - x I) = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2}:
// a sign change p_{i-1} -> p_i is a negative pivot q_i = p_i / p_{i-1} of
// LDL^T(T - x I) -- the count dstebz takes from q_i = d_i - x - e^2/q_{i-1}.
// The division-free form puts ONE fma on the loop-carried chain (the
// e^2 p_{i-2} product and d_i - x are off it) instead of a ~125-cycle ddiv;
// T is scaled by 1/||T|| and the pair (p_{i-1}, p_i) is rescaled by a power
// of two every 8 steps (signs and ratios exact), so nothing over- or
// underflows.  An exact zero takes the sign opposite to its predecessor (a
// negative pivot), as a |q| < pivmin pivot does in the division form.
__device__ __forceinline__ int sturm_count(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                           double x, double inv_t) {
  const double inv_t2 = inv_t * inv_t;
  double pm = 1.0;
  double p = (d[0] - x) * inv_t;
  if (p == 0.0) p = -1e-290;
  int cnt = p < 0.0;
#pragma unroll 4
  for (int i = 1; i < n; ++i) {
    const double a = (d[i] - x) * inv_t;
    const double t = (e2[i - 1] * inv_t2) * pm;
    double pn = fma(a, p, -t);
    if (pn == 0.0) pn = (p < 0.0) ? 1e-290 : -1e-290;
    cnt += (pn < 0.0) != (p < 0.0);
    pm = p;
    p = pn;
    if ((i & 7) == 0) {
      const long long ep = (__double_as_longlong(p) >> 52) & 0x7ff;
      const long long eq = (__double_as_longlong(pm) >> 52) & 0x7ff;
      const long long e = ep > eq ? ep : eq;                 // biased exponent of the larger
      const double sc = __longlong_as_double((2046 - e) << 52);  // 2^(1023 - (e - 1023)), exact
      p *= sc;
      pm *= sc;
    }
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
__global__ void bisect_kernel(const double* __restrict__ dg, const double* __restrict__ e2g, int n,
                              const double* __restrict__ bounds, double* __restrict__ w) {
  // d and e^2 staged in shared memory once per block: the Sturm recurrence
  // then reads them at shared-memory latency, off the carried chain
  extern __shared__ double bis_smem[];
  double* d = bis_smem;
  double* e2 = bis_smem + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    d[i] = dg[i];
    if (i + 1 < n) e2[i] = e2g[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= n) return;
  double lo = bounds[0], hi = bounds[1];
  const double pivmin = bounds[2];
  const double inv_t = bounds[3] > 0.0 ? 1.0 / bounds[3] : 1.0;
  // absolute floor: the reduction already perturbs eigenvalues by O(eps*||T||)
  const double abs_floor = 1e-3 * 2.220446049250313e-16 * bounds[3];
  for (int it = 0; it < 40; ++it) {
    const double width = hi - lo;
    if (width <= 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi)) * 2.0 || width <= pivmin ||
        width <= abs_floor)
      break;
    const double x = lo + width * (double)(lane + 1) / 33.0;
    const int c = sturm_count(d, e2, n, x, inv_t);
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
  // Branch-free (lanes hold different shifts, so a branch would run both
  // sides): one reciprocal per step on the recurrence; Dg keeps the clamped
  // reciprocal pivot for the back substitutions.
  auto clamp_rcp = [&](double dg) {
    if (fabs(dg) < tiny) dg = (dg < 0.0) ? -tiny : tiny;
    return 1.0 / dg;
  };
  double a = d[0] - lam;
  double b = n > 1 ? e[0] : 0.0;
  for (int i = 0; i < n - 1; ++i) {
    const double c = e[i];
    const double a_next = d[i + 1] - lam;
    const double b_next = (i + 2 < n) ? e[i + 1] : 0.0;
    const bool keep = fabs(a) >= fabs(c);  // no interchange
    const double piv = keep ? ((a == 0.0) ? tiny : a) : c;
    const double rp = fast_rcp(piv);  // on the carried chain: MUFU + 2 Newton steps, not a ~125-cycle DDIV
    const double l = (keep ? c : a) * rp;
    Dg[IX(i)] = (fabs(piv) < tiny) ? clamp_rcp(piv) : rp;
    U1[IX(i)] = keep ? b : a_next;
    U2[IX(i)] = keep ? 0.0 : b_next;
    Lm[IX(i)] = l;
    Pv[IX(i)] = keep ? 0 : 1;
    const double a2 = keep ? a_next - l * b : b - l * a_next;
    b = keep ? b_next : -l * b_next;
    a = a2;
  }
  Dg[IX(n - 1)] = clamp_rcp((a == 0.0) ? tiny : a);
  unsigned long long s = 0x9E3779B97F4A7C15ULL * (unsigned long long)(k + 1);
  double scale = 1.0;
  // two solves: the shift is accurate to ~1e-3 eps ||T|| (bisection), so the
  // first solve already amplifies the wanted direction by ~1/(eps*||T||).
  // The recurrences are branch-free and their operands are fetched 8 steps
  // at a time, so the L2 latency is paid once per 8 steps, not per step.
  constexpr int PF = 16;
  for (int it = 0; it < 2; ++it) {
    // forward: z <- L^{-1} P (scale * z); the start vector is generated in pass 0
    double zc;
    if (it == 0) {
      s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
      zc = (double)((s * 2685821657736338717ULL) >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    } else {
      zc = Z[IX(0)] * scale;
    }
    for (int i0 = 0; i0 < n - 1; i0 += PF) {
      double lv[PF], zv[PF];
      int pv[PF];
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int i = i0 + q;
        const bool ok = i < n - 1;
        lv[q] = ok ? Lm[IX(i)] : 0.0;
        pv[q] = ok ? Pv[IX(i)] : 0;
        if (it == 0) {
          s ^= s >> 12; s ^= s << 25; s ^= s >> 27;
          zv[q] = (double)((s * 2685821657736338717ULL) >> 11) * (2.0 / 9007199254740992.0) - 1.0;
        } else {
          zv[q] = ok ? Z[IX(i + 1)] * scale : 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int i = i0 + q;
        if (i < n - 1) {
          const double zn = zv[q], l = lv[q];
          const double keep = pv[q] ? zn : zc;       // value stored at row i
          const double next = pv[q] ? zc - l * zn : zn - l * zc;
          Z[IX(i)] = keep;
          zc = next;
        }
      }
    }
    Z[IX(n - 1)] = zc;
    // backward: U x = y (Dg holds reciprocal pivots), track max |x| for the next scale
    double x1 = 0.0, x2 = 0.0, mx = 0.0;
    for (int i0 = n - 1; i0 >= 0; i0 -= PF) {
      double zv[PF], u1[PF], u2[PF], rd[PF];
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int i = i0 - q;
        const bool ok = i >= 0;
        zv[q] = ok ? Z[IX(i)] : 0.0;
        u1[q] = ok ? U1[IX(i)] : 0.0;
        u2[q] = ok ? U2[IX(i)] : 0.0;
        rd[q] = ok ? Dg[IX(i)] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const int i = i0 - q;
        if (i >= 0) {
          const double xi = (zv[q] - u1[q] * x1 - u2[q] * x2) * rd[q];
          Z[IX(i)] = xi;
          x2 = x1;
          x1 = xi;
          mx = fmax(mx, fabs(xi));
        }
      }
    }
    scale = (mx > 0.0) ? 1.0 / mx : 1.0;
  }
  double ss = 0.0, ss1 = 0.0;
#pragma unroll 16
  for (int i = 0; i < n; ++i) {
    const double z = Z[IX(i)] * scale;
    if (i & 1)
      ss1 = fma(z, z, ss1);
    else
      ss = fma(z, z, ss);
  }
  ss += ss1;
  const double inv = scale / sqrt(ss);
#pragma unroll 16
  for (int i = 0; i < n; ++i) Z[IX(i)] *= inv;
#undef IX
}

// modified Gram-Schmidt (twice) over a cluster [k0, k1) of columns of Z (n x n row-major)
__device__ void cluster_mgs_one(double* Z, int n, const int k0, const int k1) {
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

// Clusters of the ascending eigenvalues w: maximal runs [k0, k1), k1 - k0 > 1,
// of neighbours within ctol = 1e-8 * max(|lambda|) (bounds[3]).  One warp, 32
// entries per step: a run starts where the gap to the left is open and the gap
// to the right closed, ends where the reverse holds; the k-th start pairs with
// the k-th end.  Written to clusters[0 .. 2 ncl) and count[0] on the device, so
// the eigensolver never waits for the host.
__global__ void cluster_find_kernel(const double* __restrict__ w, const double* __restrict__ bounds, int n,
                                    int* __restrict__ clusters, int* __restrict__ count) {
  const int lane = threadIdx.x;
  const double ctol = 1e-8 * fmax(bounds[3], 1e-300);
  const unsigned below = (1u << lane) - 1u;
  int cs = 0, ce = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    bool st = false, en = false;
    if (i < n) {
      const double wi = w[i];
      const bool prev_close = i > 0 && wi - w[i - 1] <= ctol;
      const bool next_close = i + 1 < n && w[i + 1] - wi <= ctol;
      st = !prev_close && next_close;
      en = prev_close && !next_close;
    }
    const unsigned bs = __ballot_sync(~0u, st), be = __ballot_sync(~0u, en);
    if (st) clusters[2 * (cs + __popc(bs & below))] = i;
    if (en) clusters[2 * (ce + __popc(be & below)) + 1] = i + 1;
    cs += __popc(bs);
    ce += __popc(be);
  }
  if (lane == 0) count[0] = cs;
}

// grid-stride over the clusters found by cluster_find_kernel (count on the device)
__global__ void __launch_bounds__(256) cluster_mgs_kernel(double* Z, int n, const int* clusters, const int* count) {
  const int ncl = count[0];
  for (int c = blockIdx.x; c < ncl; c += gridDim.x) cluster_mgs_one(Z, n, clusters[2 * c], clusters[2 * c + 1]);
}

// T factor of each block of kWY reflectors (dlarft, forward, columnwise):
// T_ii = tau_i, T[0:i, i] = -tau_i T[0:i, 0:i] (V[:, 0:i]^T v_i).  Vr rows hold
// the reflectors with explicit zeros left of the unit entry.
constexpr int kWY = 32;
__global__ void __launch_bounds__(256) build_T_kernel(const double* __restrict__ Vr, const double* __restrict__ tau,
                                                    int n, int nrefl, double* __restrict__ T) {
  __shared__ double G[kWY][kWY + 1];
  __shared__ double Ts[kWY][kWY + 1];
  const int b = blockIdx.x, J = b * kWY;
  const int bs = min(kWY, nrefl - J);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  // G[k][i] = v_{J+k} . v_{J+i}, k < i (overlap starts at column J+i+1)
  for (int pr = wp; pr < kWY * kWY; pr += 8) {
    const int k = pr / kWY, i = pr % kWY;
    if (k >= i || i >= bs) continue;
    const double* a = Vr + (long long)(J + k) * n;
    const double* c = Vr + (long long)(J + i) * n;
    double sacc = 0.0;
    for (int col = J + i + 1 + lane; col < n; col += 32) sacc = fma(a[col], c[col], sacc);
    sacc = warp_sum(sacc);
    if (lane == 0) G[k][i] = sacc;
  }
  for (int e = threadIdx.x; e < kWY * kWY; e += 256) Ts[e / kWY][e % kWY] = 0.0;
  __syncthreads();
  for (int i = 0; i < bs; ++i) {
    const double ti = tau[J + i];
    if (threadIdx.x < i) {
      const int r = threadIdx.x;
      double acc = 0.0;
      for (int k = r; k < i; ++k) acc = fma(Ts[r][k], G[k][i], acc);
      Ts[r][i] = -ti * acc;
    }
    if (threadIdx.x == 0) Ts[i][i] = ti;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kWY * kWY; e += 256) T[(long long)b * kWY * kWY + e] = Ts[e / kWY][e % kWY];
}

// All reflector blocks applied to a tile of kTC eigenvector columns by one
// CTA (columns are independent: no inter-CTA dependency, one launch):
// for b = last..0:  Y = V_b^T Z_tile, Y = T_b Y, Z_tile -= V_b Y.
// Register-blocked for shared-memory bandwidth: in Y = V^T Z a lane owns one
// reflector k and all kTC columns (Z row broadcast, V row conflict-free), four
// warps split the reflector length and fold in fixed order; in Z -= V Y a
// thread owns one row c and all kTC columns.  ~2.6x fewer shared-memory
// wavefronts per FMA than one output per thread.
constexpr int kWyRedWarps = 4;
__device__ __forceinline__ void wy_cp_async8(double* smem, const double* gmem) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gmem));
}

template <int kTC>
__global__ void __launch_bounds__(256) wy_apply_kernel(double* __restrict__ Z, int n, const double* __restrict__ Vr,
                                                     const double* __restrict__ T, int nrefl, double* __restrict__ V,
                                                     long long ldv, int stage_v) {
  extern __shared__ double zs[];  // n x kTC, then (staged) the block's reflector rows
  __shared__ double red[kWyRedWarps][kWY][kTC];  // per-warp partials; red[0] then holds Y
  __shared__ double Y2[kWY][kTC];
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int c0 = blockIdx.x * kTC;
  const int tc = min(kTC, n - c0);
  for (int e = tid; e < n * kTC; e += 256) {
    const int i = e / kTC, t = e % kTC;
    zs[e] = (t < tc) ? Z[(long long)i * n + c0 + t] : 0.0;
  }
  const int nblk = (nrefl + kWY - 1) / kWY;
  double* vb = stage_v ? zs + (size_t)n * kTC : nullptr;
  const int LDV = n + 1;
  for (int b = nblk - 1; b >= 0; --b) {
    const int J = b * kWY;
    const int bsb = min(kWY, nrefl - J);
    if (vb) {
      // stage the block's reflector rows with asynchronous 8-byte copies: every
      // copy of the thread in flight at once, one wait (the plain load/store
      // loop paid an L2 round trip per few elements)
      for (int q = 0; q < bsb; ++q) {
        const double* src = Vr + (long long)(J + q) * n;
        double* dst = vb + q * LDV;
        for (int c = J + 1 + tid; c < n; c += 256) wy_cp_async8(dst + c, src + c);
      }
      asm volatile("cp.async.commit_group;\n" ::);
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    // (1) partials of Y[k][:] over a quarter of the reflector length
    if (wp < kWyRedWarps) {
      double acc[kTC];
#pragma unroll
      for (int t = 0; t < kTC; ++t) acc[t] = 0.0;
      if (lane < bsb) {
        const double* vrow = vb ? vb + lane * LDV : Vr + (long long)(J + lane) * n;
        for (int c = J + 1 + wp; c < n; c += kWyRedWarps) {
          const double v = vrow[c];
          const double* zr = zs + c * kTC;
#pragma unroll
          for (int t = 0; t < kTC; ++t) acc[t] = fma(v, zr[t], acc[t]);
        }
      }
#pragma unroll
      for (int t = 0; t < kTC; ++t) red[wp][lane][t] = acc[t];
    }
    __syncthreads();
    if (tid < kWY * kTC) {  // fixed-order fold -> Y (in red[0])
      const int k = tid / kTC, t = tid % kTC;
      double y = red[0][k][t];
#pragma unroll
      for (int w = 1; w < kWyRedWarps; ++w) y += red[w][k][t];
      red[0][k][t] = y;
    }
    __syncthreads();
    // (2) Y2 = T_b Y (T from global; 32 x 32, read through L1)
    if (tid < kWY * kTC) {
      const int k = tid / kTC, t = tid % kTC;
      const double* Trow = T + (long long)b * kWY * kWY + k * kWY;
      double a2 = 0.0;
      for (int q = 0; q < bsb; ++q) a2 = fma(Trow[q], red[0][q][t], a2);
      Y2[k][t] = a2;
    }
    __syncthreads();
    // (3) Z rows -= V_b^T-row . Y2
    for (int c = J + 1 + tid; c < n; c += 256) {
      double acc[kTC];
#pragma unroll
      for (int t = 0; t < kTC; ++t) acc[t] = zs[c * kTC + t];
      for (int q = 0; q < bsb; ++q) {
        const double v = vb ? vb[q * LDV + c] : Vr[(long long)(J + q) * n + c];
#pragma unroll
        for (int t = 0; t < kTC; ++t) acc[t] = fma(-v, Y2[q][t], acc[t]);
      }
#pragma unroll
      for (int t = 0; t < kTC; ++t) zs[c * kTC + t] = acc[t];
    }
    __syncthreads();
  }
  for (int e = tid; e < n * kTC; e += 256) {
    const int i = e / kTC, tt = e % kTC;
    if (tt < tc) V[(long long)i * ldv + c0 + tt] = zs[e];
  }
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
  // CTAs: every CTA re-reads the broadcast vectors each column, so fewer,
  // fatter CTAs cut L2 contention (tunable: LR_TD_ROWS = rows per CTA)
  // (clamped to >= 1: 0 would divide by zero below)
  static const int rows_pref = env_int_clamped("LR_TD_ROWS", 8, 1, 1 << 20);  // swept: tools/td_rows_probe.py
  // one CTA (no grid barrier) up to single_max (tunable: LR_TD_SINGLE_MAX, clamped to the
  // sizes whose one-CTA rows still fit shared memory)
  static const int single_max = env_int_clamped("LR_TD_SINGLE_MAX", 96, 0, 156);
  int G = n <= single_max ? 1 : (n + rows_pref - 1) / rows_pref;
  if (G > sms) G = sms;
  int rows_per = (n + G - 1) / G;
  G = (n + rows_per - 1) / rows_per;
  size_t smem = ((size_t)rows_per * (n + 1) + 3 * (size_t)n) * sizeof(double);
  pl.global_rows = smem > 200 * 1024;
  if (pl.global_rows) smem = 3 * (size_t)n * sizeof(double);
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
  // | WY T factors (one kWY x kWY block per 32 reflectors)
  return 6 * N + 8 + N * N + 4 * N + 5 * N * N + N * N / 2 + N + N + 64 + N * (N + 1) +
         ((N + kWY - 1) / kWY + 1) * kWY * kWY + kPvSlots;
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
    LR_CHECK_CUDA(cudaFuncSetAttribute(tridiag_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    LR_CHECK_CUDA(cudaFuncSetAttribute(tridiag_kernel<1024, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       220 * 1024));
    LR_CHECK_CUDA(cudaFuncSetAttribute(wy_apply_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 214 * 1024));
    LR_CHECK_CUDA(cudaFuncSetAttribute(wy_apply_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 214 * 1024));
    attr = true;
  }
  int occ = 0;
  const bool single = pl.G == 1;
  const void* tdk = single ? (const void*)tridiag_kernel<1024, true> : (const void*)tridiag_kernel<256>;
  if (single) pl.smem += (size_t)n * sizeof(double);  // p in shared memory
  LR_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tdk, single ? 1024 : 256, pl.smem));
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
  // per-CTA p.v partials (2 x G), after the WY T factors
  P.pvbuf = reinterpret_cast<double*>(clus) + N + 64 + N * (N + 1) + ((N + kWY - 1) / kWY + 1) * kWY * kWY;
  P.rows_global = pl.global_rows ? reinterpret_cast<double*>(clus) + N + 64 : nullptr;
  static const bool timing_env = getenv("LR_SYEVD_TIMING") != nullptr;
  // phase clocks borrow the eigenvalue buffer w (written only after the reduction)
  P.prof = (timing_env && n >= 8) ? reinterpret_cast<long long*>(w) : nullptr;
  if (P.prof) LR_CHECK_CUDA(cudaMemsetAsync(w, 0, 8 * sizeof(double), s));
  LR_CHECK_CUDA(cudaMemsetAsync(tau, 0, N * sizeof(double), s));
  LR_CHECK_CUDA(cudaMemsetAsync(Vr, 0, N * N * sizeof(double), s));  // zeros left of each unit entry
  static const bool timing = getenv("LR_SYEVD_TIMING") != nullptr;
  cudaEvent_t ev[6];
  if (timing)
    for (int i = 0; i < 6; ++i) {
      cudaEventCreate(&ev[i]);
    }
  if (timing) cudaEventRecord(ev[0], s);
  void* args[] = {&P};
  LR_CHECK_CUDA(cudaLaunchCooperativeKernel(tdk, dim3(pl.G), dim3(single ? 1024 : 256), args, pl.smem, s));
  count_launches(1);
  if (timing) cudaEventRecord(ev[1], s);
  if (P.prof) {
    long long hp[5];
    cudaMemcpyAsync(hp, P.prof, sizeof(hp), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "tridiag n=%d G=%d cycles/col: p+publish %.0f barrier %.0f w+x %.0f update %.0f reflector %.0f\n", n,
            pl.G, (double)hp[0] / n, (double)hp[1] / n, (double)hp[2] / n, (double)hp[3] / n, (double)hp[4] / n);
  }
  // 2. eigenvalues (ascending) by multisection
  tri_prep_kernel<<<1, 256, 0, s>>>(d, e, n, e2, bounds);
  LR_CHECK_LAUNCH();
  {
    const size_t bsm = 2 * (size_t)n * sizeof(double);
    LR_REQUIRE(bsm <= 200 * 1024, "syevd: n = %d exceeds the bisection staging limit", n);
    static bool battr = false;
    if (!battr) {
      LR_CHECK_CUDA(cudaFuncSetAttribute(bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      battr = true;
    }
    bisect_kernel<<<(n * 32 + 255) / 256, 256, bsm, s>>>(d, e2, n, bounds, w);
  }
  LR_CHECK_LAUNCH();
  if (timing) cudaEventRecord(ev[2], s);
  // 3. eigenvectors of T
  inviter_kernel<<<(n + 63) / 64, 64, 0, s>>>(d, e, n, w, bounds, Z, U1, U2, Lm, Dg, Pv);
  LR_CHECK_LAUNCH();
  if (timing) cudaEventRecord(ev[3], s);
  // 4. clusters, found on the device (no host round trip inside the eigensolver)
  int* ncl_dev = clus + 2 * N;  // inside the 64-double pad after the cluster pairs
  cluster_find_kernel<<<1, 32, 0, s>>>(w, bounds, n, clus, ncl_dev);
  LR_CHECK_LAUNCH();
  cluster_mgs_kernel<<<std::max(1, std::min(n / 2, 64)), 256, 0, s>>>(Z, n, clus, ncl_dev);
  LR_CHECK_LAUNCH();
  if (clusters_host) {  // optional diagnostic: costs a stream sync
    LR_CHECK_CUDA(cudaMemcpyAsync(clusters_host, ncl_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
    LR_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  if (timing) cudaEventRecord(ev[4], s);
  // 5. back-transform and eigenvalues out
  // blocked (compact WY) back-transform: Z <- B_0 (B_1 (... (B_last Z))),
  // B_b = H_J ... H_{J+31} = I - V_b T_b V_b^T, three DMMA GEMMs per block
  if (n > 2) {
    const int nrefl = n - 2;  // reflectors 0 .. n-3
    const int nblk = (nrefl + kWY - 1) / kWY;
    // nblk x kWY x kWY T factors in their own region (reusing Lm overflowed it for n < ~32)
    double* Tb = reinterpret_cast<double*>(clus) + N + 64 + N * (N + 1);
    build_T_kernel<<<nblk, 256, 0, s>>>(Vr, tau, n, nrefl, Tb);
    LR_CHECK_LAUNCH();
    const size_t vsm = (size_t)kWY * (n + 1) * sizeof(double);
    if ((size_t)n * 8 * sizeof(double) <= 200 * 1024) {
      const size_t zsm = (size_t)n * 8 * sizeof(double);
      const int stage = zsm + vsm <= 214 * 1024;  // + ~10 KB static fits the 227 KB per CTA
      wy_apply_kernel<8><<<(n + 7) / 8, 256, stage ? zsm + vsm : zsm, s>>>(Z, n, Vr, Tb, nrefl, V, ldv, stage);
    } else {
      const size_t zsm = (size_t)n * 2 * sizeof(double);
      LR_REQUIRE(zsm <= 200 * 1024, "syevd: n = %d too large for the back-transform tile", n);
      wy_apply_kernel<2><<<(n + 1) / 2, 256, zsm, s>>>(Z, n, Vr, Tb, nrefl, V, ldv, 0);
    }
    LR_CHECK_LAUNCH();
  } else {
    int st = lr_copy2d_f64(Z, n, V, ldv, n, n, 0, stream);
    if (st) return st;
  }
  LR_CHECK_CUDA(cudaMemcpyAsync(d_out, w, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (timing) {
    cudaEventRecord(ev[5], s);
    cudaEventSynchronize(ev[5]);
    int ncl = 0;
    cudaMemcpy(&ncl, ncl_dev, sizeof(int), cudaMemcpyDeviceToHost);
    float t[5];
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    fprintf(stderr, "syevd n=%d G=%d: tridiag %.3f bisect %.3f inviter %.3f clusters(%d) %.3f backtr %.3f ms\n", n,
            pl.G, t[0], t[1], t[2], ncl, t[3], t[4]);
    for (int i = 0; i < 6; ++i) cudaEventDestroy(ev[i]);
  }
  return LR_OK;
}

}  // extern "C"
