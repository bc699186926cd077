// Blocked upper Cholesky (A = R^T R) and triangular inverse R^{-1} for the
// W x W Grams of CholeskyQR2 / shifted CholeskyQR3 -- the GPU replacement for
// the Householder QR of `orth` (linalg.py:101-124; survey K3).  Diagonal
// 64x64 blocks are factored and inverted in shared memory by one CTA; panel
// and trailing updates are DMMA GEMMs (lr_gemm.cu).  A device flag makes the
// remaining work a no-op after a non-positive pivot; the host reads `info`.
#include <cooperative_groups.h>
#include <stdlib.h>

#include "lr_common.cuh"

namespace lr {

namespace cg = cooperative_groups;

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

// ------------------------------------------------------------------------
// One cooperative kernel for W <= kCoopMaxN (every W of the BASELINE configs):
// the host-driven blocked path above costs ~50 launches of tiny GEMMs per
// call (2.5 ms at W = 660); here the whole factorization + inverse is one
// launch with ONE grid barrier per 32-column block step.
//
// Step J (after the barrier; R_JJ and inv(R_JJ) are final):
//   every trailing tile (K, L), J < K <= L, is updated by exactly one CTA:
//     P_K = inv(R_JJ)^T A[J,K] (and P_L), A[K,L] -= P_K^T P_L
//   (the panel products are recomputed per tile instead of paying a second
//   barrier); the owner of the diagonal tile (K,K) parks P_K = R[J,K] in a
//   double-buffered panel workspace that step J+1 copies into A[J,K] (A[J,*]
//   is still being read during step J).  CTA 0 owns tile (J+1, J+1) and
//   factors it in shared memory right after updating it: the next step's
//   diagonal block is ready at the barrier.
// Inverse: X = R^{-1} by independent (block column, 8-column slice) units,
// bottom-up inside a unit with the slice kept in shared memory.
constexpr int CB = 32;
constexpr int CB_THREADS = 256;
constexpr int CB_LD = CB + 1;
constexpr int kCoopMaxN = 2048;  // nb <= 64
constexpr int kCoopSmemDoubles = 6 * CB * CB_LD;

__device__ __forceinline__ void cb_load(const double* __restrict__ A, long long lda, int n, int I, int K,
                                        double (*t)[CB_LD]) {
  for (int e = threadIdx.x; e < CB * CB; e += CB_THREADS) {
    const int i = e >> 5, c = e & 31;
    const int gi = I * CB + i, gc = K * CB + c;
    t[i][c] = (gi < n && gc < n) ? A[(long long)gi * lda + gc] : 0.0;
  }
}

__device__ __forceinline__ void cb_store(double* __restrict__ A, long long lda, int n, int I, int K,
                                         const double (*t)[CB_LD]) {
  for (int e = threadIdx.x; e < CB * CB; e += CB_THREADS) {
    const int i = e >> 5, c = e & 31;
    const int gi = I * CB + i, gc = K * CB + c;
    if (gi < n && gc < n) A[(long long)gi * lda + gc] = t[i][c];
  }
}

// out = D^T X (D upper: D^T lower -> k <= i), 32 x 32; thread owns row i, 4 cols
// three tiles at once: every global load of the thread is issued before any
// shared store (one L2 round trip instead of one per tile); null src -> skip
__device__ __forceinline__ void cb_load3(const double* A0, long long ld0, int n0, int I0, int K0, double (*t0)[CB_LD],
                                         const double* A1, long long ld1, int n1, int I1, int K1, double (*t1)[CB_LD],
                                         const double* A2, long long ld2, int n2, int I2, int K2,
                                         double (*t2)[CB_LD]) {
  constexpr int PER = CB * CB / CB_THREADS;
  double v0[PER], v1[PER], v2[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = threadIdx.x + u * CB_THREADS, i = e >> 5, c = e & 31;
    {
      const int gi = I0 * CB + i, gc = K0 * CB + c;
      v0[u] = (gi < n0 && gc < n0) ? A0[(long long)gi * ld0 + gc] : 0.0;
    }
    if (A1) {
      const int gi = I1 * CB + i, gc = K1 * CB + c;
      v1[u] = (gi < n1 && gc < n1) ? A1[(long long)gi * ld1 + gc] : 0.0;
    }
    {
      const int gi = I2 * CB + i, gc = K2 * CB + c;
      v2[u] = (gi < n2 && gc < n2) ? A2[(long long)gi * ld2 + gc] : 0.0;
    }
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = threadIdx.x + u * CB_THREADS, i = e >> 5, c = e & 31;
    t0[i][c] = v0[u];
    if (A1) t1[i][c] = v1[u];
    t2[i][c] = v2[u];
  }
}

__device__ __forceinline__ void cb_dtx(const double (*D)[CB_LD], const double (*X)[CB_LD], double (*out)[CB_LD]) {
  const int i = threadIdx.x >> 3, c0 = (threadIdx.x & 7) * 4;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (int k = 0; k <= i; ++k) {
    const double d = D[k][i];
    a0 = fma(d, X[k][c0], a0);
    a1 = fma(d, X[k][c0 + 1], a1);
    a2 = fma(d, X[k][c0 + 2], a2);
    a3 = fma(d, X[k][c0 + 3], a3);
  }
  out[i][c0] = a0;
  out[i][c0 + 1] = a1;
  out[i][c0 + 2] = a2;
  out[i][c0 + 3] = a3;
}

// T -= P^T Q (32 x 32 x 32)
__device__ __forceinline__ void cb_sub_ptq(const double (*P)[CB_LD], const double (*Q)[CB_LD], double (*T)[CB_LD]) {
  const int i = threadIdx.x >> 3, c0 = (threadIdx.x & 7) * 4;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 8
  for (int k = 0; k < CB; ++k) {
    const double p = P[k][i];
    a0 = fma(p, Q[k][c0], a0);
    a1 = fma(p, Q[k][c0 + 1], a1);
    a2 = fma(p, Q[k][c0 + 2], a2);
    a3 = fma(p, Q[k][c0 + 3], a3);
  }
  T[i][c0] -= a0;
  T[i][c0 + 1] -= a1;
  T[i][c0 + 2] -= a2;
  T[i][c0 + 3] -= a3;
}

// Factor the (updated) diagonal tile t of block J in place (upper R, strict
// lower part zeroed; rows / cols >= n padded with the identity) and write
// x = inv(R).  Warp-synchronous: lane c keeps column c of the tile in
// registers and every row broadcast is a shuffle, so the 32-step recurrences
// carry no block barriers (a __syncthreads per step made this 25x slower).
// Returns the 1-based global column of a non-positive pivot, 0 if fine;
// called by ALL threads (warp 0 computes), result block-uniform.
__device__ __forceinline__ double cb_rsqrt(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  // Newton: y <- y (1.5 - 0.5 d y^2), twice (the seed has ~2^-22 relative error)
  const double hd = 0.5 * d;
  y = y * fma(-hd * y, y, 1.5);
  y = y * fma(-hd * y, y, 1.5);
  return y;
}

__device__ int cb_factor(double (*t)[CB_LD], double (*x)[CB_LD], double* rowbuf, int J, int n) {
  __shared__ int s_bad;
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x;
    double a[CB];
#pragma unroll
    for (int i = 0; i < CB; ++i) {
      const bool pad = (J * CB + i >= n) || (J * CB + lane >= n);
      a[i] = pad ? (i == lane ? 1.0 : 0.0) : t[i][lane];
    }
    int bad = 0;
    double rinv_lane = 1.0;  // lane j keeps 1 / R[j][j]
#pragma unroll
    for (int j = 0; j < CB; ++j) {
      const double d = __shfl_sync(FULL, a[j], j);
      if (!(d > 0.0)) {
        bad = J * CB + j + 1;
        break;
      }
      // LAPACK dpotf2 scales the row by 1/R_jj.  1/sqrt(d) from the MUFU
      // seed and two Newton steps (the library sqrt / rsqrt sit on this
      // column-to-column chain for ~100+ cycles each); R_jj = d / sqrt(d)
      const double ri = cb_rsqrt(d);
      const double r = d * ri;
      double v = (lane == j) ? r : a[j] * ri;  // R[j][lane]
      if (lane < j) v = 0.0;
      if (lane == j) rinv_lane = ri;
      a[j] = v;
#pragma unroll
      for (int i = j + 1; i < CB; ++i) a[i] = fma(-__shfl_sync(FULL, v, i), v, a[i]);
    }
    if (lane == 0) s_bad = bad;
    if (!bad) {
      double xr[CB];
#pragma unroll
      for (int i = CB - 1; i >= 0; --i) {
        double s0 = (i == lane) ? 1.0 : 0.0, s1 = 0.0;
#pragma unroll
        for (int k = i + 1; k < CB; k += 2) {
          s0 = fma(-__shfl_sync(FULL, a[i], k), xr[k], s0);
          if (k + 1 < CB) s1 = fma(-__shfl_sync(FULL, a[i], k + 1), xr[k + 1], s1);
        }
        xr[i] = (s0 + s1) * __shfl_sync(FULL, rinv_lane, i);
      }
#pragma unroll
      for (int i = 0; i < CB; ++i) {
        t[i][lane] = (lane < i) ? 0.0 : a[i];
        x[i][lane] = xr[i];
      }
    }
  }
  __syncthreads();
  return s_bad;
}

__device__ __forceinline__ void cb_tile_of(int t, int J, int nb, int& K, int& L) {
  int len = nb - J - 1;
  K = J + 1;
  while (t >= len) {
    t -= len;
    ++K;
    --len;
  }
  L = K + t;
}

__device__ __forceinline__ unsigned long long cb_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// trace (debug, LR_POTRF_TRACE): CTA 0 stamps globaltimer at phase ends
#define CB_STAMP(k)                                                  \
  do {                                                               \
    if (trace && blockIdx.x == 0 && threadIdx.x == 0 && (k) < 128) \
      trace[k] = cb_now();                                           \
  } while (0)

__global__ void __launch_bounds__(CB_THREADS) chol_coop_kernel(int n, double* A, long long lda, double shift,
                                                               double* Rinv, long long ldr, double* ws,
                                                               int* info, unsigned long long* trace) {
  cg::grid_group grid = cg::this_grid();
  CB_STAMP(0);
  extern __shared__ double cb_smem[];
  double(*dinv)[CB_LD] = reinterpret_cast<double(*)[CB_LD]>(cb_smem);
  double(*pk)[CB_LD] = reinterpret_cast<double(*)[CB_LD]>(cb_smem + 1 * CB * CB_LD);
  double(*pl)[CB_LD] = reinterpret_cast<double(*)[CB_LD]>(cb_smem + 2 * CB * CB_LD);
  double(*ld)[CB_LD] = reinterpret_cast<double(*)[CB_LD]>(cb_smem + 3 * CB * CB_LD);
  double(*tt)[CB_LD] = reinterpret_cast<double(*)[CB_LD]>(cb_smem + 4 * CB * CB_LD);
  double(*al)[CB_LD] = reinterpret_cast<double(*)[CB_LD]>(cb_smem + 5 * CB * CB_LD);
  __shared__ double rowbuf[CB];
  __shared__ int s_flag;
  const int nb = (n + CB - 1) / CB;
  const int np = nb * CB;  // padded order of the inverse accumulator
  const int G = gridDim.x, b = blockIdx.x;
  double* Dinv = ws;                                 // nb x CB x CB
  double* Pws = ws + (long long)nb * CB * CB;        // 2 x nb x CB x CB
  double* Acc = Pws + 2LL * nb * CB * CB;            // np x np: E - sum R^T W (inverse, right-looking)
  const bool want_inv = Rinv != nullptr;

  if (shift != 0.0)
    for (int i = b * CB_THREADS + threadIdx.x; i < n; i += G * CB_THREADS) A[(long long)i * lda + i] += shift;
  if (shift != 0.0) grid.sync();
  if (want_inv)
    for (long long e = (long long)b * CB_THREADS + threadIdx.x; e < (long long)np * np;
         e += (long long)G * CB_THREADS)
      Acc[e] = (e / np == e % np) ? 1.0 : 0.0;

  if (b == 0) {
    cb_load(A, lda, n, 0, 0, tt);
    const int bad = cb_factor(tt, pk, rowbuf, 0, n);
    if (bad) {
      if (threadIdx.x == 0) *info = bad;
    } else {
      cb_store(A, lda, n, 0, 0, tt);
      for (int e = threadIdx.x; e < CB * CB; e += CB_THREADS) Dinv[e] = pk[e >> 5][e & 31];
    }
  }
  CB_STAMP(1);
  grid.sync();
  CB_STAMP(2);

  for (int J = 0; J < nb; ++J) {
    if (threadIdx.x == 0) s_flag = *reinterpret_cast<volatile int*>(info);
    __syncthreads();
    if (s_flag != 0) return;  // uniform: every CTA read the flag after the same barrier
    // park the previous step's panel R[J-1, K] (K >= J) into A
    if (J > 0) {
      const double* P = Pws + (long long)((J - 1) & 1) * nb * CB * CB;
      for (int K = J + b; K < nb; K += G) {
        const double* src = P + (long long)K * CB * CB;
        for (int e = threadIdx.x; e < CB * CB; e += CB_THREADS) {
          const int i = e >> 5, c = e & 31;
          const int gi = (J - 1) * CB + i, gc = K * CB + c;
          if (gi < n && gc < n) A[(long long)gi * lda + gc] = src[e];
        }
      }
    }
    // work items of step J:
    //   [0, Tc)        Cholesky trailing tiles (K, L), J < K <= L     (t = 0: CTA 0, then factor)
    //   [Tc, Tc+Ti)    inverse updates Acc[K, L] -= R_JK^T W_JL, K > J >= L
    //   [Tc+Ti, T)     finalize W_JL = inv(R_JJ)^T Acc[J, L] -> Rinv[L, J] = W_JL^T, L <= J
    const int nr = nb - J - 1;
    const int Tc = nr * (nr + 1) / 2;
    const int Ti = want_inv ? nr * (J + 1) : 0;
    const int T = Tc + Ti + (want_inv ? J + 1 : 0);
    bool have_dinv = false;
    const int first = (b == 0) ? 0 : (G == 1 ? 1 : b);
    const int stride = (G == 1) ? 1 : G - 1;
    for (int t = first; t < T; t = (b == 0 && G > 1) ? T : (t == 0 ? 1 : t + stride)) {
      if (!have_dinv) {
        const double* D = Dinv + (long long)J * CB * CB;
        for (int e = threadIdx.x; e < CB * CB; e += CB_THREADS) dinv[e >> 5][e & 31] = D[e];
        have_dinv = true;
      }
      if (t < Tc) {
        int K, L;
        cb_tile_of(t, J, nb, K, L);
        // the operand tiles in flight at once (one L2 round trip)
        cb_load3(A, lda, n, J, K, ld, K != L ? A : nullptr, lda, n, J, L, al, A, lda, n, K, L, tt);
        __syncthreads();
        cb_dtx(dinv, ld, pk);
        if (K != L) cb_dtx(dinv, al, pl);
        __syncthreads();
        cb_sub_ptq(pk, K == L ? pk : pl, tt);
        __syncthreads();
        if (K == L) {
          double* dst = Pws + (long long)(J & 1) * nb * CB * CB + (long long)K * CB * CB;
          for (int e = threadIdx.x; e < CB * CB; e += CB_THREADS) dst[e] = pk[e >> 5][e & 31];
        }
        if (t == 0) {  // CTA 0: next diagonal block
          if (3 * J + 64 < 126) CB_STAMP(3 * J + 64);
          const int bad = cb_factor(tt, pl, rowbuf, K, n);
          if (3 * J + 65 < 126) CB_STAMP(3 * J + 65);
          if (bad) {
            if (threadIdx.x == 0) atomicExch(info, bad);
          } else {
            cb_store(A, lda, n, K, K, tt);
            double* D = Dinv + (long long)K * CB * CB;
            for (int e = threadIdx.x; e < CB * CB; e += CB_THREADS) D[e] = pl[e >> 5][e & 31];
          }
        } else {
          cb_store(A, lda, n, K, L, tt);
        }
      } else if (t < Tc + Ti) {
        const int u = t - Tc;
        const int K = J + 1 + u / (J + 1), L = u % (J + 1);
        cb_load3(A, lda, n, J, K, ld, Acc, np, np, J, L, al, Acc, np, np, K, L, tt);
        __syncthreads();
        cb_dtx(dinv, ld, pk);   // R_JK
        cb_dtx(dinv, al, pl);   // W_JL
        __syncthreads();
        cb_sub_ptq(pk, pl, tt);
        __syncthreads();
        cb_store(Acc, np, np, K, L, tt);
      } else {
        const int L = t - Tc - Ti;
        cb_load(Acc, np, np, J, L, al);
        __syncthreads();
        cb_dtx(dinv, al, pl);
        __syncthreads();
        for (int e = threadIdx.x; e < CB * CB; e += CB_THREADS) {
          const int i = e >> 5, c = e & 31;  // W_JL[i][c] -> Rinv[L*CB + c][J*CB + i]
          const int gr = L * CB + c, gc = J * CB + i;
          if (gr < n && gc < n) Rinv[(long long)gr * ldr + gc] = pl[i][c];
        }
      }
      __syncthreads();
    }
    CB_STAMP(3 + 2 * J);
    grid.sync();
    CB_STAMP(4 + 2 * J);
  }

  // zero the strict lower block triangle of R (diagonal tiles were cleaned by
  // cb_factor) and of R^{-1}
  for (long long e = (long long)b * CB_THREADS + threadIdx.x; e < (long long)n * n;
       e += (long long)G * CB_THREADS) {
    const int i = (int)(e / n), c = (int)(e % n);
    if (i / CB > c / CB) {
      A[(long long)i * lda + c] = 0.0;
      if (want_inv) Rinv[(long long)i * ldr + c] = 0.0;
    }
  }
  CB_STAMP(120);
}

}  // namespace lr

using namespace lr;

extern "C" {

long long lr_potrf_workspace_doubles(int n) {
  // blocked path: Dinv blocks + panel temp; cooperative path: Dinv + 2 panels
  long long nblk = (n + CH_NB - 1) / CH_NB;
  long long blocked = nblk * CH_NB * CH_NB + (long long)CH_NB * n + 64;
  long long nb = (n + CB - 1) / CB;
  long long coop = 3 * nb * CB * CB + (nb * CB) * (nb * CB) + 64;
  return blocked > coop ? blocked : coop;
}

static int potrf_coop(int n, double* A, long long lda, double shift, double* Rinv, long long ldr,
                      double* work, int* info_host, int* info_dev, cudaStream_t s) {
  const int nb = (n + CB - 1) / CB;
  const size_t smem = (size_t)kCoopSmemDoubles * sizeof(double);
  static bool attr = false;
  if (!attr) {
    LR_CHECK_CUDA(cudaFuncSetAttribute(chol_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  int occ = 0;
  LR_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, chol_coop_kernel, CB_THREADS, smem));
  // widest step: Cholesky tiles + inverse updates + finalize ~ nb^2 / 2
  int G = (nb * nb) / 2 + 2;
  if (G > sm_count()) G = sm_count();
  if (G > occ * sm_count()) G = occ * sm_count();
  if (G < 1) G = 1;
  int* info = reinterpret_cast<int*>(work + 3LL * nb * CB * CB + (long long)nb * CB * nb * CB);
  LR_CHECK_CUDA(cudaMemsetAsync(info, 0, sizeof(int), s));
  static const bool tracing = getenv("LR_POTRF_TRACE") != nullptr;
  static unsigned long long* trace = nullptr;
  if (tracing && !trace) LR_CHECK_CUDA(cudaMallocManaged(&trace, 128 * sizeof(unsigned long long)));
  void* args[] = {&n, &A, &lda, &shift, &Rinv, &ldr, &work, &info, &trace};
  LR_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)chol_coop_kernel, dim3((unsigned)G), dim3(CB_THREADS),
                                            args, smem, s));
  LR_CHECK_LAUNCH();
  if (info_dev) LR_CHECK_CUDA(cudaMemcpyAsync(info_dev, info, sizeof(int), cudaMemcpyDeviceToDevice, s));
  if (info_host) {
    LR_CHECK_CUDA(cudaMemcpyAsync(info_host, info, sizeof(int), cudaMemcpyDeviceToHost, s));
    LR_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  if (tracing) {
    LR_CHECK_CUDA(cudaStreamSynchronize(s));
    fprintf(stderr, "potrf_coop n=%d G=%d:", n, G);
    for (int k = 1; k < 4 + 2 * nb; ++k)
      if (trace[k]) fprintf(stderr, " %d:%.1f", k, (trace[k] - trace[0]) * 1e-3);
    fprintf(stderr, "\n  CTA0 diag tile updated / factored:");
    for (int k = 64; k < 126; ++k)
      if (trace[k]) fprintf(stderr, " %d:%.1f", k, (trace[k] - trace[0]) * 1e-3);
    fprintf(stderr, " end:%.1f us\n", (trace[120] - trace[0]) * 1e-3);
    for (int k = 0; k < 128; ++k) trace[k] = 0;
  }
  return LR_OK;
}

static int potrf_impl(int n, double* A, long long lda, double shift, double* Rinv, long long ldr, double* work,
                      int* info_host, int* info_dev, void* stream);

int lr_potrf_inv_f64(int n, double* A, long long lda, double shift, double* Rinv, long long ldr,
                     double* work, int* info_host, void* stream) {
  return potrf_impl(n, A, lda, shift, Rinv, ldr, work, info_host, nullptr, stream);
}

int lr_potrf_inv_async_f64(int n, double* A, long long lda, double shift, double* Rinv, long long ldr,
                           double* work, int* info_dev, void* stream) {
  LR_REQUIRE(info_dev != nullptr, "potrf_async: info_dev is required");
  return potrf_impl(n, A, lda, shift, Rinv, ldr, work, nullptr, info_dev, stream);
}

static int potrf_impl(int n, double* A, long long lda, double shift, double* Rinv, long long ldr, double* work,
                      int* info_host, int* info_dev, void* stream) {
  LR_REQUIRE(n >= 1 && lda >= n && ldr >= n, "potrf: bad shape");
  cudaStream_t s = as_stream(stream);
  static const bool blocked_only = getenv("LR_POTRF_BLOCKED") != nullptr;
  if (n <= kCoopMaxN && !blocked_only)
    return potrf_coop(n, A, lda, shift, Rinv, ldr, work, info_host, info_dev, s);
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
  if (info_dev) LR_CHECK_CUDA(cudaMemcpyAsync(info_dev, info, sizeof(int), cudaMemcpyDeviceToDevice, s));
  if (info_host) {
    LR_CHECK_CUDA(cudaMemcpyAsync(info_host, info, sizeof(int), cudaMemcpyDeviceToHost, s));
    LR_CHECK_CUDA(cudaStreamSynchronize(s));
  }
  return LR_OK;
}

}  // extern "C"
