// Tall-skinny LU with partial pivoting returning P^T L, the replacement for
// scipy.linalg.lu(X, permute_l=True) inside `lu_pl` (linalg.py:127-150;
// survey K4).
//
// One cooperative persistent kernel.  Rows are split into contiguous slabs,
// one per CTA; a panel of nb columns of the slab lives in shared memory.  Per
// column: every CTA proposes its largest |x| among rows not yet pivoted,
// publishes (|x|, row, panel row) and one grid barrier later every CTA picks
// the same winner (largest |x|, ties -> smallest row), so no row swaps are
// ever moved through memory: pivot rows are only marked.  After a panel the
// pivot rows' trailing entries are solved with the panel's unit-lower block
// (forward substitution, redundantly per CTA) and each CTA updates its own
// rows' trailing columns.  Finally pivot rows get their unit entry and zeros
// to its right, which is exactly P^T L.
//
// Latency-bound by construction (one grid barrier per column); reported as
// time and share of the step, not a roofline fraction.
#include <cooperative_groups.h>

#include <cstdlib>

#include "lr_common.cuh"

namespace cg = cooperative_groups;

namespace lr {

#ifndef LR_LU_THREADS
#define LR_LU_THREADS 256
#endif
constexpr int LU_THREADS = LR_LU_THREADS;
constexpr int LU_CHUNK = 128;  // widest U12 chunk of trailing columns (panel-end update)
constexpr int LU_NBMAX = 32;   // widest panel (prow slots are LU_NBMAX doubles)
constexpr int LU_CPL = 10;     // candidates per lane in the winner fold: G <= 320 CTAs
constexpr int kCandWords = 2 * 2;            // per CTA: 2 slots x {value, row}
constexpr int kRowWords = 2 * LU_NBMAX;      // per CTA: 2 slots x panel row

struct LuParams {
  double* X;
  long long ldx;
  int m, n, nb, rows_per;
  int ch;               // U12 chunk width (multiple of 8); row stride ch + 4 (conflict-free DMMA B fragments)
  const double* stats;  // {sumsq, max|x|, nonfinite}
  double* cand;         // [2][G][2]  {|x|, row}
  double* prow;         // [2][G][LU_NBMAX]
  unsigned* bar;        // column barrier counter: G arrivals per column (zeroed before the launch)
  int* pivrow;          // [n]
  double* status;       // {bad col or -1, pivot, tol}
  long long* prof;      // optional per-phase clock totals of CTA 0 (LR_LU_PROFILE)
};

// 1/x on the column chain: MUFU seed + two Newton steps (within an ulp of
// the IEEE quotient; pivots are nonzero and far from the denormal range,
// |pivot| >= 1e-14 max|X| or the factorization stops)
__device__ __forceinline__ double lu_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ void better(double& v, int& r, double v2, int r2) {
  if (v2 > v || (v2 == v && r2 < r)) {
    v = v2;
    r = r2;
  }
}

__device__ __forceinline__ void lu_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Column loop, per column j = J + jj (one split grid barrier per column):
//   1. CTA candidate (look-ahead value from the previous column's pass):
//      block fold, warp 0 publishes {|x|, row} and the candidate's panel row
//      with the still-pending update of step j-1 applied to the copy;
//   2. arrive on the column barrier (fence + one atomic by thread 0);
//   3. the pending update of step j-1 on panel columns > j, overlapping the
//      barrier latency;
//   4. wait (acquire spin on the counter);
//   5. warp 0 folds the G candidates (ties -> smallest row; all loads in
//      flight at once) and fetches the winner's published row;
//   6. multipliers of column j, update of column j+1 only, and the next
//      column's local candidate.
// The published row copy and the deferred in-place update evaluate the same
// fma(-l, u, x), so the pivot row seen by every CTA is bit-identical to the
// owner's.  (A barrier-free exchange of self-validating tagged words was
// measured slower: 1.02 vs 0.89 ms at 100000 x 110 -- every CTA polling
// every candidate costs more than one counter.)
__global__ void __launch_bounds__(LU_THREADS, (512 / LU_THREADS) > 0 ? (512 / LU_THREADS) : 1) lu_kernel(LuParams p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double lu_smem[];
  const int nb = p.nb, LD = nb + 1;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const int r0 = cta * p.rows_per;
  const int r1 = min(p.m, r0 + p.rows_per);
  const int nr = max(0, r1 - r0);
  double* P = lu_smem;                                   // rows_per x LD
  const int LDU = p.ch + 4;
  double* U12 = P + (((long long)p.rows_per * LD + 1) & ~1LL);  // nb x LDU, 16-byte aligned
  double* urow = U12 + nb * LDU;                         // nb
  double* L11 = urow + nb;                               // nb x nb
  int* pivflag = reinterpret_cast<int*>(L11 + nb * nb);  // rows_per
  __shared__ double red_v[LU_THREADS / 32];
  __shared__ int red_r[LU_THREADS / 32];
  __shared__ double win_v;
  __shared__ int pivs[LU_NBMAX];
  long long* prof = (blockIdx.x == 0 && threadIdx.x == 0) ? p.prof : nullptr;
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  double cbv = -1.0;  // local candidate for the current column
  int cbr = 0x7fffffff;

  const double maxabs = p.stats[1];
  const double tol = 1e-14 * maxabs;
  if (maxabs == 0.0 || p.stats[2] != 0.0) return;  // handled by the host wrapper
  for (int i = tid; i < nr; i += LU_THREADS) pivflag[i] = -1;
  // 16-byte column pairs in the panel-end update: even ld, aligned base, even panel width
  const bool vec2 = (p.ldx % 2 == 0) && ((reinterpret_cast<uintptr_t>(p.X) & 15u) == 0) && (nb % 2 == 0);

  for (int J = 0; J < p.n; J += nb) {
    const int jb = min(nb, p.n - J);
    for (int e = tid; e < nr * jb; e += LU_THREADS) {
      int i = e / jb, c = e - (e / jb) * jb;
      P[i * LD + c] = p.X[(long long)(r0 + i) * p.ldx + J + c];
    }
    __syncthreads();
    cbv = -1.0;
    cbr = 0x7fffffff;
    for (int i = tid; i < nr; i += LU_THREADS)
      if (pivflag[i] < 0) better(cbv, cbr, fabs(P[i * LD]), r0 + i);
    for (int jj = 0; jj < jb; ++jj) {
      const int j = J + jj;
      const int par = j & 1;
      if (prof) t0 = clock64();
      // (1) CTA candidate
      double bv = cbv;
      int br = cbr;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        int r2 = __shfl_xor_sync(0xffffffffu, br, o);
        better(bv, br, v2, r2);
      }
      if (lane == 0) {
        red_v[wid] = bv;
        red_r[wid] = br;
      }
      __syncthreads();
      // every warp folds the per-warp winners (all threads learn the CTA
      // candidate row, which warp 0 alone updates below)
      int rc;
      {
        double v = (lane < LU_THREADS / 32) ? red_v[lane] : -1.0;
        int r = (lane < LU_THREADS / 32) ? red_r[lane] : 0x7fffffff;
#pragma unroll
        for (int o = LU_THREADS / 64; o > 0; o >>= 1) {
          double v2 = __shfl_xor_sync(0xffffffffu, v, o);
          int r2 = __shfl_xor_sync(0xffffffffu, r, o);
          better(v, r, v2, r2);
        }
        v = __shfl_sync(0xffffffffu, v, 0);
        rc = __shfl_sync(0xffffffffu, r, 0);
        if (wid == 0) {
          if (lane == 0) {
            p.cand[(par * G + cta) * 2 + 0] = v;
            p.cand[(par * G + cta) * 2 + 1] = (double)rc;
          }
          if (rc != 0x7fffffff) {
            double* row = P + (rc - r0) * LD;
            double* dst = p.prow + ((long long)par * G + cta) * LU_NBMAX;
            const double l = jj > 0 ? row[jj - 1] : 0.0;
            for (int c = jj + lane; c < jb; c += 32) {
              double x = row[c];
              if (jj > 0 && c > jj) {
                x = fma(-l, urow[c], x);
                row[c] = x;  // its pending update, done here instead of in (3)
              }
              dst[c] = x;
            }
          }
          // (2) arrive: the lanes' stores are ordered before thread 0's fence
          __syncwarp();
          if (lane == 0) {
            // release-ordered arrive (cumulative over the warp's stores made
            // visible to lane 0 by the __syncwarp): no separate full fence
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(p.bar) : "memory");
          }
        }
      }
      if (prof) t1 = clock64();
      // (3) pending update of step j-1 on columns jj+1.. (column jj was done in (6))
      if (jj > 0 && jj + 1 < jb) {
        for (int i = tid; i < nr; i += LU_THREADS) {
          if (pivflag[i] >= 0 || r0 + i == rc) continue;
          double* row = P + i * LD;
          const double l = row[jj - 1];
          for (int c = jj + 1; c < jb; ++c) row[c] = fma(-l, urow[c], row[c]);
        }
      }
      // (4) wait: every CTA has arrived for column j
      if (tid == 0) {
        const unsigned target = (unsigned)(j + 1) * (unsigned)G;
        while (ld_acquire_gpu(p.bar) < target) {
        }
      }
      __syncthreads();
      if (prof) t2 = clock64();
      // (5) global winner, same in every CTA
      if (wid == 0) {
        double v = -1.0;
        int r = 0x7fffffff;
        {
          // all of this lane's candidate loads in flight at once (G <= 32 * LU_CPL
          // is enforced by the plan), folded in index order afterwards
          const double2* cp = reinterpret_cast<const double2*>(p.cand) + par * G;
          double2 cr[LU_CPL];
#pragma unroll
          for (int u = 0; u < LU_CPL; ++u) {
            const int c = lane + 32 * u;
            cr[u] = c < G ? __ldcg(cp + c) : make_double2(-1.0, 2147483647.0);
          }
#pragma unroll
          for (int u = 0; u < LU_CPL; ++u) better(v, r, cr[u].x, (int)cr[u].y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          double v2 = __shfl_xor_sync(0xffffffffu, v, o);
          int r2 = __shfl_xor_sync(0xffffffffu, r, o);
          better(v, r, v2, r2);
        }
        if (prof) prof[5] += clock64() - t2;
        const int wc = r / p.rows_per;  // slabs are contiguous
        const double* wrow = p.prow + ((long long)par * G + wc) * LU_NBMAX;
        if (r != 0x7fffffff)
          for (int c = jj + lane; c < jb; c += 32) urow[c] = __ldcg(wrow + c);
        if (prof) prof[6] += clock64() - t2 + (long long)(urow[jj] * 0.0);
        if (lane == 0) {
          win_v = v;
          if (r >= r0 && r < r1 && v >= tol && v != 0.0) pivflag[r - r0] = j;
          if (cta == 0) p.pivrow[j] = r;
        }
      }
      __syncthreads();
      if (!(win_v >= tol) || win_v == 0.0) {
        if (cta == 0 && tid == 0) {
          p.status[0] = (double)j;
          p.status[1] = win_v;
          p.status[2] = tol;
        }
        return;  // uniform across the grid
      }
      if (prof) t3 = clock64();
      // (6) multipliers (LAPACK dgetf2: scale by 1/pivot), column jj+1, next candidate
      const double rpiv = lu_rcp(urow[jj]);
      cbv = -1.0;
      cbr = 0x7fffffff;
      const bool look = jj + 1 < jb;
      for (int i = tid; i < nr; i += LU_THREADS) {
        if (pivflag[i] >= 0) continue;
        double* row = P + i * LD;
        const double l = row[jj] * rpiv;
        row[jj] = l;
        if (look) {
          const double x = fma(-l, urow[jj + 1], row[jj + 1]);
          row[jj + 1] = x;
          better(cbv, cbr, fabs(x), r0 + i);
        }
      }
      if (prof) {
        const long long t4 = clock64();
        prof[0] += t1 - t0;
        prof[1] += t2 - t1;
        prof[2] += t3 - t2;
        prof[3] += t4 - t3;
      }
    }
    __syncthreads();
    // write the panel back
    const long long tp0 = prof ? clock64() : 0;
    for (int e = tid; e < nr * jb; e += LU_THREADS) {
      int i = e / jb, c = e - (e / jb) * jb;
      p.X[(long long)(r0 + i) * p.ldx + J + c] = P[i * LD + c];
    }
    const int rest = p.n - J - jb;
    if (prof && rest <= 0) prof[4] += clock64() - tp0;
    if (rest > 0) {
      grid.sync();
      // the panel's pivot rows (known to every CTA from the winner folds)
      if (tid < jb) pivs[tid] = __ldcg(p.pivrow + J + tid);
      __syncthreads();
      // unit-lower L11 from the pivot rows' multipliers
      for (int e = tid; e < jb * jb; e += LU_THREADS) {
        int a = e / jb, b = e - (e / jb) * jb;
        L11[a * nb + b] = (b < a) ? __ldcg(p.X + (long long)pivs[a] * p.ldx + J + b) : 0.0;
      }
      const long long tu0 = prof ? clock64() : 0;
      for (int c0 = 0; c0 < rest; c0 += p.ch) {
        const int cw = min(p.ch, rest - c0);
        const long long cbase = J + jb + c0;
#pragma unroll 4
        for (int e = tid; e < jb * cw; e += LU_THREADS) {
          int a = e / cw, c = e - (e / cw) * cw;
          U12[a * LDU + c] = __ldcg(p.X + (long long)pivs[a] * p.ldx + cbase + c);
        }
        __syncthreads();
        // U12 = L11^{-1} U12: one column per thread, held in registers
        for (int c = tid; c < cw; c += LU_THREADS) {
          double u[LU_NBMAX];
#pragma unroll
          for (int a = 0; a < LU_NBMAX; ++a) u[a] = a < jb ? U12[a * LDU + c] : 0.0;
#pragma unroll
          for (int a = 1; a < LU_NBMAX; ++a) {
            if (a < jb) {
              double s = u[a];
#pragma unroll
              for (int b = 0; b < a; ++b) s = fma(-L11[a * nb + b], u[b], s);
              u[a] = s;
            }
          }
#pragma unroll
          for (int a = 1; a < LU_NBMAX; ++a)
            if (a < jb) U12[a * LDU + c] = u[a];
        }
        __syncthreads();
        // X[rows, chunk] -= L[rows, panel] U12 on the tensor cores (DMMA
        // m8n8k4): a warp owns 16 rows x 32 columns, its accumulators start
        // as the X tile and go back in place (pivot rows and edges masked)
        {
          const int ntc = (cw + 31) / 32;
          const int ntiles = ((nr + 15) / 16) * ntc;
          const int gid = lane >> 2, tig = lane & 3;
          double nxt[2][4][2];
          auto load_tile = [&](int t, double (&dst)[2][4][2]) {
            const int rb = (t / ntc) * 16, cb = (t % ntc) * 32;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int row = rb + i * 8 + gid;
              const bool lv = row < nr && pivflag[row] < 0;
              const double* xr = p.X + (long long)(r0 + row) * p.ldx + cbase;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int col = cb + j * 8 + 2 * tig;
                if (lv && vec2 && col + 1 < cw) {
                  const double2 v = *reinterpret_cast<const double2*>(xr + col);
                  dst[i][j][0] = v.x;
                  dst[i][j][1] = v.y;
                } else {
                  dst[i][j][0] = (lv && col < cw) ? xr[col] : 0.0;
                  dst[i][j][1] = (lv && col + 1 < cw) ? xr[col + 1] : 0.0;
                }
              }
            }
          };
          if (wid < ntiles) load_tile(wid, nxt);
          for (int t = wid; t < ntiles; t += LU_THREADS / 32) {
            const int rb = (t / ntc) * 16, cb = (t % ntc) * 32;
            double acc[2][4][2];
            bool live[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int row = rb + i * 8 + gid;
              live[i] = row < nr && pivflag[row] < 0;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                acc[i][j][0] = nxt[i][j][0];
                acc[i][j][1] = nxt[i][j][1];
              }
            }
            if (t + LU_THREADS / 32 < ntiles) load_tile(t + LU_THREADS / 32, nxt);  // next tile in flight
            for (int k0 = 0; k0 < jb; k0 += 4) {
              const int k = k0 + tig;
              double af[2], bf[4];
#pragma unroll
              for (int i = 0; i < 2; ++i) af[i] = k < jb ? -P[min(rb + i * 8 + gid, nr - 1) * LD + k] : 0.0;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int col = cb + j * 8 + gid;
                bf[j] = (k < jb && col < cw) ? U12[k * LDU + col] : 0.0;
              }
#pragma unroll
              for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) lu_dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              if (!live[i]) continue;
              double* xr = p.X + (long long)(r0 + rb + i * 8 + gid) * p.ldx + cbase;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int col = cb + j * 8 + 2 * tig;
                if (vec2 && col + 1 < cw) {
                  *reinterpret_cast<double2*>(xr + col) = make_double2(acc[i][j][0], acc[i][j][1]);
                } else {
                  if (col < cw) xr[col] = acc[i][j][0];
                  if (col + 1 < cw) xr[col + 1] = acc[i][j][1];
                }
              }
            }
          }
        }
        __syncthreads();
      }
      if (prof) {
        prof[4] += clock64() - tp0;
        prof[7] += clock64() - tu0;
      }
    }
  }
  // pivot rows: unit entry at their step, zeros to the right
  for (int i = tid; i < nr; i += LU_THREADS) {
    const int j = pivflag[i];
    if (j < 0) continue;
    double* row = p.X + (long long)(r0 + i) * p.ldx;
    row[j] = 1.0;
    for (int c = j + 1; c < p.n; ++c) row[c] = 0.0;
  }
  if (cta == 0 && tid == 0) p.status[0] = -1.0;
}

// ---------------------------------------------------------------------------
// Small blocks (the whole m x n block fits one CTA's shared memory: cfg1 /
// the SVT loop's 1000 x 16 Krylov blocks): one CTA, no grid barrier.  Same
// pivot rule (largest |x| among rows not yet pivoted, ties -> smallest row),
// same reciprocal scaling, same P^T L output and status codes as lu_kernel.
constexpr int LUS_THREADS = 1024;

__global__ void __launch_bounds__(LUS_THREADS) lu_small_kernel(double* X, long long ldx, int m, int n,
                                                              double* status) {
  extern __shared__ double lus[];
  const int LD = n + 1;
  double* P = lus;                                        // m x LD
  int* pivflag = reinterpret_cast<int*>(P + (long long)m * LD);  // m
  __shared__ double rv[LUS_THREADS / 32];
  __shared__ int rr[LUS_THREADS / 32];
  __shared__ double s_v, s_rpiv;
  __shared__ int s_r, s_bad;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double mx = 0.0;
  int nonfin = 0;
  for (int e = tid; e < m * n; e += LUS_THREADS) {
    const int i = e / n, c = e - (e / n) * n;
    const double x = X[(long long)i * ldx + c];
    P[i * LD + c] = x;
    if (!isfinite(x)) nonfin = 1;
    mx = fmax(mx, fabs(x));
  }
  for (int i = tid; i < m; i += LUS_THREADS) pivflag[i] = -1;
  mx = block_max<LUS_THREADS>(mx, rv);
  nonfin = __syncthreads_or(nonfin);
  if (tid == 0) s_v = mx;
  __syncthreads();
  const double maxabs = s_v;
  if (nonfin || maxabs == 0.0) {
    if (tid == 0) status[0] = nonfin ? -3.0 : -2.0;
    return;
  }
  const double tol = 1e-14 * maxabs;
  // candidate for column 0; later columns get theirs from the fused update pass
  double bv = -1.0;
  int br = 0x7fffffff;
  for (int i = tid; i < m; i += LUS_THREADS) better(bv, br, fabs(P[i * LD]), i);
  for (int j = 0; j < n; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int r2 = __shfl_xor_sync(0xffffffffu, br, o);
      better(bv, br, v2, r2);
    }
    if (lane == 0) {
      rv[wid] = bv;
      rr[wid] = br;
    }
    __syncthreads();
    if (wid == 0) {
      double v = lane < LUS_THREADS / 32 ? rv[lane] : -1.0;
      int r = lane < LUS_THREADS / 32 ? rr[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const int r2 = __shfl_xor_sync(0xffffffffu, r, o);
        better(v, r, v2, r2);
      }
      if (lane == 0) {
        s_v = v;
        s_r = r;
        s_bad = !(v >= tol) || v == 0.0;
        if (!s_bad) {
          pivflag[r] = j;
          s_rpiv = lu_rcp(P[r * LD + j]);  // LAPACK dgetf2: scale by 1/pivot
        }
      }
    }
    __syncthreads();
    if (s_bad) {
      if (tid == 0) {
        status[0] = (double)j;
        status[1] = s_v;
        status[2] = tol;
      }
      return;
    }
    const double* up = P + s_r * LD;  // the pivot row (never modified again)
    const double rpiv = s_rpiv;
    // one pass per row: multiplier, trailing update, next column's candidate
    bv = -1.0;
    br = 0x7fffffff;
    for (int i = tid; i < m; i += LUS_THREADS) {
      if (pivflag[i] >= 0) continue;
      double* row = P + i * LD;
      const double l = row[j] * rpiv;
      row[j] = l;
      for (int c = j + 1; c < n; ++c) row[c] = fma(-l, up[c], row[c]);
      if (j + 1 < n) better(bv, br, fabs(row[j + 1]), i);
    }
  }
  __syncthreads();  // the last pass's rows are read by other threads below
  // pivot rows: unit entry at their step, zeros to the right; write back
  for (int e = tid; e < m * n; e += LUS_THREADS) {
    const int i = e / n, c = e - (e / n) * n;
    const int pj = pivflag[i];
    double x = P[i * LD + c];
    if (pj >= 0 && c >= pj) x = (c == pj) ? 1.0 : 0.0;
    X[(long long)i * ldx + c] = x;
  }
  if (tid == 0) status[0] = -1.0;
}

static size_t lu_small_smem(int m, int n) {
  return (size_t)m * (n + 1) * sizeof(double) + (size_t)m * sizeof(int) + 16;
}
constexpr size_t kLuSmallMaxSmem = 200 * 1024;

struct LuPlan {
  int G, nb, ch, rows_per;
  size_t smem;
};

static size_t lu_smem_bytes(int rows_per, int nb, int ch) {
  return (size_t)rows_per * (nb + 1) * 8 + (size_t)nb * (ch + 4) * 8 + (size_t)nb * 8 +
         (size_t)nb * nb * 8 + (size_t)rows_per * 4 + 24;
}

static LuPlan lu_plan(int m, int n) {
  LuPlan pl{};
  const int sms = sm_count();
  // CTAs per SM (tunable: LR_LU_OCC); fewer CTAs = fewer candidates per
  // column and a cheaper barrier, more = less per-column work per CTA
  // One CTA per SM by default: with two (LR_LU_OCC=2, ~17 % faster per call) the factor of a Krylov block was
  // occasionally wrong at block widths 32 / 48 -- 12 of 3000 repetitions, multipliers ~1e5, status "ok" -- and never
  // with one (0 of 7000; profiles/r02bk_bki_determinism.txt).  The cause inside the two-CTA layout is not found yet.
  static const int occ_pref = getenv("LR_LU_OCC") ? (atoi(getenv("LR_LU_OCC")) >= 2 ? 2 : 1) : 1;
  for (int occ = occ_pref; occ >= 1; --occ) {
    // per-CTA dynamic shared memory: an occ-th of the SM's, and never above the kernel's opt-in (220 KB, lu_impl)
    size_t limit = (226 * 1024) / occ - 1024;
    if (limit > 218 * 1024) limit = 218 * 1024;
    int G = sms * occ;
    if (G > 32 * LU_CPL) G = 32 * LU_CPL;
    if (G > (m + 31) / 32) G = (m + 31) / 32;
    if (G < 1) G = 1;
    int rows_per = (m + G - 1) / G;
    G = (m + rows_per - 1) / rows_per;
    // widest panel first (the panel-end update streams the trailing columns
    // once per panel: nb = 32 moves ~2.3x fewer bytes than 16 at n = 110),
    // with the widest U12 chunk that still fits
    for (int nb = LU_NBMAX; nb >= 1; nb >>= 1) {
      int nbe = nb > n ? n : nb;
      for (int ch = LU_CHUNK; ch >= (nb >= 16 ? 32 : 8); ch -= 8) {
        size_t sm = lu_smem_bytes(rows_per, nbe, ch);
        if (sm <= limit) {
          pl.G = G;
          pl.nb = nbe;
          pl.ch = ch;
          pl.rows_per = rows_per;
          pl.smem = sm;
          return pl;
        }
      }
    }
  }
  pl.G = 0;
  return pl;
}

}  // namespace lr

using namespace lr;

extern "C" {

long long lr_lu_workspace_doubles(int m, int n) {
  LuPlan pl = lu_plan(m, n);
  long long G = pl.G > 0 ? pl.G : 1;
  return kCandWords * G + kRowWords * G + n + 8 + lr_stats_partials() + 10;
}

// status_dev (async variant): {code, pivot, tol} with the host wrapper's codes
// (-1 ok, -2 zero matrix, -3 non-finite, j >= 0 first bad column)
__global__ void lu_status_kernel(const double* status, const double* stats, double* out) {
  if (threadIdx.x != 0) return;
  if (stats != nullptr && stats[2] != 0.0) {
    out[0] = -3.0;
  } else if (stats != nullptr && stats[1] == 0.0) {
    out[0] = -2.0;
  } else {
    out[0] = status[0];
    out[1] = status[1];
    out[2] = status[2];
  }
}

static int lu_impl(int m, int n, double* X, long long ldx, double* work, double* status_host, double* status_dev,
                   void* stream);

int lr_lu_pl_f64(int m, int n, double* X, long long ldx, double* work, double* status_host,
                 void* stream) {
  return lu_impl(m, n, X, ldx, work, status_host, nullptr, stream);
}

int lr_lu_pl_async_f64(int m, int n, double* X, long long ldx, double* work, double* status_dev, void* stream) {
  LR_REQUIRE(status_dev != nullptr, "lu_pl_async: status_dev is required");
  return lu_impl(m, n, X, ldx, work, nullptr, status_dev, stream);
}

static int lu_impl(int m, int n, double* X, long long ldx, double* work, double* status_host, double* status_dev,
                   void* stream) {
  LR_REQUIRE(m >= n && n >= 1, "lu_pl requires m >= n, got %dx%d", m, n);
  LR_REQUIRE(ldx >= n, "lu_pl: ldx < n");
  cudaStream_t s = as_stream(stream);
  static const bool no_small = getenv("LR_LU_NO_SMALL") != nullptr;
  if (!no_small && lu_small_smem(m, n) <= kLuSmallMaxSmem) {
    static bool attr_small = false;
    if (!attr_small) {
      LR_CHECK_CUDA(cudaFuncSetAttribute(lu_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kLuSmallMaxSmem));
      attr_small = true;
    }
    double* status = work;
    lu_small_kernel<<<1, LUS_THREADS, lu_small_smem(m, n), s>>>(X, ldx, m, n, status);
    LR_CHECK_LAUNCH();
    if (status_dev) {
      lu_status_kernel<<<1, 32, 0, s>>>(status, nullptr, status_dev);
      LR_CHECK_LAUNCH();
      return LR_OK;
    }
    double host[4];
    LR_CHECK_CUDA(cudaMemcpyAsync(host, status, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    LR_CHECK_CUDA(cudaStreamSynchronize(s));
    status_host[0] = host[0];
    status_host[1] = host[1];
    status_host[2] = host[2];
    return LR_OK;
  }
  LuPlan pl = lu_plan(m, n);
  LR_REQUIRE(pl.G > 0, "lu_pl: %d rows do not fit the cooperative plan", m);
  const long long G = pl.G;
  double* cand = work;
  double* prow = cand + kCandWords * G;
  int* pivrow = reinterpret_cast<int*>(prow + kRowWords * G);
  double* status = work + (kCandWords + kRowWords) * G + n;  // n ints fit in n doubles
  double* stats = status + 4;
  double* partial = stats + 4;
  int st = lr_block_stats_f64(X, m, n, ldx, partial, stats, stream);
  if (st) return st;
  // status zeroed here; the kernel's first act writes status[0] (-1 ok, -2 zero matrix,
  // -3 non-finite, j >= 0 first bad column).  The wrapper reads `stats` before status, so the
  // early exits (zero / non-finite input) never reach the column decision.
  LR_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(double), s));
  static bool attr = false;
  if (!attr) {
    LR_CHECK_CUDA(cudaFuncSetAttribute(lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = true;
  }
  int max_blocks = 0;
  LR_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks, lu_kernel, LU_THREADS, pl.smem));
  LR_REQUIRE((long long)max_blocks * sm_count() >= G, "lu_pl: cooperative grid %lld exceeds residency %d",
             G, max_blocks * sm_count());
  LuParams prm;
  prm.X = X;
  prm.ldx = ldx;
  prm.m = m;
  prm.n = n;
  prm.nb = pl.nb;
  prm.ch = pl.ch;
  prm.rows_per = pl.rows_per;
  prm.stats = stats;
  prm.cand = cand;
  prm.prow = prow;
  prm.pivrow = pivrow;
  prm.status = status;
  static const bool profile = getenv("LR_LU_PROFILE") != nullptr;
  long long* dprof = reinterpret_cast<long long*>(partial + lr_stats_partials());
  prm.prof = profile ? dprof : nullptr;
  if (profile) LR_CHECK_CUDA(cudaMemsetAsync(dprof, 0, 8 * sizeof(long long), s));
  prm.bar = reinterpret_cast<unsigned*>(dprof + 8);  // after the 8 profile slots
  LR_CHECK_CUDA(cudaMemsetAsync(prm.bar, 0, sizeof(unsigned), s));
  void* args[] = {&prm};
  LR_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)lu_kernel, dim3((unsigned)G), dim3(LU_THREADS), args,
                                            pl.smem, s));
  count_launches(1);
  if (profile) {
    long long hp[8];
    LR_CHECK_CUDA(cudaMemcpyAsync(hp, dprof, sizeof(hp), cudaMemcpyDeviceToHost, s));
    LR_CHECK_CUDA(cudaStreamSynchronize(s));
    fprintf(stderr,
            "lu %dx%d G=%lld nb=%d ch=%d cycles/col: local %.0f barrier %.0f winner %.0f (cand %.0f row %.0f) update %.0f; panel ends total %.0f (after barrier %.0f)\n",
            m, n, G, pl.nb, pl.ch, (double)hp[0] / n, (double)hp[1] / n, (double)hp[2] / n, (double)hp[5] / n,
            (double)hp[6] / n, (double)hp[3] / n, (double)hp[4], (double)hp[7]);
  }
  if (status_dev) {
    lu_status_kernel<<<1, 32, 0, s>>>(status, stats, status_dev);
    LR_CHECK_LAUNCH();
    return LR_OK;
  }
  double host[8];
  LR_CHECK_CUDA(cudaMemcpyAsync(host, status, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
  LR_CHECK_CUDA(cudaMemcpyAsync(host + 4, stats, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
  LR_CHECK_CUDA(cudaStreamSynchronize(s));
  if (host[6] != 0.0) {
    status_host[0] = -3.0;
  } else if (host[5] == 0.0) {
    status_host[0] = -2.0;
  } else {
    status_host[0] = host[0];
    status_host[1] = host[1];
    status_host[2] = host[2];
  }
  return LR_OK;
}

}  // extern "C"
