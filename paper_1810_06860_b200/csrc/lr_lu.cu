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
constexpr int LU_CHUNK = 64;  // trailing columns per U12 chunk

struct LuParams {
  double* X;
  long long ldx;
  int m, n, nb, rows_per;
  const double* stats;  // {sumsq, max|x|, nonfinite}
  double* cand;         // [2][G][2]  {|x|, row}
  double* prow;         // [2][G][nb]
  int* pivrow;          // [n]
  double* status;       // {bad col or -1, pivot, tol}
  long long* prof;      // optional per-phase clock totals of CTA 0 (LR_LU_PROFILE)
};

__device__ __forceinline__ void better(double& v, int& r, double v2, int r2) {
  if (v2 > v || (v2 == v && r2 < r)) {
    v = v2;
    r = r2;
  }
}

__global__ void __launch_bounds__(LU_THREADS) lu_kernel(LuParams p) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double lu_smem[];
  const int nb = p.nb, LD = nb + 1;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const int r0 = cta * p.rows_per;
  const int r1 = min(p.m, r0 + p.rows_per);
  const int nr = max(0, r1 - r0);
  double* P = lu_smem;                                   // rows_per x LD
  double* U12 = P + (long long)p.rows_per * LD;          // nb x LU_CHUNK
  double* urow = U12 + nb * LU_CHUNK;                    // nb
  double* L11 = urow + nb;                               // nb x nb
  int* pivflag = reinterpret_cast<int*>(L11 + nb * nb);  // rows_per
  __shared__ double red_v[LU_THREADS / 32];
  __shared__ int red_r[LU_THREADS / 32];
  __shared__ double win_v;
  long long* prof = (blockIdx.x == 0 && threadIdx.x == 0) ? p.prof : nullptr;
  long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  double cbv = -1.0;  // look-ahead candidate for the next column
  int cbr = 0x7fffffff;

  const double maxabs = p.stats[1];
  const double tol = 1e-14 * maxabs;
  if (maxabs == 0.0 || p.stats[2] != 0.0) return;  // handled by the host wrapper
  for (int i = tid; i < nr; i += LU_THREADS) pivflag[i] = -1;
  int par = 0;

  for (int J = 0; J < p.n; J += nb) {
    const int jb = min(nb, p.n - J);
    for (int e = tid; e < nr * jb; e += LU_THREADS) {
      int i = e / jb, c = e - (e / jb) * jb;
      P[i * LD + c] = p.X[(long long)(r0 + i) * p.ldx + J + c];
    }
    __syncthreads();
    for (int jj = 0; jj < jb; ++jj) {
      const int j = J + jj;
      // local argmax among un-pivoted rows
      if (prof) t0 = clock64();
      double bv = -1.0;
      int br = 0x7fffffff;
      if (jj == 0) {
        for (int i = tid; i < nr; i += LU_THREADS)
          if (pivflag[i] < 0) better(bv, br, fabs(P[i * LD + jj]), r0 + i);
      } else {  // found during the previous column's update (look-ahead)
        bv = cbv;
        br = cbr;
      }
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
      if (wid == 0) {
        // CTA candidate: warp 0 folds the per-warp winners and publishes
        // (|x|, row) plus the candidate's panel row (one element per lane)
        double v = (lane < LU_THREADS / 32) ? red_v[lane] : -1.0;
        int r = (lane < LU_THREADS / 32) ? red_r[lane] : 0x7fffffff;
#pragma unroll
        for (int o = LU_THREADS / 64; o > 0; o >>= 1) {
          double v2 = __shfl_xor_sync(0xffffffffu, v, o);
          int r2 = __shfl_xor_sync(0xffffffffu, r, o);
          better(v, r, v2, r2);
        }
        v = __shfl_sync(0xffffffffu, v, 0);
        r = __shfl_sync(0xffffffffu, r, 0);
        if (lane == 0) {
          p.cand[(par * G + cta) * 2 + 0] = v;
          p.cand[(par * G + cta) * 2 + 1] = (double)r;
        }
        if (r != 0x7fffffff)
          for (int c = lane; c < jb; c += 32) p.prow[((long long)par * G + cta) * nb + c] = P[(r - r0) * LD + c];
      }
      if (prof) t1 = clock64();
      grid.sync();
      if (prof) t2 = clock64();
      if (wid == 0) {
        // global winner, same in every CTA: warp 0 alone loads the G
        // candidates (G/32 independent L2 loads per lane), folds them with
        // shuffles and fetches the winner's panel row -- no block-level
        // reduction between the two L2 round trips
        double v = -1.0;
        int r = 0x7fffffff;
        for (int c = lane; c < G; c += 32) {
          const double2 cr = __ldcg(reinterpret_cast<const double2*>(p.cand) + par * G + c);
          better(v, r, cr.x, (int)cr.y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          double v2 = __shfl_xor_sync(0xffffffffu, v, o);
          int r2 = __shfl_xor_sync(0xffffffffu, r, o);
          better(v, r, v2, r2);
        }
        const int wc = r / p.rows_per;  // slabs are contiguous
        const double* wrow = p.prow + ((long long)par * G + wc) * nb;
        for (int c = lane; c < jb; c += 32) urow[c] = __ldcg(wrow + c);
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
      const double rpiv = 1.0 / urow[jj];  // LAPACK dgetf2/dgetrf2: scale by 1/pivot
      cbv = -1.0;
      cbr = 0x7fffffff;
      const bool look = jj + 1 < jb;
      for (int i = tid; i < nr; i += LU_THREADS) {
        if (pivflag[i] >= 0) continue;
        double* row = P + i * LD;
        const double l = row[jj] * rpiv;
        row[jj] = l;
        for (int c = jj + 1; c < jb; ++c) row[c] = fma(-l, urow[c], row[c]);
        if (look) better(cbv, cbr, fabs(row[jj + 1]), r0 + i);
      }
      __syncthreads();
      par ^= 1;
      if (prof) {
        const long long t4 = clock64();
        prof[0] += t1 - t0;
        prof[1] += t2 - t1;
        prof[2] += t3 - t2;
        prof[3] += t4 - t3;
      }
    }
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
      // unit-lower L11 from the pivot rows' multipliers
      for (int e = tid; e < jb * jb; e += LU_THREADS) {
        int a = e / jb, b = e - (e / jb) * jb;
        L11[a * nb + b] = (b < a) ? p.X[(long long)p.pivrow[J + a] * p.ldx + J + b] : 0.0;
      }
      __syncthreads();
      for (int c0 = 0; c0 < rest; c0 += LU_CHUNK) {
        const int cw = min(LU_CHUNK, rest - c0);
        for (int e = tid; e < jb * cw; e += LU_THREADS) {
          int a = e / cw, c = e - (e / cw) * cw;
          U12[a * LU_CHUNK + c] = p.X[(long long)p.pivrow[J + a] * p.ldx + J + jb + c0 + c];
        }
        __syncthreads();
        // forward substitution with the unit-lower L11, parallel over columns
        for (int c = tid; c < cw; c += LU_THREADS)
          for (int a = 1; a < jb; ++a) {
            double s = U12[a * LU_CHUNK + c];
            for (int b = 0; b < a; ++b) s = fma(-L11[a * nb + b], U12[b * LU_CHUNK + c], s);
            U12[a * LU_CHUNK + c] = s;
          }
        __syncthreads();
        // X[rows, chunk] -= L[rows, panel] U12: thread = (column c, row lane);
        // 8 rows per iteration so 8 global loads are in flight per thread
        {
          constexpr int RL = LU_THREADS / LU_CHUNK;  // row lanes
          const int c = tid % LU_CHUNK, rl = tid / LU_CHUNK;
          if (c < cw) {
            for (int ib = rl; ib < nr; ib += RL * 8) {
              double xv[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int i = ib + u * RL;
                xv[u] = (i < nr && pivflag[i] < 0) ? p.X[(long long)(r0 + i) * p.ldx + J + jb + c0 + c] : 0.0;
              }
              for (int a = 0; a < jb; ++a) {
                const double u12 = U12[a * LU_CHUNK + c];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  const int i = min(ib + u * RL, nr - 1);
                  xv[u] = fma(-P[i * LD + a], u12, xv[u]);
                }
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int i = ib + u * RL;
                if (i < nr && pivflag[i] < 0) p.X[(long long)(r0 + i) * p.ldx + J + jb + c0 + c] = xv[u];
              }
            }
          }
        }
        __syncthreads();
      }
      if (prof) prof[4] += clock64() - tp0;
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
          s_rpiv = 1.0 / P[r * LD + j];  // LAPACK dgetf2: scale by 1/pivot
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
  int G, nb, rows_per;
  size_t smem;
};

static size_t lu_smem_bytes(int rows_per, int nb) {
  return (size_t)rows_per * (nb + 1) * 8 + (size_t)nb * LU_CHUNK * 8 + (size_t)nb * 8 +
         (size_t)nb * nb * 8 + (size_t)rows_per * 4 + 16;
}

static LuPlan lu_plan(int m, int n) {
  LuPlan pl{};
  const int sms = sm_count();
  // CTAs per SM (tunable: LR_LU_OCC); fewer CTAs = fewer candidates per
  // column and a cheaper barrier, more = less per-column work per CTA
  static const int occ_pref = getenv("LR_LU_OCC") ? atoi(getenv("LR_LU_OCC")) : 2;
  for (int occ = occ_pref; occ >= 1; --occ) {
    const size_t limit = (226 * 1024) / occ - 1024;
    int G = sms * occ;
    if (G > (m + 31) / 32) G = (m + 31) / 32;
    if (G < 1) G = 1;
    int rows_per = (m + G - 1) / G;
    G = (m + rows_per - 1) / rows_per;
    for (int nb = 32; nb >= 1; nb >>= 1) {
      int nbe = nb > n ? n : nb;
      size_t sm = lu_smem_bytes(rows_per, nbe);
      if (sm <= limit) {
        pl.G = G;
        pl.nb = nbe;
        pl.rows_per = rows_per;
        pl.smem = sm;
        return pl;
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
  return 4 * G + 2 * G * 32 + n + 8 + lr_stats_partials() + 16;
}

int lr_lu_pl_f64(int m, int n, double* X, long long ldx, double* work, double* status_host,
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
  double* prow = cand + 4 * G;
  int* pivrow = reinterpret_cast<int*>(prow + 2 * G * 32);
  double* status = prow + 2 * G * 32 + n;  // n ints fit in n doubles
  double* stats = status + 4;
  double* partial = stats + 4;
  int st = lr_block_stats_f64(X, m, n, ldx, partial, stats, stream);
  if (st) return st;
  LR_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(double), s));
  // status[0] preset to -3 (not run) so an early exit is visible
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
  void* args[] = {&prm};
  LR_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)lu_kernel, dim3((unsigned)G), dim3(LU_THREADS), args,
                                            pl.smem, s));
  count_launches(1);
  if (profile) {
    long long hp[8];
    LR_CHECK_CUDA(cudaMemcpyAsync(hp, dprof, sizeof(hp), cudaMemcpyDeviceToHost, s));
    LR_CHECK_CUDA(cudaStreamSynchronize(s));
    fprintf(stderr,
            "lu %dx%d G=%lld nb=%d cycles/col: local %.0f barrier %.0f winner %.0f update %.0f; panel ends total %.0f\n",
            m, n, G, pl.nb, (double)hp[0] / n, (double)hp[1] / n, (double)hp[2] / n, (double)hp[3] / n,
            (double)hp[4]);
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
