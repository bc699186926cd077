// Sparse kernels of the hot path: SpMM over a row-compressed pattern (CSR for
// Y*X, the persistent CSC copy for Y^T*X), the sampled dense-dense product,
// and the fused SVT step (SDDMM + residual + in-place update of both copies).
//
// Roofline: these are gathers of dense rows (w or r doubles per stored entry)
// that live in L2 (the dense operands of every BASELINE config fit in the
// 126 MB L2), plus a compulsory HBM stream of 12 B/nnz (SpMM) or 40 B/nnz
// (SVT step).  Work is split into "items" (a row, or a chunk of a long row)
// so Zipf-shaped rows (cfg4: up to 26,744 entries) do not serialize a warp.
#include <stdio.h>
#include <stdlib.h>

#include "lr_common.cuh"

namespace lr {

struct Item {
  int row, beg, end, slot;
};

__device__ __forceinline__ Item load_item(const int* __restrict__ items, const int* __restrict__ ptr,
                                          int i) {
  Item it;
  if (items) {
    int4 v = reinterpret_cast<const int4*>(items)[i];
    it.row = v.x;
    it.beg = v.y;
    it.end = v.z;
    it.slot = v.w;
  } else {
    it.row = i;
    it.beg = __ldg(ptr + i);
    it.end = __ldg(ptr + i + 1);
    it.slot = -1;
  }
  return it;
}

// ------------------------------------------------------------------- SpMM
// Scalar traits: the fp64 path moves double2 (16 B) per lane and column
// pair, the optional fp32 path (north_star "fp32 mode") float2 (8 B), so
// every gathered row costs half the L2 bytes.
template <typename Sc>
struct Vec2T;
template <>
struct Vec2T<double> {
  using type = double2;
  static __device__ __forceinline__ double2 make(double a, double b) { return make_double2(a, b); }
};
template <>
struct Vec2T<float> {
  using type = float2;
  static __device__ __forceinline__ float2 make(float a, float b) { return make_float2(a, b); }
};

// A group of G lanes owns one item; lane g covers column pairs
// c = 2*(g + G*t), t < T, of a column tile of width 2*G*T starting at c0.
// VEC2: double2 loads/stores (requires 16B-aligned rows); tail columns scalar.
// Q: stored entries per lane kept in flight (4; 8 for one-pair-per-lane
// narrow products, whose gathers are too small to cover the L2 latency)
#ifndef LR_SPMM_MINB
#define LR_SPMM_MINB 4
#endif
template <int G, int T, bool VEC2, int Q = 4, typename Sc = double>
__global__ void __launch_bounds__(256, LR_SPMM_MINB) spmm_kernel(const int* __restrict__ ptr,
                                                   const int* __restrict__ idx,
                                                   const Sc* __restrict__ val,
                                                   const int* __restrict__ items, int n_items,
                                                   const Sc* __restrict__ X, long long ldx, int w,
                                                   Sc* __restrict__ Y, long long ldy,
                                                   Sc* __restrict__ scratch, int n_tiles) {
  using V2 = typename Vec2T<Sc>::type;
  constexpr int GROUPS = 32 / G;
  constexpr int TILE = 2 * G * T;  // columns per tile
  const int lane = threadIdx.x & 31;
  const int g = lane % G;
  const int grp = lane / G;
  const long long warp_global = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long n_units = (long long)((n_items + GROUPS - 1) / GROUPS) * n_tiles;

  for (long long u = warp_global; u < n_units; u += n_warps) {
    const int tile = (int)(u % n_tiles);
    const int item_i = (int)(u / n_tiles) * GROUPS + grp;
    const bool active = item_i < n_items;
    Item it{0, 0, 0, -1};
    if (active) it = load_item(items, ptr, item_i);
    const int c0 = tile * TILE;
    V2 acc[T];
#pragma unroll
    for (int t = 0; t < T; ++t) acc[t] = Vec2T<Sc>::make(Sc(0), Sc(0));

    if (active) {
      int e = it.beg;
      // process Q entries per step for memory-level parallelism
      for (; e + Q <= it.end; e += Q) {
        int cj[Q];
        Sc vj[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          cj[q] = __ldg(idx + e + q);
          vj[q] = __ldg(val + e + q);
        }
        V2 xv[Q][T];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const Sc* xr = X + (long long)cj[q] * ldx + c0;
#pragma unroll
          for (int t = 0; t < T; ++t) {
            const int c = 2 * (g + G * t);
            if (VEC2 && c0 + c + 1 < w) {
              xv[q][t] = __ldg(reinterpret_cast<const V2*>(xr + c));
            } else {
              xv[q][t].x = (c0 + c < w) ? __ldg(xr + c) : Sc(0);
              xv[q][t].y = (c0 + c + 1 < w) ? __ldg(xr + c + 1) : Sc(0);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
          for (int t = 0; t < T; ++t) {
            acc[t].x = fma(vj[q], xv[q][t].x, acc[t].x);
            acc[t].y = fma(vj[q], xv[q][t].y, acc[t].y);
          }
      }
      for (; e < it.end; ++e) {
        const int cj = __ldg(idx + e);
        const Sc vj = __ldg(val + e);
        const Sc* xr = X + (long long)cj * ldx + c0;
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int c = 2 * (g + G * t);
          V2 xv;
          if (VEC2 && c0 + c + 1 < w) {
            xv = __ldg(reinterpret_cast<const V2*>(xr + c));
          } else {
            xv.x = (c0 + c < w) ? __ldg(xr + c) : Sc(0);
            xv.y = (c0 + c + 1 < w) ? __ldg(xr + c + 1) : Sc(0);
          }
          acc[t].x = fma(vj, xv.x, acc[t].x);
          acc[t].y = fma(vj, xv.y, acc[t].y);
        }
      }
      Sc* dst = (it.slot >= 0) ? (scratch + (long long)it.slot * w + c0)
                                   : (Y + (long long)it.row * ldy + c0);
      const bool dst_vec = VEC2 && (it.slot < 0 || (w % 2 == 0));
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int c = 2 * (g + G * t);
        if (dst_vec && c0 + c + 1 < w) {
          *reinterpret_cast<V2*>(dst + c) = acc[t];
        } else {
          if (c0 + c < w) dst[c] = acc[t].x;
          if (c0 + c + 1 < w) dst[c + 1] = acc[t].y;
        }
      }
    }
  }
}

// sum partial rows of split items, in slot order
template <typename Sc>
__global__ void spmm_split_reduce_kernel(const int* __restrict__ splits, int n_splits,
                                         const Sc* __restrict__ scratch, int w,
                                         Sc* __restrict__ Y, long long ldy) {
  const long long total = (long long)n_splits * w;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(t / w), c = (int)(t - (long long)s * w);
    const int4 sp = reinterpret_cast<const int4*>(splits)[s];
    // the partial rows are added in slot order (a fixed, sequential sum); the loads do not
    // depend on the sum, so 16 of them are in flight at a time (a Zipf-hot column of cfg4 has
    // ~200 slots: one L2 round trip per slot otherwise)
    Sc acc = Sc(0);
    int k = sp.y;
    for (; k + 16 <= sp.z; k += 16) {
      Sc v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldg(scratch + (long long)(k + u) * w + c);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc += v[u];
    }
    for (; k < sp.z; ++k) acc += __ldg(scratch + (long long)k * w + c);
    Y[(long long)sp.x * ldy + c] = acc;
  }
}

// SpMV (w == 1): one warp per item, lanes stride the entries, tree-reduce.
__global__ void __launch_bounds__(256) spmv_kernel(const int* __restrict__ ptr,
                                                   const int* __restrict__ idx,
                                                   const double* __restrict__ val,
                                                   const int* __restrict__ items, int n_items,
                                                   const double* __restrict__ X, long long ldx,
                                                   double* __restrict__ Y, long long ldy,
                                                   double* __restrict__ scratch) {
  const int lane = threadIdx.x & 31;
  const long long warp_global = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long i = warp_global; i < n_items; i += n_warps) {
    Item it = load_item(items, ptr, (int)i);
    double acc = 0.0;
    for (int e = it.beg + lane; e < it.end; e += 32)
      acc = fma(__ldg(val + e), __ldg(X + (long long)__ldg(idx + e) * ldx), acc);
    acc = warp_sum(acc);
    if (lane == 0) {
      if (it.slot >= 0)
        scratch[it.slot] = acc;
      else
        Y[(long long)it.row * ldy] = acc;
    }
  }
}

// --------------------------------------------------------------- SDDMM / SVT
// One warp per item; the item's row of U*S is staged in shared memory
// (broadcast reads); each lane owns one stored entry at a time and walks the
// r columns of V[j,:] with double2 loads.
constexpr int kSvtThreads = 256;
constexpr int kSvtBlocksPerSm = 4;
constexpr int kMaxRankSmem = 1024;  // per-warp staging of U*S (doubles)

template <bool FUSED, bool VEC2>
__global__ void __launch_bounds__(kSvtThreads) sddmm_kernel(
    const int* __restrict__ ptr, const int* __restrict__ idx, const int* __restrict__ items,
    int n_items, const double* __restrict__ U, long long ldu, const double* __restrict__ S,
    const double* __restrict__ V, long long ldv, int r, double* __restrict__ x_out,
    const double* __restrict__ m_vals, double* __restrict__ y_csr, double* __restrict__ y_csc,
    const int* __restrict__ inv_perm, double step, int apply, double* __restrict__ partial) {
  extern __shared__ double sh_us[];  // (threads/32) * r
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* us = sh_us + wib * r;
  const long long warp_global = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  double ss = 0.0, mx = 0.0;
  for (long long i = warp_global; i < n_items; i += n_warps) {
    Item it = load_item(items, ptr, (int)i);
    __syncwarp();
    for (int t = lane; t < r; t += 32) us[t] = U[(long long)it.row * ldu + t] * S[t];
    __syncwarp();
    for (int e = it.beg + lane; e < it.end; e += 32) {
      const int j = __ldg(idx + e);
      const double* vr = V + (long long)j * ldv;
      double acc = 0.0;
      int t = 0;
      if (VEC2) {
        for (; t + 1 < r; t += 2) {
          double2 v2 = __ldg(reinterpret_cast<const double2*>(vr + t));
          acc = fma(us[t], v2.x, acc);
          acc = fma(us[t + 1], v2.y, acc);
        }
      }
      for (; t < r; ++t) acc = fma(us[t], __ldg(vr + t), acc);
      if (FUSED) {
        const double mv = __ldg(m_vals + e);
        const double d = acc - mv;
        ss = fma(d, d, ss);
        mx = fmax(mx, fabs(d));
        if (apply) {
          // Y.data += step * (m - x): same rounding sequence as numpy
          const double ynew = add_rn(y_csr[e], mul_rn(step, add_rn(mv, -acc)));
          y_csr[e] = ynew;
          y_csc[__ldg(inv_perm + e)] = ynew;
        }
      } else {
        x_out[e] = acc;
      }
    }
  }
  if (FUSED) {
    double S2 = block_sum<kSvtThreads>(ss, red);
    double M2 = block_max<kSvtThreads>(mx, red);
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = S2;
      partial[2 * blockIdx.x + 1] = M2;
    }
  }
}

// Group variant (r <= 256): G lanes per item share one CSR row, lane g holds
// the U*S values of its column pairs in registers and gathers the matching
// slice of each V row (one coalesced read of 8r bytes per entry per group
// instead of 32 lanes each walking a different V row); the G partial dots are
// folded with a fixed xor-butterfly and lane 0 of the group finishes the
// entry.  Q entries in flight per group.  Every entry's value depends only on
// (U row, S, V row): the sharded engine's two value copies stay identical.
template <int G, int T, bool FUSED, int Q = 4>
__global__ void __launch_bounds__(kSvtThreads) svt_group_kernel(
    const int* __restrict__ ptr, const int* __restrict__ idx, const int* __restrict__ items, int n_items,
    const double* __restrict__ U, long long ldu, const double* __restrict__ S, const double* __restrict__ V,
    long long ldv, int r, double* __restrict__ x_out, const double* __restrict__ m_vals,
    double* __restrict__ y_csr, double* __restrict__ y_csc, const int* __restrict__ inv_perm, double step,
    int apply, double* __restrict__ partial) {
  constexpr int GROUPS = 32 / G;
  const int lane = threadIdx.x & 31, g = lane % G, grp = lane / G;
  // groups of a warp walk items of different lengths: shuffles name only their own group
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  const long long warp_global = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long n_units = (n_items + GROUPS - 1) / GROUPS;
  double ss = 0.0, mx = 0.0;
  for (long long u = warp_global; u < n_units; u += n_warps) {
    const int item_i = (int)u * GROUPS + grp;
    if (item_i >= n_items) continue;  // group-uniform
    const Item it = load_item(items, ptr, item_i);
    double2 us[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int c = 2 * (g + G * t);
      const double* ur = U + (long long)it.row * ldu;
      us[t].x = (c < r) ? ur[c] * S[c] : 0.0;
      us[t].y = (c + 1 < r) ? ur[c + 1] * S[c + 1] : 0.0;
    }
    for (int e0 = it.beg; e0 < it.end; e0 += Q) {
      double part[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        part[q] = 0.0;
        const int e = e0 + q;
        if (e < it.end) {
          const double* vr = V + (long long)__ldg(idx + e) * ldv;
#pragma unroll
          for (int t = 0; t < T; ++t) {
            const int c = 2 * (g + G * t);
            double2 v;
            if (c + 1 < r) {
              v = __ldg(reinterpret_cast<const double2*>(vr + c));
            } else {
              v.x = (c < r) ? __ldg(vr + c) : 0.0;
              v.y = 0.0;
            }
            part[q] = fma(us[t].x, v.x, part[q]);
            part[q] = fma(us[t].y, v.y, part[q]);
          }
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < Q; ++q) part[q] += __shfl_xor_sync(gmask, part[q], o);
      if (g == 0) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int e = e0 + q;
          if (e >= it.end) break;
          const double acc = part[q];
          if (FUSED) {
            const double mv = __ldg(m_vals + e);
            const double d = acc - mv;
            ss = fma(d, d, ss);
            mx = fmax(mx, fabs(d));
            if (apply) {
              const double ynew = add_rn(y_csr[e], mul_rn(step, add_rn(mv, -acc)));
              y_csr[e] = ynew;
              y_csc[__ldg(inv_perm + e)] = ynew;
            }
          } else {
            x_out[e] = acc;
          }
        }
      }
    }
  }
  if (FUSED) {
    __shared__ double red[32];
    const double S2 = block_sum<kSvtThreads>(ss, red);
    const double M2 = block_max<kSvtThreads>(mx, red);
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = S2;
      partial[2 * blockIdx.x + 1] = M2;
    }
  }
}

// Batch variant (any rank): a warp owns one item and walks it in batches of
// 32 consecutive stored entries.  Lane l loads entry b0 + l's column, M value
// and Y value with one coalesced access each; the dots run in rounds, a group
// of G lanes per entry (lane g holds U*S of its column pairs c = 2(g + G t) in
// registers and reads the matching 16-byte slices of V[j,:], so every V row is
// read as G*16 contiguous bytes), Q rounds of gathers in flight; a fixed
// xor-butterfly folds the G partials and one shuffle hands entry q's value to
// lane q, which finishes it (residual partials, Y += step (m - x), coalesced
// store; the CSC copy's scattered store only when y_csc is given).  Ranks
// wider than 2 G T run as column chunks with the x partials summed in chunk
// order.
template <int G, int T, int Q, bool FUSED>
__global__ void __launch_bounds__(kSvtThreads) svt_batch_kernel(
    const int* __restrict__ ptr, const int* __restrict__ idx, const int* __restrict__ items, int n_items,
    const double* __restrict__ U, long long ldu, const double* __restrict__ S, const double* __restrict__ V,
    long long ldv, int r, double* __restrict__ x_out, const double* __restrict__ m_vals,
    double* __restrict__ y_csr, double* __restrict__ y_csc, const int* __restrict__ inv_perm, double step,
    int apply, double* __restrict__ partial) {
  constexpr int E = 32 / G;  // entries per round
  constexpr int CH = 2 * G * T;  // rank columns per chunk
  const int lane = threadIdx.x & 31, g = lane % G, grp = lane / G;
  const long long warp_global = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0);
  double ss = 0.0, mx = 0.0;
  for (long long ii = warp_global; ii < n_items; ii += n_warps) {
    const Item it = load_item(items, ptr, (int)ii);
    const double* ur = U + (long long)it.row * ldu;
    for (int b0 = it.beg; b0 < it.end; b0 += 32) {
      const int nE = min(32, it.end - b0);
      const int e = b0 + lane;
      const bool own = lane < nE;
      const int jl = own ? __ldg(idx + e) : 0;
      double ml = 0.0, yl = 0.0;
      if (FUSED && own) {
        ml = __ldg(m_vals + e);
        if (apply) yl = y_csr[e];
      }
      double xl = 0.0;
      const int rounds = (nE + E - 1) / E;
      for (int c0 = 0; c0 < r; c0 += CH) {
        double2 us[T];
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int c = c0 + 2 * (g + G * t);
          us[t].x = (c < r) ? __ldg(ur + c) * __ldg(S + c) : 0.0;
          us[t].y = (c + 1 < r) ? __ldg(ur + c + 1) * __ldg(S + c + 1) : 0.0;
        }
        for (int rho0 = 0; rho0 < rounds; rho0 += Q) {
          double part[Q];
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            part[q] = 0.0;
            const int ent = (rho0 + q) * E + grp;  // entry of this group in round rho0 + q
            const int j = __shfl_sync(0xffffffffu, jl, ent & 31);
            if (ent < nE) {
              const double* vr = V + (long long)j * ldv + c0;
#pragma unroll
              for (int t = 0; t < T; ++t) {
                const int c = 2 * (g + G * t);
                double2 v;
                if (vec && c0 + c + 1 < r) {
                  v = __ldg(reinterpret_cast<const double2*>(vr + c));
                } else {
                  v.x = (c0 + c < r) ? __ldg(vr + c) : 0.0;
                  v.y = (c0 + c + 1 < r) ? __ldg(vr + c + 1) : 0.0;
                }
                part[q] = fma(us[t].x, v.x, part[q]);
                part[q] = fma(us[t].y, v.y, part[q]);
              }
            }
          }
#pragma unroll
          for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
            for (int q = 0; q < Q; ++q) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
          // hand entry (rho0 + q) * E + grp's value to the lane that owns it
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const double v = __shfl_sync(0xffffffffu, part[q], (lane % E) * G);
            if (lane / E == rho0 + q) xl += v;
          }
        }
      }
      if (own) {
        if (FUSED) {
          const double d = xl - ml;
          ss = fma(d, d, ss);
          mx = fmax(mx, fabs(d));
          if (apply) {
            const double ynew = add_rn(yl, mul_rn(step, add_rn(ml, -xl)));
            y_csr[e] = ynew;
            if (y_csc) y_csc[__ldg(inv_perm + e)] = ynew;
          }
        } else {
          x_out[e] = xl;
        }
      }
    }
  }
  if (FUSED) {
    __shared__ double red[32];
    const double S2 = block_sum<kSvtThreads>(ss, red);
    const double M2 = block_max<kSvtThreads>(mx, red);
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = S2;
      partial[2 * blockIdx.x + 1] = M2;
    }
  }
}

// Flat variant (the default): the stored entries are cut into tiles of 32*K
// consecutive CSR slots, one warp per tile (uniform work per warp whatever
// the row lengths -- cfg4 rows run from 10 to 8,344 entries).  Lane l owns
// slots base + 32k + l (k < K): one coalesced load each of the column index,
// M value and Y value, all K in flight together.  The row of every slot comes
// from the tile's first row (tile_row[], one binary search per tile per
// pattern) and a warp-wide count of the row boundaries ptr[] at or below the
// slot.  The tile's (column, row) pairs go to shared memory; the dots then
// run in rounds with a group of G lanes per entry (lane g multiplies its T
// column pairs c = 2(g + G t) of U[row,:] * S by the matching 16-byte slices
// of V[j,:], so every V row is read as G*16 contiguous bytes), Q rounds of
// gathers in flight, a fixed xor-butterfly per group, the result parked in
// shared memory; each lane then finishes its own K slots with coalesced
// stores.  Ranks wider than 2 G T run as column chunks (x partials summed in
// chunk order).  Per entry the sum is fixed by (U row, S, V row) alone.
constexpr int kFlatWarps = 8;

template <int G, int T, int K, int Q, bool FUSED>
__global__ void __launch_bounds__(kFlatWarps * 32) svt_flat_kernel(
    const int* __restrict__ ptr, const int* __restrict__ idx, long long nnz, int m,
    const int* __restrict__ tile_row, long long n_tiles, const double* __restrict__ U, long long ldu,
    const double* __restrict__ S, const double* __restrict__ V, long long ldv, int r, double* __restrict__ x_out,
    const double* __restrict__ m_vals, double* __restrict__ y_csr, double* __restrict__ y_csc,
    const int* __restrict__ inv_perm, double step, int apply, double* __restrict__ partial) {
  constexpr int E = 32 / G;    // entries per round
  constexpr int TE = 32 * K;   // entries per tile
  constexpr int CH = 2 * G * T;  // rank columns per chunk
  constexpr int ROUNDS = TE / E;
  __shared__ int2 sh_jr[kFlatWarps][TE];
  __shared__ double sh_x[kFlatWarps][TE];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, g = lane % G, grp = lane / G;
  const long long warp_global = (long long)blockIdx.x * kFlatWarps + wib;
  const long long n_warps = (long long)gridDim.x * kFlatWarps;
  const bool vec = ((ldv & 1) == 0) && ((ldu & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(U) & 15) == 0);
  int2* jr = sh_jr[wib];
  double* xs = sh_x[wib];
  double ss = 0.0, mx = 0.0;
  for (long long t = warp_global; t < n_tiles; t += n_warps) {
    const long long base = t * TE;
    const long long last = min(base + TE, nnz) - 1;
    int jk[K], rk[K];
    double mk[K], yk[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const long long e = base + 32 * k + lane;
      const bool own = e <= last;
      jk[k] = own ? __ldg(idx + e) : 0;
      mk[k] = (FUSED && own) ? __ldg(m_vals + e) : 0.0;
      yk[k] = (FUSED && own && apply) ? y_csr[e] : 0.0;
    }
    // rows: r0 + #{row boundaries ptr[r0+1..] <= slot}
    const int r0 = __ldg(tile_row + t);
#pragma unroll
    for (int k = 0; k < K; ++k) rk[k] = r0;
    for (int rb = r0;; rb += 32) {
      const int bi = rb + 1 + lane;
      const long long b = (bi <= m) ? (long long)__ldg(ptr + bi) : (1LL << 62);
#pragma unroll 8
      for (int i = 0; i < 32; ++i) {
        const long long bv = __shfl_sync(0xffffffffu, b, i);
#pragma unroll
        for (int k = 0; k < K; ++k) rk[k] += (bv <= base + 32 * k + lane) ? 1 : 0;
      }
      if (__shfl_sync(0xffffffffu, b, 31) > last) break;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) jr[32 * k + lane] = make_int2(jk[k], rk[k]);
    __syncwarp();
    const int nE = (int)(last - base + 1);
    for (int c0 = 0; c0 < r; c0 += CH) {
      double2 sv[T];
#pragma unroll
      for (int tt = 0; tt < T; ++tt) {
        const int c = c0 + 2 * (g + G * tt);
        sv[tt].x = (c < r) ? __ldg(S + c) : 0.0;
        sv[tt].y = (c + 1 < r) ? __ldg(S + c + 1) : 0.0;
      }
      for (int rho0 = 0; rho0 < ROUNDS; rho0 += Q) {
        double part[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          part[q] = 0.0;
          const int ent = (rho0 + q) * E + grp;
          if (ent < nE) {
            const int2 e2 = jr[ent];
            const double* vr = V + (long long)e2.x * ldv + c0;
            const double* ur = U + (long long)e2.y * ldu + c0;
#pragma unroll
            for (int tt = 0; tt < T; ++tt) {
              const int c = 2 * (g + G * tt);
              double2 v, u;
              if (vec && c0 + c + 1 < r) {
                v = __ldg(reinterpret_cast<const double2*>(vr + c));
                u = __ldg(reinterpret_cast<const double2*>(ur + c));
              } else {
                v.x = (c0 + c < r) ? __ldg(vr + c) : 0.0;
                v.y = (c0 + c + 1 < r) ? __ldg(vr + c + 1) : 0.0;
                u.x = (c0 + c < r) ? __ldg(ur + c) : 0.0;
                u.y = (c0 + c + 1 < r) ? __ldg(ur + c + 1) : 0.0;
              }
              part[q] = fma(u.x * sv[tt].x, v.x, part[q]);
              part[q] = fma(u.y * sv[tt].y, v.y, part[q]);
            }
          }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
          for (int q = 0; q < Q; ++q) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
        if (g == 0) {
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const int ent = (rho0 + q) * E + grp;
            if (ent < TE) xs[ent] = (c0 == 0) ? part[q] : xs[ent] + part[q];
          }
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const long long e = base + 32 * k + lane;
      if (e > last) continue;
      const double xl = (r > 0) ? xs[32 * k + lane] : 0.0;
      if (FUSED) {
        const double d = xl - mk[k];
        ss = fma(d, d, ss);
        mx = fmax(mx, fabs(d));
        if (apply) {
          const double ynew = add_rn(yk[k], mul_rn(step, add_rn(mk[k], -xl)));
          y_csr[e] = ynew;
          if (y_csc) y_csc[__ldg(inv_perm + e)] = ynew;
        }
      } else {
        x_out[e] = xl;
      }
    }
    __syncwarp();
  }
  if (FUSED) {
    __shared__ double red[32];
    const double S2 = block_sum<kFlatWarps * 32>(ss, red);
    const double M2 = block_max<kFlatWarps * 32>(mx, red);
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = S2;
      partial[2 * blockIdx.x + 1] = M2;
    }
  }
}

// tile_row[t] = the row holding CSR slot t * tile_entries (binary search in ptr)
__global__ void tile_rows_kernel(const int* __restrict__ ptr, int m, long long nnz, int tile_entries,
                                 long long n_tiles, int* __restrict__ tile_row) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles;
       t += (long long)gridDim.x * blockDim.x) {
    const long long e = t * tile_entries;
    int lo = 0, hi = m - 1;  // last row with ptr[row] <= e
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((long long)ptr[mid] <= e) lo = mid; else hi = mid - 1;
    }
    tile_row[t] = lo;
  }
}

// one warp: lane-strided partial sums, fixed shuffle tree (deterministic; a
// single-thread serial fold over the ~1.2K block partials cost ~45 us per
// SVT iteration)
__global__ void svt_finish_kernel(const double* partial, int n, double* out2) {
  const int lane = threadIdx.x;
  if (lane >= 32) return;
  double s = 0.0, m = 0.0;
  for (int i = lane; i < n; i += 32) {
    s += partial[2 * i];
    m = fmax(m, partial[2 * i + 1]);
  }
  s = warp_sum(s);
  m = warp_max(m);
  if (lane == 0) {
    out2[0] = s;
    out2[1] = m;
  }
}

__global__ void pattern_axpy_kernel(double* __restrict__ y_csr, double* __restrict__ y_csc,
                                    const int* __restrict__ inv_perm,
                                    const double* __restrict__ delta, double alpha, long long nnz) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
       e += (long long)gridDim.x * blockDim.x) {
    const double d = (alpha == 1.0) ? delta[e] : alpha * delta[e];
    const double ynew = add_rn(y_csr[e], d);
    y_csr[e] = ynew;
    if (y_csc) y_csc[inv_perm[e]] = ynew;
  }
}

// ------------------------------------------------- line-aligned group kernels
// The gathers of both sparse products are bound by the L1 data pipe, not by
// L2 or HBM (ncu, cfg4 w = 22: L1 wavefronts 82 % of peak, L2 44 %, DRAM
// 10 %; profiles/r02f_*): a warp load costs one wavefront per distinct
// 128-byte line it touches.  These kernels therefore
//   * read every gathered row as whole aligned 16-byte chunks starting at the
//     row's 128-byte line (lane g of a G-lane group owns chunks g + G t,
//     t < T; `shift` = the elements between the line start and column 0), so
//     an aligned row of b bytes costs ceil(b / 128) wavefronts;
//   * load the stored entries' column index / value (and M, Y) as coalesced
//     per-group batches of 32 consecutive entries (one HBM round trip per 32
//     entries instead of a broadcast load per entry);
//   * keep each G-lane group on its own sequence of work items (grid-stride
//     per group; the warp runs until its last group is done), so Zipf-length
//     rows do not idle the other groups of a warp.
// Over-reads stay inside the allocation: the first chunk starts at the
// 128-byte line of column 0 (CUDA allocations are >= 256-byte aligned) and
// the last ends at the next 16-byte boundary of the row.
template <typename Sc>
struct Chunk16;
template <>
struct Chunk16<double> {
  using type = double2;
  static constexpr int VE = 2;
  static __device__ __forceinline__ void fma_into(double v, const double2& x, double2& a) {
    a.x = fma(v, x.x, a.x);
    a.y = fma(v, x.y, a.y);
  }
  static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ double get(const double2& c, int i) { return i == 0 ? c.x : c.y; }
};
template <>
struct Chunk16<float> {
  using type = float4;
  static constexpr int VE = 4;
  static __device__ __forceinline__ void fma_into(float v, const float4& x, float4& a) {
    a.x = fmaf(v, x.x, a.x);
    a.y = fmaf(v, x.y, a.y);
    a.z = fmaf(v, x.z, a.z);
    a.w = fmaf(v, x.w, a.w);
  }
  static __device__ __forceinline__ float4 zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
  static __device__ __forceinline__ float get(const float4& c, int i) {
    return i == 0 ? c.x : (i == 1 ? c.y : (i == 2 ? c.z : c.w));
  }
};

constexpr int kGroupBatch = 32;  // stored entries per group batch
// build-time tuning of the group kernels (tools/r02/group_variants.sh)
#ifndef LR_GRP_MINB
#define LR_GRP_MINB 2
#endif
#ifndef LR_SVT_MINB
#define LR_SVT_MINB 3  // r02k sweep: 3 CTAs/SM beat 2 at every rank (r = 48: 1.48 -> 1.19 ms)
#endif
#ifndef LR_SPMM_QLO
#define LR_SPMM_QLO 8
#endif
#ifndef LR_SPMM_QHI
#define LR_SPMM_QHI 4
#endif
#ifndef LR_SVT_Q1
#define LR_SVT_Q1 8
#endif
#ifndef LR_SVT_Q2
#define LR_SVT_Q2 4
#endif
#ifndef LR_SVT_Q3
#define LR_SVT_Q3 2
#endif

// Y (rows x w) = A X over a row-compressed pattern, w <= G T VE - shift.
// Per output element the entries are accumulated in storage order (fma), as
// in the item kernel above: results are bit-identical to it.
//
// HOT (shared-memory staging of the block rows a skewed pattern gathers most):
// the index stream holds -(rank + 1) for the hot_max most frequent indices
// (rank by occurrence count, ties by index) and the plain index otherwise;
// the CTA stages the packed chunks of the H most frequent rows of X (gathered
// into `hot.buf` by hot_rows_kernel) into shared memory with one TMA bulk copy
// (cp.async.bulk + mbarrier) while its first index batches are in flight, and
// every gather of a rank < H reads shared memory instead of L2 (cfg4's Zipf
// columns: the 1280 hottest of 26,744 carry ~60 % of the stored entries).
// Ranks in [H, hot_max) look the index up in `order`.  The staged chunks are
// copies of the chunks the plain kernel loads, the lane map and the summation
// order are the same: results are bit-identical to the plain kernel.
struct HotRows {
  const void* buf;   // H x nchunk 16-byte chunks, packed (global)
  const int* order;  // rank -> index, hot_max entries
  int H, nchunk;
};

__device__ __forceinline__ unsigned hot_smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

constexpr int kHotThreads = 512;           // one CTA per SM owns the whole shared memory
constexpr int kHotSmemBytes = 220 * 1024;  // staged rows (227 KB per CTA less the barrier / reserved)
constexpr int kHotMaxRows = 4096;          // ranks encoded in the index stream

template <typename CT>
__global__ void hot_rows_kernel(const CT* __restrict__ Xs, long long ld_chunks, const int* __restrict__ order,
                                int H, int nchunk, CT* __restrict__ buf) {
  const long long total = (long long)H * nchunk;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(i / nchunk), k = (int)(i - (long long)s * nchunk);
    buf[i] = __ldg(Xs + (long long)__ldg(order + s) * ld_chunks + k);
  }
}

template <int G, int T, int Q, typename Sc, bool HOT = false>
__global__ void __launch_bounds__(HOT ? kHotThreads : 256, HOT ? 1 : LR_GRP_MINB) spmm_group_kernel(
    const int* __restrict__ ptr, const int* __restrict__ idx, const Sc* __restrict__ val,
    const int* __restrict__ items, int n_items, const Sc* __restrict__ X, long long ldx, int w, int shift,
    Sc* __restrict__ Y, long long ldy, Sc* __restrict__ scratch, HotRows hot = HotRows{nullptr, nullptr, 0, 0}) {
  using C = Chunk16<Sc>;
  using CT = typename C::type;
  constexpr int VE = C::VE;
  constexpr int GROUPS = 32 / G;
  constexpr int KB = kGroupBatch / G;  // batch entries per lane
  extern __shared__ __align__(128) unsigned char lr_hot_smem[];  // [0, 128): the barrier; rows behind it
  unsigned long long& hot_bar = *reinterpret_cast<unsigned long long*>(lr_hot_smem);
  if constexpr (HOT) {
    const unsigned bytes = (unsigned)hot.H * (unsigned)hot.nchunk * 16u;
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(hot_smem_u32(&hot_bar)));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(hot_smem_u32(&hot_bar)),
                   "r"(bytes)
                   : "memory");
      for (unsigned off = 0; off < bytes; off += 32768u) {
        const unsigned sz = bytes - off < 32768u ? bytes - off : 32768u;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                hot_smem_u32(lr_hot_smem + 128 + off)),
            "l"(reinterpret_cast<const unsigned char*>(hot.buf) + off), "r"(sz), "r"(hot_smem_u32(&hot_bar))
            : "memory");
      }
    }
    __syncthreads();  // the barrier is initialised before anyone polls it
  }
  const CT* hot_rows = reinterpret_cast<const CT*>(lr_hot_smem + 128);
  const int lane = threadIdx.x & 31, g = lane % G, grp = lane / G, gbase = grp * G;
  const long long n_groups = (long long)gridDim.x * (blockDim.x >> 5) * GROUPS;
  long long it = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * GROUPS + grp;
  // software pipeline: the next batch's column indices / values (and the
  // next item's descriptor) are in flight while the current batch gathers
  Item cur{0, 0, 0, -1}, nxt{0, 0, 0, -1};
  if (it < n_items) cur = load_item(items, ptr, (int)it);
  if (it + n_groups < n_items) nxt = load_item(items, ptr, (int)(it + n_groups));
  int e = cur.beg;
  int jk[KB];
  Sc vk[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    const bool ok = g + G * k < cur.end - e;
    jk[k] = ok ? ld_stream(idx + e + g + G * k) : 0;
    vk[k] = ok ? ld_stream(val + e + g + G * k) : Sc(0);
  }
  CT acc[T];
#pragma unroll
  for (int t = 0; t < T; ++t) acc[t] = C::zero();
  const Sc* Xs = X - shift;
  if constexpr (HOT) {
    // the staged rows have landed (phase 0 of the one-shot barrier)
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "HOT_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        "@!p bra HOT_WAIT_%=;\n"
        "}\n" ::"r"(hot_smem_u32(&hot_bar))
        : "memory");
  }
  while (__any_sync(0xffffffffu, it < n_items)) {
    const bool act = it < n_items;
    const int nb = act ? min(kGroupBatch, cur.end - e) : 0;
    const bool same = act && e + nb < cur.end;
    const int ne = same ? e + nb : nxt.beg;
    const int nn = same ? cur.end - ne : ((it + n_groups < n_items) ? nxt.end - ne : 0);
    int jn[KB];
    Sc vn[KB];
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const bool ok = g + G * k < nn;
      jn[k] = ok ? ld_stream(idx + ne + g + G * k) : 0;
      vn[k] = ok ? ld_stream(val + ne + g + G * k) : Sc(0);
    }
#pragma unroll
    for (int q0 = 0; q0 < kGroupBatch; q0 += Q) {
      if (!__any_sync(0xffffffffu, q0 < nb)) break;
      CT xv[Q][T];
      Sc vq[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int ent = q0 + q;
        int j = __shfl_sync(0xffffffffu, jk[ent / G], gbase + ent % G);
        vq[q] = __shfl_sync(0xffffffffu, vk[ent / G], gbase + ent % G);
        if constexpr (HOT) {
          // one generic-address load serves both sources (no divergence
          // between the groups of a warp)
          const int rk = -j - 1;
          const bool staged = j < 0 && rk < hot.H;
          if (j < 0 && !staged) j = __ldg(hot.order + rk);
          const CT* xr = staged ? hot_rows + (long long)rk * hot.nchunk
                                : reinterpret_cast<const CT*>(Xs + (long long)j * ldx);
#pragma unroll
          for (int t = 0; t < T; ++t) {
            const int c = (g + G * t) * VE - shift;
            xv[q][t] = (ent < nb && c + VE > 0 && c < w) ? xr[g + G * t] : C::zero();
          }
        } else {
          const CT* xr = reinterpret_cast<const CT*>(Xs + (long long)j * ldx);
#pragma unroll
          for (int t = 0; t < T; ++t) {
            const int c = (g + G * t) * VE - shift;  // first column of the chunk
            xv[q][t] = (ent < nb && c + VE > 0 && c < w) ? __ldg(xr + g + G * t) : C::zero();
          }
        }
      }
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t) C::fma_into(vq[q], xv[q][t], acc[t]);
    }
    e += nb;
    if (act && e >= cur.end) {
      Sc* dst = (cur.slot >= 0) ? (scratch + (long long)cur.slot * w) : (Y + (long long)cur.row * ldy);
#pragma unroll
      for (int t = 0; t < T; ++t) {
#pragma unroll
        for (int i = 0; i < VE; ++i) {
          const int c = (g + G * t) * VE - shift + i;
          if (c >= 0 && c < w) dst[c] = C::get(acc[t], i);
        }
        acc[t] = C::zero();
      }
      it += n_groups;
      cur = nxt;
      e = cur.beg;
      if (it + n_groups < n_items) nxt = load_item(items, ptr, (int)(it + n_groups));
    }
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      jk[k] = jn[k];
      vk[k] = vn[k];
    }
  }
}

// Fused SVT step / SDDMM over CSR items (r <= 2 G T, V rows read from their
// start: the per-lane column slices, hence every entry's summation order,
// depend on (G, T, r) only -- the sharded engine's row- and column-block
// passes produce identical bits).  The item's row of U * S lives in
// registers (loaded once per item); per entry the group gathers V[j, :] as
// aligned chunks, each lane folds its columns (fma, ascending), and R = min(G, 8)
// entries' lane partials are reduced together (xor levels over the lane bits
// >= R, then a transpose-reduce over the low bits: R - 1 shuffles per R
// entries; the same tree for every entry).  Results are parked in shared
// memory and every lane finishes its own batch entries with coalesced M / Y
// traffic (residual partials, Y += step (m - x)).
// occupancy vs gathers in flight per (G, T) (profiles/r02u_svt_variants.txt):
// wide groups (G >= 16, r > 32) run 4 CTAs / SM with fewer entries in flight
// per group (r = 84: 1.74 -> 1.46 ms), narrow ones 3 CTAs / SM
template <int G, int T>
struct SvtTune {
  static constexpr int minb = G >= 16 ? 4 : LR_SVT_MINB;
  static constexpr int q = G >= 16 ? (T == 1 ? 4 : (T == 2 ? 2 : 1))
                                   : (T == 1 ? LR_SVT_Q1 : (T == 2 ? LR_SVT_Q2 : LR_SVT_Q3));
};

template <int G, int T, bool FUSED>
__global__ void __launch_bounds__(256, SvtTune<G, T>::minb) svt_group2_kernel(
    const int* __restrict__ ptr, const int* __restrict__ idx, const int* __restrict__ items, int n_items,
    const double* __restrict__ U, long long ldu, const double* __restrict__ S, const double* __restrict__ V,
    long long ldv, int r, double* __restrict__ x_out, const double* __restrict__ m_vals,
    double* __restrict__ y_csr, double* __restrict__ y_csc, const int* __restrict__ inv_perm, double step,
    int apply, double* __restrict__ partial) {
  constexpr int GROUPS = 32 / G;
  constexpr int B = (4 * G < kGroupBatch) ? 4 * G : kGroupBatch;  // batch entries per group
  constexpr int KB = B / G;
  constexpr int R = G < 8 ? G : 8;
  constexpr int QT = SvtTune<G, T>::q;
  constexpr int Q = QT < R ? QT : R;  // entries' gathers in flight (divides R)
  __shared__ double xs_all[8][B * GROUPS];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, g = lane % G, grp = lane / G, gbase = grp * G;
  double* xs = xs_all[wib] + grp * B;
  const long long n_groups = (long long)gridDim.x * (blockDim.x >> 5) * GROUPS;
  long long it = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * GROUPS + grp;
  Item cur{0, 0, 0, -1}, nxt{0, 0, 0, -1};
  double2 us[T];
  auto load_us = [&](int row) {
    const double* ur = U + (long long)row * ldu;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int c = 2 * (g + G * t);
      us[t].x = (c < r) ? __ldg(ur + c) * __ldg(S + c) : 0.0;
      us[t].y = (c + 1 < r) ? __ldg(ur + c + 1) * __ldg(S + c + 1) : 0.0;
    }
  };
  // software pipeline: the next batch's column indices (and the next item's
  // descriptor) are in flight while the current batch gathers
  if (it < n_items) {
    cur = load_item(items, ptr, (int)it);
    load_us(cur.row);
  }
  if (it + n_groups < n_items) nxt = load_item(items, ptr, (int)(it + n_groups));
  int e = cur.beg;
  int jk[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) jk[k] = (g + G * k < cur.end - e) ? ld_stream(idx + e + g + G * k) : 0;
  double ss = 0.0, mx = 0.0;
  while (__any_sync(0xffffffffu, it < n_items)) {
    const bool act = it < n_items;
    const int nb = act ? min(B, cur.end - e) : 0;
    const bool same = act && e + nb < cur.end;
    const int ne = same ? e + nb : nxt.beg;
    const int nn = same ? cur.end - ne : ((it + n_groups < n_items) ? nxt.end - ne : 0);
    int jn[KB];
#pragma unroll
    for (int k = 0; k < KB; ++k) jn[k] = (g + G * k < nn) ? ld_stream(idx + ne + g + G * k) : 0;
#pragma unroll
    for (int sb = 0; sb < B; sb += R) {
      if (!__any_sync(0xffffffffu, sb < nb)) break;
      double part[R];
#pragma unroll
      for (int q0 = 0; q0 < R; q0 += Q) {
        double2 vv[Q][T];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int ent = sb + q0 + q;
          const int j = __shfl_sync(0xffffffffu, jk[ent / G], gbase + ent % G);
          const double2* vr = reinterpret_cast<const double2*>(V + (long long)j * ldv);
#pragma unroll
          for (int t = 0; t < T; ++t) {
            const int c = 2 * (g + G * t);
            double2 v = make_double2(0.0, 0.0);
            if (ent < nb && c < r) {
              v = __ldg(vr + g + G * t);
              if (c + 1 >= r) v.y = 0.0;  // the row's padding may hold anything
            }
            vv[q][t] = v;
          }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          double p = 0.0;
#pragma unroll
          for (int t = 0; t < T; ++t) {
            p = fma(us[t].x, vv[q][t].x, p);
            p = fma(us[t].y, vv[q][t].y, p);
          }
          part[q0 + q] = p;
        }
      }
      // lane bits >= R: plain butterfly on all R partials
#pragma unroll
      for (int o = G / 2; o >= R; o >>= 1)
#pragma unroll
        for (int q = 0; q < R; ++q) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
      // low bits: transpose-reduce (lane g keeps entry g % R)
#pragma unroll
      for (int o = R / 2; o >= 1; o >>= 1) {
        const bool hi = (g & o) != 0;
#pragma unroll
        for (int q = 0; q < o; ++q) {
          const double send = hi ? part[q] : part[q + o];
          const double keep = hi ? part[q + o] : part[q];
          part[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      if (g < R) xs[sb + g] = part[0];
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const int b = g + G * k;
      if (b < nb) {
        const long long ee = e + b;
        const double xl = xs[b];
        if (FUSED) {
          // M / Y read here, not prefetched with the indices: their registers
          // would displace gathers in flight (the kernel is latency-bound)
          const double mv = ld_stream(m_vals + ee);
          const double d = xl - mv;
          ss = fma(d, d, ss);
          mx = fmax(mx, fabs(d));
          if (apply) {
            const double ynew = add_rn(ld_stream_rw(y_csr + ee), mul_rn(step, add_rn(mv, -xl)));
            y_csr[ee] = ynew;
            if (y_csc) y_csc[__ldg(inv_perm + ee)] = ynew;
          }
        } else {
          x_out[ee] = xl;
        }
      }
    }
    __syncwarp();
    e += nb;
    if (act && e >= cur.end) {
      it += n_groups;
      cur = nxt;
      e = cur.beg;
      if (it < n_items) load_us(cur.row);
      if (it + n_groups < n_items) nxt = load_item(items, ptr, (int)(it + n_groups));
    }
#pragma unroll
    for (int k = 0; k < KB; ++k) jk[k] = jn[k];
  }
  if (FUSED) {
    __shared__ double red[32];
    const double S2 = block_sum<256>(ss, red);
    const double M2 = block_max<256>(mx, red);
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = S2;
      partial[2 * blockIdx.x + 1] = M2;
    }
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <int G, int T, bool V2, int Q = 4, typename Sc = double>
static void launch_spmm_t(const int* ptr, const int* idx, const Sc* val, const int* items,
                          int n_items, const Sc* X, long long ldx, int w, Sc* Y,
                          long long ldy, Sc* scratch, cudaStream_t s) {
  constexpr int TILE = 2 * G * T;
  const int n_tiles = (w + TILE - 1) / TILE;
  constexpr int GROUPS = 32 / G;
  long long units = (long long)((n_items + GROUPS - 1) / GROUPS) * n_tiles;
  long long blocks = (units + 7) / 8;  // 8 warps per block
  long long cap = (long long)sm_count() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  spmm_kernel<G, T, V2, Q, Sc><<<(int)blocks, 256, 0, s>>>(ptr, idx, val, items, n_items, X, ldx, w, Y, ldy,
                                                           scratch, n_tiles);
}

// (G, T) per width: G lanes per item, T column pairs per lane.  Narrow
// products use few lanes and several pairs per lane so a warp keeps 4-16
// items (gathers) in flight and no lane idles on padding columns;
// LR_SPMM_GT="G,T" overrides for experiments.
template <bool V2, typename Sc = double>
static void dispatch_spmm(const int* ptr, const int* idx, const Sc* val, const int* items,
                          int n_items, const Sc* X, long long ldx, int w, Sc* Y,
                          long long ldy, Sc* scratch, cudaStream_t s) {
  const int pairs = (w + 1) / 2;
  static const char* env = getenv("LR_SPMM_GT");
  int G = 0, T = 0;
  if (env) sscanf(env, "%d,%d", &G, &T);
  if (G == 0) {
    if (pairs <= 1) { G = 1; T = 1; }
    else if (pairs <= 2) { G = 2; T = 1; }
    else if (pairs <= 4) { G = 4; T = 1; }
    else if (pairs <= 8) { G = 8; T = 1; }
    else if (pairs <= 16) { G = 8; T = 2; }   // cfg4 w = 22: 1029 -> 715 us (tools/spmm_gt_sweep.sh)
    else if (pairs <= 32) { G = 16; T = 2; }  // w = 33 / 45: 849 -> 808, 895 -> 847 us
    else if (pairs <= 64) { G = 32; T = 2; }
    else { G = 32; T = 3; }
  }
  static const int q_env = getenv("LR_SPMM_Q") ? atoi(getenv("LR_SPMM_Q")) : 0;
  const int Qv = q_env ? q_env : (T == 1 ? 8 : 4);
#define LR_SPMM_CASE(g, t)                                                                              \
  if (G == g && T == t) {                                                                               \
    if constexpr (t == 1) {                                                                             \
      if (Qv == 8)                                                                                      \
        return launch_spmm_t<g, t, V2, 8, Sc>(ptr, idx, val, items, n_items, X, ldx, w, Y, ldy, scratch, s); \
    }                                                                                                   \
    return launch_spmm_t<g, t, V2, 4, Sc>(ptr, idx, val, items, n_items, X, ldx, w, Y, ldy, scratch, s);        \
  }
  LR_SPMM_CASE(1, 1) LR_SPMM_CASE(2, 1) LR_SPMM_CASE(4, 1) LR_SPMM_CASE(8, 1) LR_SPMM_CASE(16, 1)
  LR_SPMM_CASE(32, 1) LR_SPMM_CASE(32, 2) LR_SPMM_CASE(32, 3)
  LR_SPMM_CASE(2, 2) LR_SPMM_CASE(2, 3) LR_SPMM_CASE(2, 4) LR_SPMM_CASE(4, 2) LR_SPMM_CASE(4, 3)
  LR_SPMM_CASE(4, 4) LR_SPMM_CASE(8, 2) LR_SPMM_CASE(8, 3) LR_SPMM_CASE(8, 4) LR_SPMM_CASE(16, 2)
  LR_SPMM_CASE(16, 3)
#undef LR_SPMM_CASE
  launch_spmm_t<32, 3, V2, 4, Sc>(ptr, idx, val, items, n_items, X, ldx, w, Y, ldy, scratch, s);
}

static bool aligned_bytes(const void* p, unsigned a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// (G, T) of the line-aligned kernels: a group spans >= 8 chunks (one
// 128-byte line per lane sweep; a 4-lane group would visit a line in two
// instructions, two wavefronts) unless the row fits 4 chunks; then the fewest
// chunk slots G*T covering `chunks` (ties: the smaller group, more entries per
// warp instruction); T <= 4.  Returns false past 128 chunks.
static bool pick_group(int chunks, int& G, int& T) {
  if (chunks <= 4) {
    G = 4;
    T = 1;
    return true;
  }
  static const int Gs[3] = {8, 16, 32};
  int best = 1 << 30;
  G = T = 0;
  for (int gi = 0; gi < 3; ++gi)
    for (int t = 1; t <= 4; ++t)
      if (Gs[gi] * t >= chunks && Gs[gi] * t < best) {
        best = Gs[gi] * t;
        G = Gs[gi];
        T = t;
      }
  return G > 0;
}

static int occupancy_blocks(const void* fn) {
  int o = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, 256, 0);
  return o < 1 ? 1 : o;
}

template <int G, int T, typename Sc>
static void launch_spmm_group_t(const int* ptr, const int* idx, const Sc* val, const int* items, int n_items,
                                const Sc* X, long long ldx, int w, int shift, Sc* Y, long long ldy, Sc* scratch,
                                cudaStream_t s) {
  constexpr int Q = T <= 2 ? LR_SPMM_QLO : LR_SPMM_QHI;
  constexpr int GROUPS = 32 / G;
  static int occ = -1;
  if (occ < 0) {
    // no shared memory: the whole unified L1 for the gathered rows
    cudaFuncSetAttribute(spmm_group_kernel<G, T, Q, Sc>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    occ = occupancy_blocks(reinterpret_cast<const void*>(spmm_group_kernel<G, T, Q, Sc>));
  }
  const long long warps = ((long long)n_items + GROUPS - 1) / GROUPS;
  long long blocks = (warps + 7) / 8;
  const long long cap = (long long)sm_count() * occ;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  spmm_group_kernel<G, T, Q, Sc><<<(int)blocks, 256, 0, s>>>(ptr, idx, val, items, n_items, X, ldx, w, shift, Y,
                                                             ldy, scratch);
}

// host-side description of a pattern side's hot-row encoding (see HotRows)
struct HotDesc {
  const int* idx_hot;   // the index stream with the hot ranks encoded
  const int* order;     // rank -> index
  int hot_max;          // ranks encoded (<= kHotMaxRows)
  void* buf;            // staging block in global memory
  long long buf_bytes;
};

// rows staged for a chunk of nchunk 16-byte chunks per row (0: not worth a launch)
static int hot_rows_for(const HotDesc* hd, int nchunk) {
  if (!hd || !hd->idx_hot || !hd->order || !hd->buf || nchunk <= 0) return 0;
  long long H = kHotSmemBytes / ((long long)nchunk * 16);
  if (H > hd->hot_max) H = hd->hot_max;
  if (H > hd->buf_bytes / ((long long)nchunk * 16)) H = hd->buf_bytes / ((long long)nchunk * 16);
  return H >= 32 ? (int)H : 0;
}

template <int G, int T, typename Sc>
static void launch_spmm_hot_t(const int* ptr, const HotDesc* hd, int H, int nchunk, const Sc* val, const int* items,
                              int n_items, const Sc* X, long long ldx, int w, int shift, Sc* Y, long long ldy,
                              Sc* scratch, cudaStream_t s) {
  using CT = typename Chunk16<Sc>::type;
  constexpr int VE = Chunk16<Sc>::VE;
  constexpr int Q = T <= 2 ? LR_SPMM_QLO : LR_SPMM_QHI;
  constexpr int GROUPS = 32 / G;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(spmm_group_kernel<G, T, Q, Sc, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         128 + kHotSmemBytes);
    attr = true;
  }
  const long long total = (long long)H * nchunk;
  int gb = (int)((total + 255) / 256);
  if (gb > sm_count() * 4) gb = sm_count() * 4;
  hot_rows_kernel<CT><<<gb, 256, 0, s>>>(reinterpret_cast<const CT*>(X - shift), ldx / VE, hd->order, H, nchunk,
                                         reinterpret_cast<CT*>(hd->buf));
  const long long warps = ((long long)n_items + GROUPS - 1) / GROUPS;
  long long blocks = (warps + kHotThreads / 32 - 1) / (kHotThreads / 32);
  if (blocks > sm_count()) blocks = sm_count();
  if (blocks < 1) blocks = 1;
  HotRows hot{hd->buf, hd->order, H, nchunk};
  spmm_group_kernel<G, T, Q, Sc, true><<<(int)blocks, kHotThreads, 128 + (size_t)total * 16, s>>>(
      ptr, hd->idx_hot, val, items, n_items, X, ldx, w, shift, Y, ldy, scratch, hot);
}

// the group kernel for one column chunk; false: not applicable (unaligned rows)
template <typename Sc>
static bool spmm_group(const int* ptr, const int* idx, const Sc* val, const int* items, int n_items, const Sc* X,
                       long long ldx, int w, Sc* Y, long long ldy, Sc* scratch, cudaStream_t s,
                       const HotDesc* hd = nullptr) {
  static const char* fam = getenv("LR_SPMM_KERNEL");
  if (fam && fam[0] == 'i') return false;  // "items": the round-1 kernel
  constexpr int VE = 16 / (int)sizeof(Sc);
  // rows share one offset from their 128-byte line only if the row stride is whole lines; then
  // the chunks are read from the line start and X itself may sit at any element (a column slice
  // of a Krylov block at an odd column offset); otherwise column 0 must start a 16-byte chunk
  const bool lines = (ldx * (long long)sizeof(Sc)) % 128 == 0;
  if (!aligned_bytes(X, (unsigned)sizeof(Sc)) || (ldx * (long long)sizeof(Sc)) % 16 != 0) return false;
  if (!lines && !aligned_bytes(X, 16)) return false;
  const int shift = lines ? (int)((reinterpret_cast<uintptr_t>(X) & 127u) / sizeof(Sc)) : 0;
  int G, T;
  const int nchunk = (w + shift + VE - 1) / VE;
  if (!pick_group(nchunk, G, T)) return false;
  if constexpr (sizeof(Sc) == 8) {
    const int H = hot_rows_for(hd, nchunk);
    if (H > 0) {
#define LR_SPH(g, t)                                                                                         \
  if (G == g && T == t) {                                                                                    \
    launch_spmm_hot_t<g, t, Sc>(ptr, hd, H, nchunk, val, items, n_items, X, ldx, w, shift, Y, ldy, scratch,  \
                                s);                                                                          \
    return true;                                                                                             \
  }
      LR_SPH(4, 1) LR_SPH(8, 1) LR_SPH(8, 2) LR_SPH(8, 3) LR_SPH(8, 4) LR_SPH(16, 1) LR_SPH(16, 2) LR_SPH(16, 3)
      LR_SPH(16, 4) LR_SPH(32, 1) LR_SPH(32, 2) LR_SPH(32, 3) LR_SPH(32, 4)
#undef LR_SPH
    }
  }
#define LR_SPG(g, t)                                                                                         \
  if (G == g && T == t) {                                                                                    \
    launch_spmm_group_t<g, t, Sc>(ptr, idx, val, items, n_items, X, ldx, w, shift, Y, ldy, scratch, s);     \
    return true;                                                                                             \
  }
  LR_SPG(4, 1) LR_SPG(4, 2) LR_SPG(4, 3) LR_SPG(4, 4) LR_SPG(8, 1) LR_SPG(8, 2) LR_SPG(8, 3) LR_SPG(8, 4)
  LR_SPG(16, 1) LR_SPG(16, 2) LR_SPG(16, 3) LR_SPG(16, 4) LR_SPG(32, 1) LR_SPG(32, 2) LR_SPG(32, 3)
  LR_SPG(32, 4)
#undef LR_SPG
  return false;
}

// Column-chunked SpMM over a row-compressed pattern, w >= 2 (shared by the
// fp64 and fp32 entry points)
template <typename Sc>
static int spmm_cols(const int* ptr, const int* idx, const Sc* val, const int* items, int n_items,
                     const int* splits, int n_splits, const Sc* X, long long ldx, int w, Sc* Y, long long ldy,
                     Sc* scratch, cudaStream_t s, const HotDesc* hd = nullptr) {
  // Products wider than kChunkCols run as column chunks: each chunk's slice
  // of X stays L2-resident while every stored entry gathers from it (the
  // W-column Y^T Q of BKI at cfg2 is 528 MB), and the <= 128-column tiles run
  // at higher occupancy than the 192-column one even when X fits in L2
  // (cfg4 CSR w = 132: 2.64 ms chunked vs 4.04 ms whole, tools/spmm_cfg4_probe.py).
  // Chunk count by a measured cost model: a pass over the entries with a
  // chunk of pc column pairs costs ~ (cap(pc) + 14) units per stored entry,
  // cap = the pair slots of dispatch_spmm's (G,T) mapping (1..96), 14 = the
  // per-pass entry overhead (fit to the cfg4 width sweep: 163 us + 11.4 us
  // per slot at 18M nnz, tools/spmm_cfg4_probe.py).  Cost = chunks x (cap +
  // 14); chunks are at most 128 columns.  E.g. w = 132: 3 chunks of 22 pairs
  // (1.77 -> 1.59 ms at cfg4) instead of 2 of 33; w = 110 stays one chunk.
  // LR_SPMM_CHUNK forces a fixed chunk width.
  static const int chunk_env = getenv("LR_SPMM_CHUNK") ? atoi(getenv("LR_SPMM_CHUNK")) : 0;
  constexpr unsigned kVecBytes = 2 * sizeof(Sc);
  const int pairs_all = (w + 1) / 2;
  auto cap = [](int pc) {
    return pc <= 1 ? 1 : pc <= 2 ? 2 : pc <= 4 ? 4 : pc <= 8 ? 8 : pc <= 16 ? 16 : pc <= 32 ? 32 : pc <= 64 ? 64 : 96;
  };
  int n_chunks = 1;
  if (chunk_env > 0) {
    n_chunks = (w + chunk_env - 1) / chunk_env;
  } else {
    long long best = -1;
    for (int c = 1; c <= pairs_all; ++c) {
      const int pc = (pairs_all + c - 1) / c;
      if (2 * pc > 128) continue;
      const long long score = (long long)c * (cap(pc) + 14);
      if (best < 0 || score < best) {
        best = score;
        n_chunks = c;
      }
      if (pc <= 8) break;  // narrower chunks only add metadata passes
    }
  }
  const int cw_even = (((w + n_chunks - 1) / n_chunks) + 1) & ~1;
  for (int c0 = 0; c0 < w; c0 += cw_even) {
    const int cw = (w - c0 < cw_even) ? (w - c0) : cw_even;
    const Sc* Xc = X + c0;
    Sc* Yc = Y + c0;
    const bool v2 = (ldx % 2 == 0) && (ldy % 2 == 0) && aligned_bytes(Xc, kVecBytes) &&
                    aligned_bytes(Yc, kVecBytes) &&
                    (scratch == nullptr || (aligned_bytes(scratch, kVecBytes) && cw % 2 == 0));
    if (spmm_group<Sc>(ptr, idx, val, items, n_items, Xc, ldx, cw, Yc, ldy, scratch, s, hd))
      ;
    else if (v2)
      dispatch_spmm<true, Sc>(ptr, idx, val, items, n_items, Xc, ldx, cw, Yc, ldy, scratch, s);
    else
      dispatch_spmm<false, Sc>(ptr, idx, val, items, n_items, Xc, ldx, cw, Yc, ldy, scratch, s);
    LR_CHECK_LAUNCH();
    if (n_splits > 0) {
      long long total = (long long)n_splits * cw;
      long long blocks = (total + 255) / 256;
      if (blocks > sm_count() * 8) blocks = sm_count() * 8;
      spmm_split_reduce_kernel<Sc><<<(int)blocks, 256, 0, s>>>(splits, n_splits, scratch, cw, Yc, ldy);
      LR_CHECK_LAUNCH();
    }
  }
  return LR_OK;
}

constexpr int kFlatK = 4;                    // entries per lane per tile
constexpr int kFlatTile = 32 * kFlatK;        // CSR slots per tile (lr_svt_tile_entries)
constexpr int kFlatMaxBlocksPerSm = 8;

template <int G, int T, int Q>
static int launch_flat_t(bool fused, const int* ptr, const int* idx, long long nnz, int m, const int* tile_row,
                         long long n_tiles, const double* U, long long ldu, const double* S, const double* V,
                         long long ldv, int r, double* x, const double* m_vals, double* y_csr, double* y_csc,
                         const int* inv_perm, double step, int apply, double* partial, cudaStream_t s) {
  static int occ[2] = {-1, -1};
  int& o = occ[fused ? 1 : 0];
  if (o < 0) {
    if (fused)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, svt_flat_kernel<G, T, kFlatK, Q, true>, kFlatWarps * 32, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, svt_flat_kernel<G, T, kFlatK, Q, false>, kFlatWarps * 32, 0);
    if (o < 1) o = 1;
    if (o > kFlatMaxBlocksPerSm) o = kFlatMaxBlocksPerSm;
  }
  long long blocks = (long long)sm_count() * o;
  const long long need = (n_tiles + kFlatWarps - 1) / kFlatWarps;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  if (fused)
    svt_flat_kernel<G, T, kFlatK, Q, true><<<(int)blocks, kFlatWarps * 32, 0, s>>>(
        ptr, idx, nnz, m, tile_row, n_tiles, U, ldu, S, V, ldv, r, x, m_vals, y_csr, y_csc, inv_perm, step, apply,
        partial);
  else
    svt_flat_kernel<G, T, kFlatK, Q, false><<<(int)blocks, kFlatWarps * 32, 0, s>>>(
        ptr, idx, nnz, m, tile_row, n_tiles, U, ldu, S, V, ldv, r, x, m_vals, y_csr, y_csc, inv_perm, step, apply,
        partial);
  ::lr::count_launches(1);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    set_error("svt_flat launch: %s", cudaGetErrorString(err));
    return -LR_ERR_CUDA;
  }
  return (int)blocks;  // > 0: blocks launched (partials written)
}

// (G, T, Q) by rank: G lanes x T column pairs cover the rank in one chunk up
// to r = 256 (wider ranks loop over chunks); LR_SVT_FLAT="G,T,Q" overrides.
static int launch_flat(bool fused, const int* ptr, const int* idx, long long nnz, int m, const int* tile_row,
                       const double* U, long long ldu, const double* S, const double* V, long long ldv, int r,
                       double* x, const double* m_vals, double* y_csr, double* y_csc, const int* inv_perm,
                       double step, int apply, double* partial, cudaStream_t s) {
  const long long n_tiles = (nnz + kFlatTile - 1) / kFlatTile;
  const int pairs = (r + 1) / 2;
  static const char* env = getenv("LR_SVT_FLAT");
  int G = 0, T = 0, Q = 0;
  if (env) sscanf(env, "%d,%d,%d", &G, &T, &Q);
  if (G == 0) {
    if (pairs <= 2) { G = 1; T = 2; Q = 4; }
    else if (pairs <= 4) { G = 2; T = 2; Q = 4; }
    else if (pairs <= 8) { G = 4; T = 2; Q = 4; }
    else if (pairs <= 16) { G = 8; T = 2; Q = 4; }
    else if (pairs <= 32) { G = 16; T = 2; Q = 4; }
    else if (pairs <= 64) { G = 32; T = 2; Q = 4; }
    else { G = 32; T = 4; Q = 2; }
  }
#define LR_FLAT(g, t, q)                                                                                      \
  if (G == g && T == t && Q == q)                                                                              \
    return launch_flat_t<g, t, q>(fused, ptr, idx, nnz, m, tile_row, n_tiles, U, ldu, S, V, ldv, r, x, m_vals, \
                                  y_csr, y_csc, inv_perm, step, apply, partial, s);
  LR_FLAT(1, 2, 4) LR_FLAT(2, 2, 4) LR_FLAT(4, 2, 4) LR_FLAT(8, 2, 4) LR_FLAT(16, 2, 4) LR_FLAT(32, 2, 4)
  LR_FLAT(32, 4, 2) LR_FLAT(1, 4, 2) LR_FLAT(2, 4, 2) LR_FLAT(4, 4, 2) LR_FLAT(8, 4, 2) LR_FLAT(16, 4, 2)
  LR_FLAT(1, 1, 4) LR_FLAT(2, 1, 4) LR_FLAT(4, 1, 4) LR_FLAT(8, 1, 4) LR_FLAT(16, 1, 4) LR_FLAT(1, 2, 2)
  LR_FLAT(2, 2, 2) LR_FLAT(4, 2, 2) LR_FLAT(8, 2, 2) LR_FLAT(4, 2, 8) LR_FLAT(8, 2, 8) LR_FLAT(2, 2, 8)
#undef LR_FLAT
  set_error("svt: no flat kernel instance for G=%d T=%d Q=%d", G, T, Q);
  return -LR_ERR_ARG;
}

template <int G, int T>
static int launch_svt_group2_t(bool fused, const int* ptr, const int* idx, const int* items, int n_items,
                               const double* U, long long ldu, const double* S, const double* V, long long ldv,
                               int r, double* x, const double* m_vals, double* y_csr, double* y_csc,
                               const int* inv_perm, double step, int apply, double* partial, cudaStream_t s) {
  static int occ[2] = {-1, -1};
  int& o = occ[fused ? 1 : 0];
  if (o < 0) {
    // minimal shared memory carve-out: L1 keeps the gathered V rows
    cudaFuncSetAttribute(svt_group2_kernel<G, T, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 10);
    cudaFuncSetAttribute(svt_group2_kernel<G, T, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 10);
    o = fused ? occupancy_blocks(reinterpret_cast<const void*>(svt_group2_kernel<G, T, true>))
              : occupancy_blocks(reinterpret_cast<const void*>(svt_group2_kernel<G, T, false>));
    if (o > kSvtBlocksPerSm) o = kSvtBlocksPerSm;  // the partial buffer holds sm_count * kSvtBlocksPerSm
  }
  constexpr int GROUPS = 32 / G;
  const long long warps = ((long long)n_items + GROUPS - 1) / GROUPS;
  long long blocks = (warps + 7) / 8;
  const long long cap = (long long)sm_count() * o;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (fused)
    svt_group2_kernel<G, T, true><<<(int)blocks, 256, 0, s>>>(ptr, idx, items, n_items, U, ldu, S, V, ldv, r, x,
                                                               m_vals, y_csr, y_csc, inv_perm, step, apply,
                                                               partial);
  else
    svt_group2_kernel<G, T, false><<<(int)blocks, 256, 0, s>>>(ptr, idx, items, n_items, U, ldu, S, V, ldv, r, x,
                                                                m_vals, y_csr, y_csc, inv_perm, step, apply,
                                                                partial);
  ::lr::count_launches(1);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    set_error("svt_group2 launch: %s", cudaGetErrorString(err));
    return 0;
  }
  return (int)blocks;
}

}  // namespace lr

using namespace lr;

extern "C" {

int lr_svt_step_partials(void) { return sm_count() * kSvtBlocksPerSm * 2; }

int lr_spmm_f64(const int* ptr, const int* idx, const double* val, int rows, const int* items,
                int n_items, const int* splits, int n_splits, const double* X, long long ldx, int w,
                double* Y, long long ldy, double* scratch, void* stream) {
  LR_REQUIRE(w >= 0 && ldx >= w && ldy >= w, "spmm: bad widths (w=%d ldx=%lld ldy=%lld)", w, ldx,
             ldy);
  if (w == 0 || rows == 0) return LR_OK;
  if (!items) n_items = rows;
  LR_REQUIRE(n_splits == 0 || scratch, "spmm: split schedule needs scratch");
  cudaStream_t s = as_stream(stream);
  if (w == 1) {
    long long blocks = ((long long)n_items + 7) / 8;
    long long cap = (long long)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    spmv_kernel<<<(int)blocks, 256, 0, s>>>(ptr, idx, val, items, n_items, X, ldx, Y, ldy, scratch);
    LR_CHECK_LAUNCH();
    if (n_splits > 0) {
      long long rb = ((long long)n_splits + 255) / 256;
      if (rb > sm_count() * 8) rb = sm_count() * 8;
      spmm_split_reduce_kernel<double><<<(int)rb, 256, 0, s>>>(splits, n_splits, scratch, 1, Y, ldy);
      LR_CHECK_LAUNCH();
    }
    return LR_OK;
  }
  return spmm_cols<double>(ptr, idx, val, items, n_items, splits, n_splits, X, ldx, w, Y, ldy, scratch, s);
}

int lr_spmm_hot_rows_max(void) { return kHotMaxRows; }

long long lr_spmm_hot_buf_doubles(void) { return kHotSmemBytes / 8; }

int lr_spmm_hot_f64(const int* ptr, const int* idx, const int* idx_hot, const int* hot_order, int hot_max,
                    double* hot_buf, long long hot_buf_doubles, const double* val, int rows, const int* items,
                    int n_items, const int* splits, int n_splits, const double* X, long long ldx, int w, double* Y,
                    long long ldy, double* scratch, void* stream) {
  LR_REQUIRE(w >= 2 && ldx >= w && ldy >= w, "spmm_hot: bad widths (w=%d ldx=%lld ldy=%lld; w >= 2)", w, ldx, ldy);
  LR_REQUIRE(idx && idx_hot && hot_order && hot_buf && hot_max >= 1 && hot_max <= kHotMaxRows,
             "spmm_hot: hot-row encoding missing (hot_max=%d, at most %d)", hot_max, kHotMaxRows);
  if (rows == 0) return LR_OK;
  if (!items) n_items = rows;
  LR_REQUIRE(n_splits == 0 || scratch, "spmm_hot: split schedule needs scratch");
  HotDesc hd{idx_hot, hot_order, hot_max, hot_buf, hot_buf_doubles * 8};
  return spmm_cols<double>(ptr, idx, val, items, n_items, splits, n_splits, X, ldx, w, Y, ldy, scratch,
                           as_stream(stream), &hd);
}

int lr_spmm_f32(const int* ptr, const int* idx, const float* val, int rows, const int* items, int n_items,
                const int* splits, int n_splits, const float* X, long long ldx, int w, float* Y, long long ldy,
                float* scratch, void* stream) {
  LR_REQUIRE(w >= 2 && ldx >= w && ldy >= w, "spmm_f32: bad widths (w=%d ldx=%lld ldy=%lld; w >= 2)", w, ldx,
             ldy);
  if (rows == 0) return LR_OK;
  if (!items) n_items = rows;
  LR_REQUIRE(n_splits == 0 || scratch, "spmm_f32: split schedule needs scratch");
  return spmm_cols<float>(ptr, idx, val, items, n_items, splits, n_splits, X, ldx, w, Y, ldy, scratch,
                          as_stream(stream));
}

static int launch_sddmm(bool fused, const int* ptr, const int* idx, int rows, const int* items,
                        int n_items, const double* U, long long ldu, const double* S,
                        const double* V, long long ldv, int r, double* x, const double* m_vals,
                        double* y_csr, double* y_csc, const int* inv_perm, double step, int apply,
                        double* partial, cudaStream_t s, int* nblocks = nullptr) {
  if (!items) n_items = rows;
  const int blocks = sm_count() * kSvtBlocksPerSm;
  if (nblocks) *nblocks = blocks;
  // kernel family: "group2" (default for r <= 256 with 16-byte aligned V
  // rows: line-aligned V gathers, U * S per item in registers), "batch"
  // (coalesced per-entry finishing, any rank), "legacy" (round-1 warp /
  // group kernels, r <= 1024); LR_SVT_GT="G,T,Q" overrides the batch
  // kernel's lane mapping for experiments
  static const char* fam = getenv("LR_SVT_KERNEL");
  const bool legacy = fam && fam[0] == 'l';
  const bool batch_only = fam && fam[0] == 'b';
  // the flat kernel's lane map (G lanes x T column pairs per entry, pairs
  // c = 2 (g + G t)) and reduction tree: every entry's value is bit-identical
  // to lr_svt_step_flat_f64's (tests/test_gpu_kernels.py::
  // test_sddmm_group_kernel_matches_flat)
  // lane map: the fewest chunk slots covering r (pick_group: r = 48 on 8 lanes
  // x 3 pairs, r = 84 on 16 x 3) unless that needs 4 pairs per lane (register
  // spills at 3 CTAs / SM), then the flat kernel's map (16 x 2, 32 x 2, 32 x 4)
  // -- profiles/r02s_svt_lane_map.txt; LR_SVT_MAP=flat forces the flat map
  // (every entry bit-identical to lr_svt_step_flat_f64)
  static const char* map_env = getenv("LR_SVT_MAP");
  const bool flat_only = map_env && map_env[0] == 'f' && map_env[1] == 'l';
  const int pairs = (r + 1) / 2;
  int G2 = 0, T2 = 2;
  if (!flat_only && pick_group(pairs, G2, T2) && T2 < 4) {
    // fit map chosen
  } else if ((G2 = 0, T2 = 2, pairs <= 2)) G2 = 1;
  else if (pairs <= 4) G2 = 2;
  else if (pairs <= 8) G2 = 4;
  else if (pairs <= 16) G2 = 8;
  else if (pairs <= 32) G2 = 16;
  else if (pairs <= 64) G2 = 32;
  else if (pairs <= 128) { G2 = 32; T2 = 4; }
  if (!legacy && !batch_only && r >= 1 && G2 > 0 && (ldv % 2 == 0) && aligned16(V)) {
    int nb = -1;
#define LR_SG2(g, t)                                                                                          \
  if (G2 == g && T2 == t)                                                                                     \
    nb = launch_svt_group2_t<g, t>(fused, ptr, idx, items, n_items, U, ldu, S, V, ldv, r, x, m_vals, y_csr,   \
                                   y_csc, inv_perm, step, apply, partial, s);
    LR_SG2(1, 2) LR_SG2(2, 2) LR_SG2(4, 2) LR_SG2(8, 2) LR_SG2(16, 2) LR_SG2(32, 2) LR_SG2(32, 4)
    LR_SG2(4, 1) LR_SG2(8, 1) LR_SG2(8, 3) LR_SG2(8, 4) LR_SG2(16, 1) LR_SG2(16, 3) LR_SG2(16, 4)
    LR_SG2(32, 1) LR_SG2(32, 3)
#undef LR_SG2
    if (nb > 0) {
      if (nblocks) *nblocks = nb;
      return LR_OK;
    }
    if (nb == 0) return LR_ERR_CUDA;
  }
  if (!legacy) {
    const int pairs = (r + 1) / 2;
    static const char* gt = getenv("LR_SVT_GT");
    int G = 0, T = 0, Q = 0;
    if (gt) sscanf(gt, "%d,%d,%d", &G, &T, &Q);
    if (G == 0) {
      if (pairs <= 4) { G = 1; T = 4; Q = 2; }
      else if (pairs <= 8) { G = 2; T = 4; Q = 2; }
      else if (pairs <= 16) { G = 4; T = 4; Q = 2; }
      else if (pairs <= 32) { G = 8; T = 4; Q = 2; }
      else if (pairs <= 64) { G = 16; T = 4; Q = 2; }
      else { G = 32; T = 4; Q = 2; }
    }
#define LR_SVT_BATCH(g, t, q)                                                                               \
  if (G == g && T == t && Q == q) {                                                                          \
    if (fused)                                                                                               \
      svt_batch_kernel<g, t, q, true><<<blocks, kSvtThreads, 0, s>>>(ptr, idx, items, n_items, U, ldu, S, V,  \
                                                                     ldv, r, x, m_vals, y_csr, y_csc,        \
                                                                     inv_perm, step, apply, partial);        \
    else                                                                                                     \
      svt_batch_kernel<g, t, q, false><<<blocks, kSvtThreads, 0, s>>>(ptr, idx, items, n_items, U, ldu, S, V, \
                                                                      ldv, r, x, m_vals, y_csr, y_csc,       \
                                                                      inv_perm, step, apply, partial);       \
    LR_CHECK_LAUNCH();                                                                                       \
    return LR_OK;                                                                                            \
  }
    LR_SVT_BATCH(1, 4, 2) LR_SVT_BATCH(2, 4, 2) LR_SVT_BATCH(4, 4, 2) LR_SVT_BATCH(8, 4, 2)
    LR_SVT_BATCH(16, 4, 2) LR_SVT_BATCH(32, 4, 2)
    LR_SVT_BATCH(1, 2, 4) LR_SVT_BATCH(2, 2, 4) LR_SVT_BATCH(4, 2, 4) LR_SVT_BATCH(8, 2, 4)
    LR_SVT_BATCH(16, 2, 4) LR_SVT_BATCH(32, 2, 4) LR_SVT_BATCH(1, 8, 1) LR_SVT_BATCH(2, 8, 1)
    LR_SVT_BATCH(4, 8, 1) LR_SVT_BATCH(8, 8, 1) LR_SVT_BATCH(4, 4, 4) LR_SVT_BATCH(8, 4, 4)
    LR_SVT_BATCH(8, 1, 4) LR_SVT_BATCH(4, 1, 4) LR_SVT_BATCH(16, 1, 4) LR_SVT_BATCH(16, 2, 2)
#undef LR_SVT_BATCH
    LR_REQUIRE(false, "sddmm: no batch kernel instance for G=%d T=%d Q=%d", G, T, Q);
  }
  LR_REQUIRE(r <= kMaxRankSmem, "sddmm: rank %d exceeds %d", r, kMaxRankSmem);
  const bool old_kernel = fam && fam[1] == 'w';  // "lw": legacy warp kernel only
  const bool v2ok = (ldv % 2 == 0) && aligned16(V) && (ldu >= r);
  // the group kernel wins only for wide factors (cfg4, tools/sddmm_probe.py: r = 84 2.13 vs 2.26 ms,
  // r = 160 2.99 vs 5.52 ms; r <= 40 the warp kernel is up to 2x faster)
  if (!old_kernel && r >= 64 && r <= 256 && v2ok) {
    const int pairs = (r + 1) / 2;
#define LR_SVT_GROUP(g, t)                                                                                 \
  do {                                                                                                     \
    if (fused)                                                                                             \
      svt_group_kernel<g, t, true><<<blocks, kSvtThreads, 0, s>>>(ptr, idx, items, n_items, U, ldu, S, V,  \
                                                                  ldv, r, x, m_vals, y_csr, y_csc,         \
                                                                  inv_perm, step, apply, partial);         \
    else                                                                                                   \
      svt_group_kernel<g, t, false><<<blocks, kSvtThreads, 0, s>>>(ptr, idx, items, n_items, U, ldu, S, V, \
                                                                   ldv, r, x, m_vals, y_csr, y_csc,        \
                                                                   inv_perm, step, apply, partial);        \
  } while (0)
    if (pairs <= 1) LR_SVT_GROUP(1, 1);
    else if (pairs <= 2) LR_SVT_GROUP(2, 1);
    else if (pairs <= 4) LR_SVT_GROUP(4, 1);
    else if (pairs <= 8) LR_SVT_GROUP(8, 1);
    else if (pairs <= 16) LR_SVT_GROUP(8, 2);
    else if (pairs <= 32) LR_SVT_GROUP(16, 2);
    else if (pairs <= 64) LR_SVT_GROUP(32, 2);
    else LR_SVT_GROUP(32, 4);
#undef LR_SVT_GROUP
    LR_CHECK_LAUNCH();
    return LR_OK;
  }
  const size_t smem = (size_t)(kSvtThreads / 32) * (r > 0 ? r : 1) * sizeof(double);
  const bool v2 = (ldv % 2 == 0) && aligned16(V);
  if (smem > 48 * 1024) {
    if (fused) {
      cudaFuncSetAttribute(sddmm_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(sddmm_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    } else {
      cudaFuncSetAttribute(sddmm_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(sddmm_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
  }
#define LR_SDDMM_ARGS                                                                           \
  ptr, idx, items, n_items, U, ldu, S, V, ldv, r, x, m_vals, y_csr, y_csc, inv_perm, step, apply, \
      partial
  if (fused) {
    if (v2)
      sddmm_kernel<true, true><<<blocks, kSvtThreads, smem, s>>>(LR_SDDMM_ARGS);
    else
      sddmm_kernel<true, false><<<blocks, kSvtThreads, smem, s>>>(LR_SDDMM_ARGS);
  } else {
    if (v2)
      sddmm_kernel<false, true><<<blocks, kSvtThreads, smem, s>>>(LR_SDDMM_ARGS);
    else
      sddmm_kernel<false, false><<<blocks, kSvtThreads, smem, s>>>(LR_SDDMM_ARGS);
  }
#undef LR_SDDMM_ARGS
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_sddmm_f64(const int* ptr, const int* idx, int rows, const int* items, int n_items,
                 const double* U, long long ldu, const double* S, const double* V, long long ldv,
                 int r, double* x, void* stream) {
  LR_REQUIRE(r >= 1, "sddmm: rank must be >= 1");
  return launch_sddmm(false, ptr, idx, rows, items, n_items, U, ldu, S, V, ldv, r, x, nullptr,
                      nullptr, nullptr, nullptr, 0.0, 0, nullptr, as_stream(stream));
}

int lr_svt_step_f64(const int* ptr, const int* idx, int rows, const int* items, int n_items,
                    const double* U, long long ldu, const double* S, const double* V, long long ldv,
                    int r, const double* m_vals, double* y_csr, double* y_csc, const int* inv_perm,
                    double step, int apply, double* partial, int n_partial, double* out2,
                    void* stream) {
  cudaStream_t s = as_stream(stream);
  const int blocks = sm_count() * kSvtBlocksPerSm;
  LR_REQUIRE(n_partial >= 2 * blocks, "svt_step: partial buffer too small (%d < %d)", n_partial,
             2 * blocks);
  int launched = blocks;
  {
    int st = launch_sddmm(true, ptr, idx, rows, items, n_items, U, ldu, S, V, ldv, r, nullptr,
                          m_vals, y_csr, y_csc, inv_perm, step, apply, partial, s, &launched);
    if (st != LR_OK) return st;
  }
  svt_finish_kernel<<<1, 32, 0, s>>>(partial, launched, out2);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_svt_tile_entries(void) { return kFlatTile; }

long long lr_svt_tile_count(long long nnz) { return (nnz + kFlatTile - 1) / kFlatTile; }

int lr_svt_tile_rows_i32(const int* ptr, int m, long long nnz, int* tile_row, void* stream) {
  const long long n_tiles = (nnz + kFlatTile - 1) / kFlatTile;
  if (n_tiles == 0) return LR_OK;
  LR_REQUIRE(m >= 1, "svt_tile_rows: m must be >= 1");
  long long blocks = (n_tiles + 255) / 256;
  if (blocks > sm_count() * 8) blocks = sm_count() * 8;
  tile_rows_kernel<<<(int)blocks, 256, 0, as_stream(stream)>>>(ptr, m, nnz, kFlatTile, n_tiles, tile_row);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_svt_flat_partials(void) { return sm_count() * kFlatMaxBlocksPerSm * 2; }

int lr_svt_step_flat_f64(const int* ptr, const int* idx, int m, long long nnz, const int* tile_row,
                         const double* U, long long ldu, const double* S, const double* V, long long ldv, int r,
                         const double* m_vals, double* y_csr, double* y_csc, const int* inv_perm, double step,
                         int apply, double* partial, int n_partial, double* out2, void* stream) {
  cudaStream_t s = as_stream(stream);
  LR_REQUIRE(n_partial >= lr_svt_flat_partials(), "svt_step: partial buffer too small (%d < %d)", n_partial,
             lr_svt_flat_partials());
  LR_REQUIRE(r >= 0 && (r == 0 || (ldu >= r && ldv >= r)), "svt_step: bad rank / leading dims (r=%d)", r);
  if (nnz == 0) {
    LR_CHECK_CUDA(cudaMemsetAsync(out2, 0, 2 * sizeof(double), s));
    return LR_OK;
  }
  const int blocks = launch_flat(true, ptr, idx, nnz, m, tile_row, U, ldu, S, V, ldv, r, nullptr, m_vals, y_csr,
                                 y_csc, inv_perm, step, apply, partial, s);
  if (blocks < 0) return -blocks;
  svt_finish_kernel<<<1, 32, 0, s>>>(partial, blocks, out2);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_sddmm_flat_f64(const int* ptr, const int* idx, int m, long long nnz, const int* tile_row, const double* U,
                      long long ldu, const double* S, const double* V, long long ldv, int r, double* x,
                      void* stream) {
  LR_REQUIRE(r >= 1 && ldu >= r && ldv >= r, "sddmm: bad rank / leading dims (r=%d)", r);
  if (nnz == 0) return LR_OK;
  const int blocks = launch_flat(false, ptr, idx, nnz, m, tile_row, U, ldu, S, V, ldv, r, x, nullptr, nullptr,
                                 nullptr, nullptr, 0.0, 0, nullptr, as_stream(stream));
  return blocks < 0 ? -blocks : LR_OK;
}

int lr_pattern_axpy_f64(double* y_csr, double* y_csc, const int* inv_perm, const double* delta,
                        double alpha, long long nnz, void* stream) {
  if (nnz == 0) return LR_OK;
  long long blocks = (nnz + 255) / 256;
  if (blocks > sm_count() * 8) blocks = sm_count() * 8;
  pattern_axpy_kernel<<<(int)blocks, 256, 0, as_stream(stream)>>>(y_csr, y_csc, inv_perm, delta,
                                                                  alpha, nnz);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

}  // extern "C"
