// fp64 GEMM on the tensor cores: mma.sync.aligned.m8n8k4.f64 (SASS
// DMMA.8x8x4; tcgen05 has no f64 kind).  Measured on this pool's B200:
// DMMA 37.1 TF/s vs DFMA 36.3 and cuBLAS DGEMM 35.4 (profiles/r01_fp64_peaks.txt).
//
// C[MxN] = alpha * op(A) * B + beta * C, row-major, arbitrary ld.
//   transA = 0: A is M x K  (tall A times small B: TRSM-as-GEMM, lifts, rescale)
//   transA = 1: A is K x M  (C = A^T B: Gram / projections, split-K over the
//               long K with partial tiles reduced in fixed order)
// Two tile shapes share one template: 128x64 CTA tiles with 64x32 warp tiles
// (32 DMMA per k4 step per warp, 0.375 fragment loads per DMMA) for large
// problems, 64x64 / 32x32 for small ones.  3-stage cp.async pipeline with
// 16-byte copies (zero-filled at the edges).  SYRK mode computes upper tiles
// only and mirrors them (exactly symmetric, like the reference's dsyrk).
#include <stdlib.h>

#include "lr_common.cuh"

namespace lr {

constexpr int BK_ALIGN = 32;  // split-K chunks are multiples of every tile's BK

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int src_bytes) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, int src_bytes) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BM_, int BN_, int WM_, int WN_, int BK_ = 16, int STAGES_ = 3>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, BK = BK_, STAGES = STAGES_;
  static constexpr int MT = WM / 8, NT = WN / 8;
  static constexpr int WARPS = (BM / WM) * (BN / WN);
  static constexpr int THREADS = WARPS * 32;
  static constexpr int LDA_N = BK + 4;  // A stored [m][k]
  static constexpr int LDA_T = BM + 4;  // A stored [k][m]
  static constexpr int LDB = BN + 4;    // B stored [k][n]
  static constexpr int A_STAGE = (BM * LDA_N > BK * LDA_T) ? BM * LDA_N : BK * LDA_T;
  static constexpr int B_STAGE = BK * LDB;
  static constexpr int SMEM = STAGES * (A_STAGE + B_STAGE) * (int)sizeof(double);
};
using TileL = Tile<128, 64, 64, 32>;
using TileL8 = Tile<128, 64, 32, 32>;   // 8 warps of 32x32: 16 warps/SM at 2 CTAs/SM
using TileW = Tile<128, 128, 64, 32>;   // 8 warps of 64x32
using TileL32 = Tile<128, 64, 64, 32, 32, 2>;  // BK 32, 2 stages: half the barriers per DMMA
using TileL832 = Tile<128, 64, 32, 32, 32, 2>;
using TileT = Tile<64, 128, 32, 64>;    // cuBLAS-like 64x128, 4 warps of 32x64
using TileS = Tile<64, 64, 32, 32>;

template <typename T, bool TRANS_A>
__global__ void __launch_bounds__(T::THREADS) gemm_kernel(int M, int N, int K, double alpha,
                                                         const double* __restrict__ A, long long lda,
                                                         const double* __restrict__ B, long long ldb, double beta,
                                                         double* __restrict__ C, long long ldc, int flags,
                                                         double* __restrict__ work, int k_chunk, int vec16) {
  const int tn = blockIdx.x, tm = blockIdx.y, z = blockIdx.z;
  if ((flags & LR_GEMM_SYRK_UPPER) && (tn + 1) * T::BN <= tm * T::BM) return;  // tile entirely below diagonal
  extern __shared__ __align__(16) double g_smem[];
  double* As = g_smem;
  double* Bs = g_smem + T::STAGES * T::A_STAGE;

  const int m0 = tm * T::BM, n0 = tn * T::BN;
  const int k_begin = z * k_chunk;
  int k_end = min(K, k_begin + k_chunk);
  if (flags & LR_GEMM_B_UPPER) k_end = min(k_end, n0 + T::BN);
  const int nk = (k_end > k_begin) ? (k_end - k_begin + T::BK - 1) / T::BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / (T::BN / T::WN), wn = warp % (T::BN / T::WN);
  const int gid = lane >> 2, tig = lane & 3;

  double acc[T::MT][T::NT][2];
#pragma unroll
  for (int i = 0; i < T::MT; ++i)
#pragma unroll
    for (int j = 0; j < T::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Warp-uniform pruning: a warp whose sub-tile lies outside C or strictly
  // below the diagonal (SYRK) issues no DMMA, and with an upper-triangular B
  // a warp stops at its last column's k (B[k][c] = 0 for k > c).  (Per-
  // fragment predication was tried: it breaks the DMMA issue stream.)
  bool warp_live;
  int warp_klim;
  {
    const int rbase = m0 + wm * T::WM, cbase = n0 + wn * T::WN;
    warp_live = rbase < M && cbase < N;
    if ((flags & LR_GEMM_SYRK_UPPER) && cbase + T::WN - 1 < rbase) warp_live = false;
    warp_klim = (flags & LR_GEMM_B_UPPER) ? min(k_end, cbase + T::WN) : k_end;
  }

  // Lean 16-byte path: every (row, pair) a thread copies is fixed for the
  // whole k loop, so offsets and the M/N edge predicates are computed once
  // and a stage is NA + NB fully unrolled cp.async with one k-bound test
  // each (the generic loop below re-derived indices per element per stage).
  constexpr int A_PAIRS = TRANS_A ? T::BM / 2 : T::BK / 2;  // 16-byte chunks per A smem row
  constexpr int A_ROWS = TRANS_A ? T::BK : T::BM;
  constexpr int NA = A_ROWS * A_PAIRS / T::THREADS;          // chunks per thread
  constexpr int A_STRIDE = T::THREADS / A_PAIRS;              // rows between a thread's chunks
  constexpr int B_PAIRS = T::BN / 2;
  constexpr int NB = T::BK * B_PAIRS / T::THREADS;
  constexpr int B_STRIDE = T::THREADS / B_PAIRS;
  static_assert(NA * T::THREADS == A_ROWS * A_PAIRS && NB * T::THREADS == T::BK * B_PAIRS, "tile/threads");
  const int a_row0 = tid / A_PAIRS, a_col = 2 * (tid % A_PAIRS);
  const int b_row0 = tid / B_PAIRS, b_col = 2 * (tid % B_PAIRS);
  int a_bytes_mn = 16;  // TRANS_A: M edge of this thread's column pair (fixed)
  if (TRANS_A) a_bytes_mn = (m0 + a_col + 1 < M) ? 16 : (m0 + a_col < M ? 8 : 0);
  const int b_bytes_n = (n0 + b_col + 1 < N) ? 16 : (n0 + b_col < N ? 8 : 0);
  unsigned a_row_ok = 0;  // !TRANS_A: M edge per chunk row (fixed)
  if (!TRANS_A) {
#pragma unroll
    for (int i = 0; i < NA; ++i)
      if (m0 + a_row0 + i * A_STRIDE < M) a_row_ok |= 1u << i;
  }
  auto load_stage_fast = [&](int st, int kt) {
    const int k0 = k_begin + kt * T::BK;
    double* as = As + st * T::A_STAGE;
    double* bs = Bs + st * T::B_STAGE;
    if (TRANS_A) {
      const double* src = A + (long long)(k0 + a_row0) * lda + m0 + a_col;
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const int kk = a_row0 + i * A_STRIDE;
        const int nb = (k0 + kk < k_end) ? a_bytes_mn : 0;
        cp_async16(as + kk * T::LDA_T + a_col, nb ? src + (long long)i * A_STRIDE * lda : A, nb);
      }
    } else {
      const int gk = k0 + a_col;
      const int kb = (gk + 1 < k_end) ? 16 : (gk < k_end ? 8 : 0);
      const double* src = A + (long long)(m0 + a_row0) * lda + gk;
#pragma unroll
      for (int i = 0; i < NA; ++i) {
        const int mm = a_row0 + i * A_STRIDE;
        const int nb = (a_row_ok >> i) & 1 ? kb : 0;
        cp_async16(as + mm * T::LDA_N + a_col, nb ? src + (long long)i * A_STRIDE * lda : A, nb);
      }
    }
    const double* bsrc = B + (long long)(k0 + b_row0) * ldb + n0 + b_col;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const int kk = b_row0 + i * B_STRIDE;
      const int nb = (k0 + kk < k_end) ? b_bytes_n : 0;
      cp_async16(bs + kk * T::LDB + b_col, nb ? bsrc + (long long)i * B_STRIDE * ldb : B, nb);
    }
  };

  auto load_stage = [&](int st, int kt) {
    if (vec16) {
      load_stage_fast(st, kt);
      return;
    }
    const int k0 = k_begin + kt * T::BK;
    double* as = As + st * T::A_STAGE;
    double* bs = Bs + st * T::B_STAGE;
    if (!TRANS_A) {
      for (int e = tid; e < T::BM * T::BK; e += T::THREADS) {
        const int mm = e / T::BK, kk = e % T::BK;
        const int gm = m0 + mm, gk = k0 + kk;
        const bool ok = gm < M && gk < k_end;
        cp_async8(as + mm * T::LDA_N + kk, ok ? A + (long long)gm * lda + gk : A, ok ? 8 : 0);
      }
    } else {
      for (int e = tid; e < T::BK * T::BM; e += T::THREADS) {
        const int kk = e / T::BM, mm = e % T::BM;
        const int gm = m0 + mm, gk = k0 + kk;
        const bool ok = gm < M && gk < k_end;
        cp_async8(as + kk * T::LDA_T + mm, ok ? A + (long long)gk * lda + gm : A, ok ? 8 : 0);
      }
    }
    for (int e = tid; e < T::BK * T::BN; e += T::THREADS) {
      const int kk = e / T::BN, nn = e % T::BN;
      const int gn = n0 + nn, gk = k0 + kk;
      const bool ok = gn < N && gk < k_end;
      cp_async8(bs + kk * T::LDB + nn, ok ? B + (long long)gk * ldb + gn : B, ok ? 8 : 0);
    }
  };

#pragma unroll
  for (int s = 0; s < T::STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<T::STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + T::STAGES - 1;
      if (nxt < nk) load_stage(nxt % T::STAGES, nxt);
      cp_async_commit();
    }
    const double* as = As + (kt % T::STAGES) * T::A_STAGE;
    const double* bs = Bs + (kt % T::STAGES) * T::B_STAGE;
    const int kg0 = k_begin + kt * T::BK;
    if (!warp_live || kg0 >= warp_klim) continue;  // warp-uniform; barriers are at the loop top
#pragma unroll
    for (int kk = 0; kk < T::BK; kk += 4) {
      double af[T::MT], bf[T::NT];
#pragma unroll
      for (int i = 0; i < T::MT; ++i) {
        const int mm = wm * T::WM + i * 8 + gid;
        af[i] = TRANS_A ? as[(kk + tig) * T::LDA_T + mm] : as[mm * T::LDA_N + kk + tig];
      }
#pragma unroll
      for (int j = 0; j < T::NT; ++j) bf[j] = bs[(kk + tig) * T::LDB + wn * T::WN + j * 8 + gid];
#pragma unroll
      for (int i = 0; i < T::MT; ++i)
#pragma unroll
        for (int j = 0; j < T::NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue
  const bool split = gridDim.z > 1;
  const bool syrk = (flags & LR_GEMM_SYRK_UPPER) != 0;
#pragma unroll
  for (int i = 0; i < T::MT; ++i) {
    const int row = m0 + wm * T::WM + i * 8 + gid;
#pragma unroll
    for (int j = 0; j < T::NT; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * T::WN + j * 8 + 2 * tig + h;
        if (row >= M || col >= N) continue;
        const double v = acc[i][j][h];
        if (split) {
          if (!syrk || row <= col) work[((long long)z * M + row) * N + col] = v;
        } else if (syrk) {
          if (row <= col) {
            double out = alpha * v;
            if (beta != 0.0) out = fma(beta, C[(long long)row * ldc + col], out);
            C[(long long)row * ldc + col] = out;
            if (row != col) C[(long long)col * ldc + row] = out;
          }
        } else {
          double out = alpha * v;
          if (beta != 0.0) out = fma(beta, C[(long long)row * ldc + col], out);
          C[(long long)row * ldc + col] = out;
        }
      }
    }
  }
}

__global__ void splitk_reduce_kernel(int M, int N, int S, const double* __restrict__ work, double alpha,
                                     double beta, double* __restrict__ C, long long ldc, int flags) {
  const bool syrk = (flags & LR_GEMM_SYRK_UPPER) != 0;
  const long long total = (long long)M * N;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(t / N), col = (int)(t - (long long)row * N);
    if (syrk && row > col) continue;
    double s = 0.0;
    for (int z = 0; z < S; ++z) s += work[(long long)z * total + t];
    double out = alpha * s;
    if (beta != 0.0) out = fma(beta, C[(long long)row * ldc + col], out);
    C[(long long)row * ldc + col] = out;
    if (syrk && row != col) C[(long long)col * ldc + row] = out;
  }
}

static int tile_pref(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

// 128x64 tiles for big products.  SYRK on square 64x64 tiles issues 9% less
// of the triangle but runs slower (2.20 vs 1.99 ms at 100000 x 660):
// LR_GEMM_SYRK_LARGE=0 selects it for experiments.
static bool use_large(int M, int N, long long K, int flags = 0) {
  static const int syrk_large = tile_pref("LR_GEMM_SYRK_LARGE", 1);
  if ((flags & LR_GEMM_SYRK_UPPER) && !syrk_large) return false;
  return (long long)M * N * K >= (1LL << 27) && M >= 128;
}

template <typename T, bool TA>
static int occupancy() {
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(gemm_kernel<T, TA>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_kernel<T, TA>, T::THREADS, T::SMEM);
    if (occ < 1) occ = 1;
  }
  return occ;
}

template <typename T>
static long long upper_tiles(int M, int N) {
  long long cnt = 0;
  const int tm_n = (M + T::BM - 1) / T::BM, tn_n = (N + T::BN - 1) / T::BN;
  for (int tm = 0; tm < tm_n; ++tm)
    for (int tn = 0; tn < tn_n; ++tn)
      if ((tn + 1) * T::BN > tm * T::BM) ++cnt;
  return cnt;
}

// split-K so the live CTAs fill whole waves of the GPU
template <typename T, bool TA>
static int choose_splits_t(int M, int N, int K, int flags) {
  if (!TA) return 1;
  long long tiles = (flags & LR_GEMM_SYRK_UPPER) ? upper_tiles<T>(M, N)
                                                 : (long long)((M + T::BM - 1) / T::BM) * ((N + T::BN - 1) / T::BN);
  // waves of split-K work: > 1 lets the block scheduler even out SMs that
  // drew short (diagonal, pruned) tiles (LR_GEMM_WAVES, experiments)
  static const int waves = tile_pref("LR_GEMM_WAVES", 1);
  const long long cap = (long long)sm_count() * occupancy<T, TA>() * waves;
  long long s = tiles >= cap ? 1 : cap / tiles;
  const long long smax = (K + 511) / 512;
  if (s > smax) s = smax;
  if (s < 1) s = 1;
  return (int)s;
}

// large-tile variant: 0 = 128x64 / 4 warps of 64x32, 1 = 128x64 / 8 warps
// of 32x32 (16 warps/SM keep the DMMA pipe fed through the fragment loads),
// 2 = 128x128 / 8 warps of 64x32, 3 = 0 with BK 32 / 2 stages (half the
// barriers per DMMA), 4 = 1 with BK 32 / 2 stages, 5 = 64x128 / 4 warps of
// 32x64, 6 = the TMA / mbarrier warp-specialised mainloop (lr_gemm_tma.cu).
// Measured (tools/gemm_probe.py, profiles/r01_gemm_variants.txt):
// A^T B (Gram) is fastest on 3 (1.95 ms at 100000 x 660; 0: 2.00, 1: 2.15),
// A B on 4 (H R^{-1} 2.00 -> 1.77 ms, H V 0.70 -> 0.60 ms).  LR_GEMM_TILE
// overrides.
static int large_variant(int transA) {
  static const int v = tile_pref("LR_GEMM_TILE", -1);
  if (v >= 0) return v;
  return transA ? 3 : 4;
}

bool gemm_tma_launch(int transA, int M, int N, int K, double alpha, const double* A, long long lda,
                     const double* B, long long ldb, double beta, double* C, long long ldc, int flags, double* work,
                     int S, int k_chunk, cudaStream_t s);
int gemm_tma_occupancy();

static int choose_splits(int transA, int M, int N, int K, int flags) {
  if (!transA) return 1;
  if (!use_large(M, N, K, flags)) return choose_splits_t<TileS, true>(M, N, K, flags);
  if (large_variant(1) == 6) {  // TMA mainloop: 128 x 64 tiles
    using T = TileL32;
    long long tiles = (flags & LR_GEMM_SYRK_UPPER) ? upper_tiles<T>(M, N)
                                                   : (long long)((M + T::BM - 1) / T::BM) * ((N + T::BN - 1) / T::BN);
    const long long cap = (long long)sm_count() * gemm_tma_occupancy();
    long long sp = tiles >= cap ? 1 : cap / tiles;
    const long long smax = (K + 511) / 512;
    if (sp > smax) sp = smax;
    return (int)(sp < 1 ? 1 : sp);
  }
  switch (large_variant(1)) {
    case 1: return choose_splits_t<TileL8, true>(M, N, K, flags);
    case 2: return choose_splits_t<TileW, true>(M, N, K, flags);
    case 3: return choose_splits_t<TileL32, true>(M, N, K, flags);
    case 4: return choose_splits_t<TileL832, true>(M, N, K, flags);
    case 5: return choose_splits_t<TileT, true>(M, N, K, flags);
    default: return choose_splits_t<TileL, true>(M, N, K, flags);
  }
}

template <typename T, bool TA>
static void launch(int M, int N, int K, double alpha, const double* A, long long lda, const double* B,
                   long long ldb, double beta, double* C, long long ldc, int flags, double* work, int S,
                   int k_chunk, int vec16, cudaStream_t s) {
  occupancy<T, TA>();
  dim3 grid((N + T::BN - 1) / T::BN, (M + T::BM - 1) / T::BM, S);
  gemm_kernel<T, TA><<<grid, T::THREADS, T::SMEM, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, flags, work,
                                                       k_chunk, vec16);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace lr

using namespace lr;

extern "C" {

long long lr_gemm_workspace_doubles(int transA, int M, int N, int K, int flags) {
  int s = choose_splits(transA, M, N, K, flags);
  return s > 1 ? (long long)s * M * N : 0;
}

int lr_gemm_f64(int transA, int M, int N, int K, double alpha, const double* A, long long lda,
                const double* B, long long ldb, double beta, double* C, long long ldc, int flags,
                double* work, long long work_doubles, void* stream) {
  LR_REQUIRE(M >= 0 && N >= 0 && K >= 0, "gemm: negative dims");
  LR_REQUIRE(ldc >= N && ldb >= N && lda >= (transA ? M : K), "gemm: bad leading dimensions");
  LR_REQUIRE(!(flags & LR_GEMM_SYRK_UPPER) || (transA && M == N), "gemm: SYRK needs transA, M == N");
  LR_REQUIRE(!(flags & LR_GEMM_B_UPPER) || (K == N), "gemm: B_UPPER needs K == N");
  if (M == 0 || N == 0) return LR_OK;
  cudaStream_t s = as_stream(stream);
  if (K == 0 && beta == 0.0) return lr_fill_f64(C, ldc, M, N, 0.0, stream);
  int S = choose_splits(transA, M, N, K, flags);
  if (S > 1 && (work == nullptr || work_doubles < (long long)S * M * N)) S = 1;
  int k_chunk = S > 1 ? ((K + S - 1) / S + BK_ALIGN - 1) / BK_ALIGN * BK_ALIGN : (K > 0 ? K : 1);
  if (S > 1) S = (K + k_chunk - 1) / k_chunk;
  const int vec16 = (lda % 2 == 0) && (ldb % 2 == 0) && aligned16(A) && aligned16(B);
  const bool large = use_large(M, N, K, flags);
  const int variant = large_variant(transA);
#define LR_GEMM_ARGS M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, flags, work, S, k_chunk, vec16, s
  if (large && variant == 6 &&
      gemm_tma_launch(transA, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, flags, work, S, k_chunk, s)) {
    // TMA + mbarrier mainloop (lr_gemm_tma.cu)
  } else if (transA) {
    if (!large)
      launch<TileS, true>(LR_GEMM_ARGS);
    else if (variant == 1)
      launch<TileL8, true>(LR_GEMM_ARGS);
    else if (variant == 2)
      launch<TileW, true>(LR_GEMM_ARGS);
    else if (variant == 3)
      launch<TileL32, true>(LR_GEMM_ARGS);
    else if (variant == 4)
      launch<TileL832, true>(LR_GEMM_ARGS);
    else if (variant == 5)
      launch<TileT, true>(LR_GEMM_ARGS);
    else
      launch<TileL, true>(LR_GEMM_ARGS);
  } else {
    if (!large)
      launch<TileS, false>(LR_GEMM_ARGS);
    else if (variant == 1)
      launch<TileL8, false>(LR_GEMM_ARGS);
    else if (variant == 2)
      launch<TileW, false>(LR_GEMM_ARGS);
    else if (variant == 3)
      launch<TileL32, false>(LR_GEMM_ARGS);
    else if (variant == 4)
      launch<TileL832, false>(LR_GEMM_ARGS);
    else if (variant == 5)
      launch<TileT, false>(LR_GEMM_ARGS);
    else
      launch<TileL, false>(LR_GEMM_ARGS);
  }
#undef LR_GEMM_ARGS
  LR_CHECK_LAUNCH();
  if (S > 1) {
    long long total = (long long)M * N;
    long long blocks = (total + 255) / 256;
    if (blocks > sm_count() * 8) blocks = sm_count() * 8;
    splitk_reduce_kernel<<<(int)blocks, 256, 0, s>>>(M, N, S, work, alpha, beta, C, ldc, flags);
    LR_CHECK_LAUNCH();
  }
  return LR_OK;
}

}  // extern "C"
