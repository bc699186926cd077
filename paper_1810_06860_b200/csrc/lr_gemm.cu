// fp64 GEMM on the tensor cores: mma.sync.aligned.m8n8k4.f64 (SASS
// DMMA.8x8x4; tcgen05 has no f64 kind).  Measured on this pool's B200:
// DMMA 37.1 TF/s vs DFMA 36.3 and cuBLAS DGEMM 35.4 (profiles/r01_fp64_peaks.txt).
//
// C[MxN] = alpha * op(A) * B + beta * C, row-major, arbitrary ld.
//   transA = 0: A is M x K  (tall A times small B: TRSM-as-GEMM, lifts, rescale)
//   transA = 1: A is K x M  (C = A^T B: Gram / projections, split-K over the
//               long K with partial tiles reduced in fixed order)
// CTA tile 64x64x16, 4 warps of 32x32, cp.async double buffering.
#include "lr_common.cuh"

namespace lr {

constexpr int BM = 64, BN = 64, BK = 16;
constexpr int WM = 32, WN = 32;
constexpr int MT = WM / 8, NT = WN / 8;
constexpr int GEMM_THREADS = 128;
constexpr int LDA_N = BK + 4;  // A stored [m][k] (transA = 0)
constexpr int LDA_T = BM + 4;  // A stored [k][m] (transA = 1)
constexpr int LDB = BN + 4;    // B stored [k][n]
constexpr int A_STAGE = (BM * LDA_N > BK * LDA_T) ? BM * LDA_N : BK * LDA_T;
constexpr int B_STAGE = BK * LDB;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src_size = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(src_size));
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

template <bool TRANS_A>
__global__ void __launch_bounds__(GEMM_THREADS) gemm_kernel(int M, int N, int K, double alpha,
                                                           const double* __restrict__ A, long long lda,
                                                           const double* __restrict__ B, long long ldb,
                                                           double beta, double* __restrict__ C,
                                                           long long ldc, int flags,
                                                           double* __restrict__ work, int k_chunk) {
  const int tn = blockIdx.x, tm = blockIdx.y, z = blockIdx.z;
  if ((flags & LR_GEMM_SYRK_UPPER) && tn < tm) return;
  __shared__ __align__(16) double As[2][A_STAGE];
  __shared__ __align__(16) double Bs[2][B_STAGE];

  const int m0 = tm * BM, n0 = tn * BN;
  int k_begin = z * k_chunk;
  int k_end = min(K, k_begin + k_chunk);
  if (flags & LR_GEMM_B_UPPER) k_end = min(k_end, n0 + BN);
  const int nk = (k_end > k_begin) ? (k_end - k_begin + BK - 1) / BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / (BN / WN), wn = warp % (BN / WN);
  const int gid = lane >> 2, tig = lane & 3;

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load_stage = [&](int st, int kt) {
    const int k0 = k_begin + kt * BK;
    double* as = As[st];
    double* bs = Bs[st];
    if (!TRANS_A) {
      // A[m][k]: 16 consecutive k per row (128 B)
#pragma unroll
      for (int i = 0; i < (BM * BK) / GEMM_THREADS; ++i) {
        const int e = tid + i * GEMM_THREADS;
        const int mm = e / BK, kk = e % BK;
        const int gm = m0 + mm, gk = k0 + kk;
        const bool ok = gm < M && gk < k_end;
        cp_async8(as + mm * LDA_N + kk, ok ? A + (long long)gm * lda + gk : A, ok);
      }
    } else {
      // A[k][m]: 64 consecutive m per k-row (512 B)
#pragma unroll
      for (int i = 0; i < (BM * BK) / GEMM_THREADS; ++i) {
        const int e = tid + i * GEMM_THREADS;
        const int kk = e / BM, mm = e % BM;
        const int gm = m0 + mm, gk = k0 + kk;
        const bool ok = gm < M && gk < k_end;
        cp_async8(as + kk * LDA_T + mm, ok ? A + (long long)gk * lda + gm : A, ok);
      }
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / GEMM_THREADS; ++i) {
      const int e = tid + i * GEMM_THREADS;
      const int kk = e / BN, nn = e % BN;
      const int gn = n0 + nn, gk = k0 + kk;
      const bool ok = gn < N && gk < k_end;
      cp_async8(bs + kk * LDB + nn, ok ? B + (long long)gk * ldb + gn : B, ok);
    }
    cp_async_commit();
  };

  if (nk > 0) load_stage(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    if (kt + 1 < nk) {
      load_stage((kt + 1) & 1, kt + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* as = As[kt & 1];
    const double* bs = Bs[kt & 1];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int mm = wm * WM + i * 8 + gid;
        af[i] = TRANS_A ? as[(kk + tig) * LDA_T + mm] : as[mm * LDA_N + kk + tig];
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = bs[(kk + tig) * LDB + wn * WN + j * 8 + gid];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }

  // epilogue
  const bool split = gridDim.z > 1;
  const bool syrk = (flags & LR_GEMM_SYRK_UPPER) != 0;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int row = m0 + wm * WM + i * 8 + gid;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * WN + j * 8 + 2 * tig + h;
        if (row >= M || col >= N) continue;
        const double v = acc[i][j][h];
        if (split) {
          work[((long long)z * M + row) * N + col] = v;
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

static int choose_splits(int transA, int M, int N, int K, int flags) {
  if (!transA) return 1;
  long long tiles = (long long)((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  if (flags & LR_GEMM_SYRK_UPPER) {
    long long t = (M + BM - 1) / BM;
    tiles = t * (t + 1) / 2;
  }
  const long long target = (long long)sm_count() * 4;
  long long s = (target + tiles - 1) / tiles;
  long long smax = (K + 255) / 256;
  if (s > smax) s = smax;
  if (s < 1) s = 1;
  return (int)s;
}

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
  if (K == 0) {
    // C = beta*C
    if (beta == 0.0) return lr_fill_f64(C, ldc, M, N, 0.0, stream);
  }
  int S = choose_splits(transA, M, N, K, flags);
  if (S > 1 && (work == nullptr || work_doubles < (long long)S * M * N)) S = 1;
  int k_chunk = S > 1 ? ((K + S - 1) / S + BK - 1) / BK * BK : (K > 0 ? K : 1);
  if (S > 1) S = (K + k_chunk - 1) / k_chunk;
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, S);
  if (transA)
    gemm_kernel<true><<<grid, GEMM_THREADS, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                                    flags, work, k_chunk);
  else
    gemm_kernel<false><<<grid, GEMM_THREADS, 0, s>>>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc,
                                                     flags, work, k_chunk);
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
