// fp64 GEMM mainloop fed by the Tensor Memory Accelerator: tensor-map TMA
// loads (cp.async.bulk.tensor, SWIZZLE_128B) into a 4-stage shared-memory
// ring, full / empty mbarriers, one producer warp, 8 DMMA consumer warps
// (mma.sync m8n8k4 f64 -- tcgen05 has no f64 kind).  Same contract and
// epilogue as gemm_kernel in lr_gemm.cu (alpha / beta, split-K partials,
// SYRK upper tiles mirrored, B upper-triangular pruning).
//
// Layout: every TMA box is 16 doubles (128 B) wide, so a smem row is one
// 128-byte line whose 16-byte chunks the hardware XOR-swizzles by
// (row mod 8); the DMMA fragment reads apply the same XOR, and the 8 rows a
// fragment touches land in 8 different bank groups.
//   A (M x K, !TRANS_A):  one box {16 k, 128 m}  -> smem [m][16]
//   A (K x M,  TRANS_A):  8 boxes {16 m, 16 k}   -> smem [box][k][16]
//   B (K x N):            4 boxes {16 n, 16 k}   -> smem [box][k][16]
// Out-of-range rows / columns of a box are zero-filled by the TMA unit.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "lr_common.cuh"

#ifndef LR_GEMM_TMA_MINB
#define LR_GEMM_TMA_MINB 1  // 132 registers, no spills (2: 96 registers, ~230 B spilled)
#endif

namespace lr {

namespace tma {

constexpr int BM = 128, BN = 64, BK = 16, STAGES = 4;
constexpr int WM = 32, WN = 32, MT = WM / 8, NT = WN / 8;
constexpr int CWARPS = (BM / WM) * (BN / WN);  // 8 consumer warps
constexpr int THREADS = (CWARPS + 1) * 32;      // + 1 producer warp
constexpr int A_STAGE = BM * BK;                // doubles
constexpr int B_STAGE = BK * BN;
constexpr int STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 2 * STAGES * 8;  // ring + alignment slack + barriers

__device__ __forceinline__ int swz(int row, int col) {  // element offset of (row, col) in a 16-wide swizzled row
  return row * 16 + ((((col >> 1) ^ (row & 7)) << 1) | (col & 1));
}

// Fragment row / column permutations that keep the swizzled fragment reads
// conflict-free (a 64-bit warp load is two 16-lane wavefronts; each must hit
// 16 distinct bank pairs).  A DMMA tile's row r comes from the lanes with
// gid = r and its column c from the B lanes with gid = c, so permuting which
// matrix row / column a lane reads only relabels C: the epilogue applies the
// same maps.
//   [k][x] boxes (B, and A when TRANS_A): x = 16 (g >> 2) + 8 ((g >> 1) & 1) + 2 f + (g & 1)
//   [m][k] box  (A when !TRANS_A):        m = 8 f + 2 (g & 3) + (g >> 2)
__device__ __forceinline__ int kx_map(int f, int g) { return 16 * (g >> 2) + 8 * ((g >> 1) & 1) + 2 * f + (g & 1); }
__device__ __forceinline__ int mk_map(int f, int g) { return 8 * f + 2 * (g & 3) + (g >> 2); }

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool TRANS_A>
__global__ void __launch_bounds__(THREADS, LR_GEMM_TMA_MINB) gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                                                           const __grid_constant__ CUtensorMap tmB, int M, int N,
                                                           int K, double alpha, double beta,
                                                           double* __restrict__ C, long long ldc, int flags,
                                                           double* __restrict__ work, int k_chunk) {
  const int tn = blockIdx.x, tm = blockIdx.y, z = blockIdx.z;
  if ((flags & LR_GEMM_SYRK_UPPER) && (tn + 1) * BN <= tm * BM) return;  // tile entirely below the diagonal
  extern __shared__ unsigned char g_raw[];
  // SWIZZLE_128B needs 1024-byte aligned destinations
  double* ring = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(g_raw) + 1023) & ~uintptr_t(1023));
  unsigned long long* full = reinterpret_cast<unsigned long long*>(ring + STAGES * (A_STAGE + B_STAGE));
  unsigned long long* empty = full + STAGES;

  const int m0 = tm * BM, n0 = tn * BN;
  const int k_begin = z * k_chunk;
  int k_end = min(K, k_begin + k_chunk);
  if (flags & LR_GEMM_B_UPPER) k_end = min(k_end, n0 + BN);
  const int nk = (k_end > k_begin) ? (k_end - k_begin + BK - 1) / BK : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == CWARPS) {  // producer
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(empty + s, ((kt / STAGES) - 1) & 1);
        double* as = ring + s * (A_STAGE + B_STAGE);
        double* bs = as + A_STAGE;
        const int k0 = k_begin + kt * BK;
        mbar_expect_tx(full + s, STAGE_BYTES);
        if (TRANS_A) {
#pragma unroll
          for (int b = 0; b < BM / 16; ++b) tma_load_2d(as + b * 256, &tmA, m0 + 16 * b, k0, full + s);
        } else {
          tma_load_2d(as, &tmA, k0, m0, full + s);
        }
#pragma unroll
        for (int b = 0; b < BN / 16; ++b) tma_load_2d(bs + b * 256, &tmB, n0 + 16 * b, k0, full + s);
      }
    }
    return;
  }

  const int wm = warp / (BN / WN), wn = warp % (BN / WN);
  const int gid = lane >> 2, tig = lane & 3;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  bool warp_live;
  int warp_klim;
  {
    const int rbase = m0 + wm * WM, cbase = n0 + wn * WN;
    warp_live = rbase < M && cbase < N;
    if ((flags & LR_GEMM_SYRK_UPPER) && cbase + WN - 1 < rbase) warp_live = false;
    warp_klim = (flags & LR_GEMM_B_UPPER) ? min(k_end, cbase + WN) : k_end;
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(full + s, (kt / STAGES) & 1);
    const double* as = ring + s * (A_STAGE + B_STAGE);
    const double* bs = as + A_STAGE;
    if (warp_live && k_begin + kt * BK < warp_klim) {
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        const int k = kk + tig;
        double af[MT], bf[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int m = wm * WM + (TRANS_A ? kx_map(i, gid) : mk_map(i, gid));
          af[i] = TRANS_A ? as[(m >> 4) * 256 + swz(k, m & 15)] : as[swz(m, k)];
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int n = wn * WN + kx_map(j, gid);
          bf[j] = bs[(n >> 4) * 256 + swz(k, n & 15)];
        }
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
  }

  const bool split = gridDim.z > 1;
  const bool syrk = (flags & LR_GEMM_SYRK_UPPER) != 0;
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int row = m0 + wm * WM + (TRANS_A ? kx_map(i, gid) : mk_map(i, gid));
#pragma unroll
    for (int j = 0; j < NT; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + wn * WN + kx_map(j, 2 * tig + h);
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

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// a 2-D row-major fp64 tensor (rows x cols, leading dimension ld) with 16 x box_rows boxes
static bool make_map(CUtensorMap* map, const double* base, long long rows, long long cols, long long ld,
                     int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  cuuint32_t box[2] = {16u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace tma

// Launch the TMA mainloop; false when the operands do not meet TMA's rules
// (16-byte aligned base, ld a multiple of 2 doubles) or the driver entry
// point is missing -- the caller then uses the cp.async kernel.
bool gemm_tma_launch(int transA, int M, int N, int K, double alpha, const double* A, long long lda,
                     const double* B, long long ldb, double beta, double* C, long long ldc, int flags, double* work,
                     int S, int k_chunk, cudaStream_t s) {
  using namespace tma;
  if ((reinterpret_cast<uintptr_t>(A) & 15u) || (reinterpret_cast<uintptr_t>(B) & 15u) || (lda & 1) || (ldb & 1))
    return false;
  CUtensorMap mA, mB;
  const bool okA = transA ? make_map(&mA, A, K, M, lda, BK) : make_map(&mA, A, M, K, lda, BM);
  if (!okA || !make_map(&mB, B, K, N, ldb, BK)) return false;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(gemm_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, S);
  if (transA)
    gemm_tma_kernel<true><<<grid, THREADS, SMEM, s>>>(mA, mB, M, N, K, alpha, beta, C, ldc, flags, work, k_chunk);
  else
    gemm_tma_kernel<false><<<grid, THREADS, SMEM, s>>>(mA, mB, M, N, K, alpha, beta, C, ldc, flags, work, k_chunk);
  return true;
}

int gemm_tma_occupancy() {
  using namespace tma;
  static int occ = -1;
  if (occ < 0) {
    cudaFuncSetAttribute(gemm_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_tma_kernel<true>, THREADS, SMEM);
    if (occ < 1) occ = 1;
  }
  return occ;
}

}  // namespace lr
