// fp32-mode Gram on the 5th-generation tensor cores: G = A^T A of a tall
// fp32 block A (K x n, row-major), the eigSVD Gram of linalg.py:189 in the
// optional fp32 mode (north_star (2)).  tcgen05.mma kind::tf32 with the
// 3xTF32 split -- a = hi + lo, both tf32, G ~ hi.hi + hi.lo + lo.hi -- so the
// products carry ~22 mantissa bits; the accumulators live in TMEM (fp32,
// 128 lanes x 128 columns each), one 128 x 128 tile of G per CTA over a chunk
// of <= 2048 rows of A, and the chunk partials are summed in fp64 in a fixed
// order by a second kernel (deterministic, no atomics).  The tensor core's
// fp32 accumulation is not round-to-nearest: every MMA into an accumulator
// loses ~0.4 ulp of it on average (one accumulator over 4096 rows: 4e-5
// relative on the diagonal, r02ee), so the hi.hi products rotate over three
// accumulators and the small hi.lo / lo.hi terms go to a fourth (85
// roundings per accumulator and chunk, summed in the epilogue).  Only tiles with
// ti <= tj run; the reduction mirrors them, so G is exactly symmetric.
//
// Staging: the fp32 -> (hi, lo) split needs the values in registers, so the
// 256 threads load A's rows themselves (each warp reads 32 consecutive
// columns of one row: 128-byte coalesced) and store both parts into the
// canonical K-major SWIZZLE_128B layout the UMMA descriptors read: operand
// row x (a column of A), k = row of A within the 32-row stage; element
// (x, k) at (x / 8) * 1024 + (x % 8) * 128 + (((k / 4) ^ (x % 8)) * 16) +
// (k % 4) * 4.  A quarter-warp's 16-byte stores (x .. x + 7, same k / 4) hit
// 8 different 16-byte bank groups.  Two stages: the loads of stage kb + 1
// are in flight while the tensor core runs stage kb's 12 MMAs; a stage is
// rewritten only after the tcgen05.commit of the MMAs that read it arrived
// on its mbarrier.
#include "lr_common.cuh"

namespace lr {
namespace tc {

constexpr int TILE = 128;                   // G tile: UMMA M = N = 128
constexpr int BK = 32;                      // rows of A per stage: 32 tf32 = one 128-byte swizzle row
constexpr int STAGES = 2;
constexpr int THREADS = 256;
constexpr int UMMA_K = 8;                   // kind::tf32: K = 32 bytes per instruction
constexpr int OP_BYTES = TILE * BK * 4;     // one operand part (hi or lo): 16 KB
constexpr int STAGE_BYTES = 4 * OP_BYTES;   // A hi, A lo, B hi, B lo
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 64;
constexpr int MAX_CHUNK = 2048;             // rows per fp32 TMEM accumulation
constexpr int N_MAIN = 3;                   // rotating hi.hi accumulators (+1 for the hi.lo / lo.hi terms)
constexpr int TMEM_COLS = 512;              // (N_MAIN + 1) x 128 columns, rounded to a power of two

// instruction descriptor: D f32 (bits 4-5 = 1), A / B tf32 (bits 7-9, 10-12 = 2),
// both K-major (bits 15, 16 = 0), N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t IDESC =
    (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TILE >> 3) << 17) | ((uint32_t)(TILE >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// shared-memory matrix descriptor, K-major SWIZZLE_128B: start address >> 4,
// leading byte offset 1 (unused by the swizzled K-major form), stride byte
// offset 1024 B between 8-row groups, version 1 (bit 46), layout 2 (bits 61-63)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ uint32_t to_tf32(float f) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(f));
  return r;
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

// bounded wait: a commit that never arrives traps (a launch error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  for (long long spin = 0;; ++spin) {
    uint32_t done;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1ll << 26)) __trap();
  }
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}

__device__ __forceinline__ void tile_of(int t, int nt, int* ti, int* tj) {
  int i = 0;
  while (t >= nt - i) {
    t -= nt - i;
    ++i;
  }
  *ti = i;
  *tj = i + t;
}

__global__ void __launch_bounds__(THREADS, 1)
    gram_tf32x3_kernel(const float* __restrict__ A, long long lda, int K, int n, int nt, int chunk_rows,
                       float* __restrict__ part) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + ((1024u - (raw & 1023u)) & 1023u);  // swizzle atoms are 1024-aligned
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + STAGES * STAGE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + STAGES);

  int ti, tj;
  tile_of(blockIdx.x, nt, &ti, &tj);
  const bool diag = ti == tj;
  const int r0 = blockIdx.y * chunk_rows;
  const int rend = min(K, r0 + chunk_rows);
  const int nkb = (rend - r0 + BK - 1) / BK;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  const int x = tid & (TILE - 1);  // operand row = column of A within the tile
  const int kq = (tid >> 7) * 16;  // this thread's 16 rows of the 32-row stage
  const int ci = ti * TILE + x, cj = tj * TILE + x;
  const bool in_i = ci < n, in_j = cj < n;
  const uint32_t xoff = (uint32_t)(x >> 3) * 1024u + (uint32_t)(x & 7) * 128u;

  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb % STAGES;
    const int rb = r0 + kb * BK + kq;
    float va[16], vb[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int r = rb + q;
      const bool rin = r < rend;
      va[q] = (rin && in_i) ? __ldg(A + (long long)r * lda + ci) : 0.f;
      vb[q] = (!diag && rin && in_j) ? __ldg(A + (long long)r * lda + cj) : 0.f;
    }
    if (kb >= STAGES) mbar_wait(&bars[s], ((kb - STAGES) / STAGES) & 1);
    unsigned char* st = smem + s * STAGE_BYTES;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = kq + 4 * q;
      const uint32_t off = xoff + ((uint32_t)((k >> 2) ^ (x & 7)) << 4);
      uint32_t h[4], l[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        h[e] = to_tf32(va[4 * q + e]);
        l[e] = to_tf32(va[4 * q + e] - __uint_as_float(h[e]));
      }
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(st + off)), "r"(h[0]), "r"(h[1]),
                   "r"(h[2]), "r"(h[3]));
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(st + OP_BYTES + off)), "r"(l[0]),
                   "r"(l[1]), "r"(l[2]), "r"(l[3]));
      if (!diag) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          h[e] = to_tf32(vb[4 * q + e]);
          l[e] = to_tf32(vb[4 * q + e] - __uint_as_float(h[e]));
        }
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(st + 2 * OP_BYTES + off)),
                     "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(st + 3 * OP_BYTES + off)),
                     "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]));
      }
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      fence_after();
      const uint32_t sa = smem_u32(st);
      const uint64_t a_hi = sw128_desc(sa), a_lo = sw128_desc(sa + OP_BYTES);
      const uint64_t b_hi = diag ? a_hi : sw128_desc(sa + 2 * OP_BYTES);
      const uint64_t b_lo = diag ? a_lo : sw128_desc(sa + 3 * OP_BYTES);
#pragma unroll
      for (int k = 0; k < BK / UMMA_K; ++k) {
        const uint64_t adv = (uint64_t)((k * UMMA_K * 4) >> 4);  // K step inside the 128-byte swizzle row
        const int step = kb * (BK / UMMA_K) + k;
        const uint32_t d_main = tmem + (uint32_t)((step % N_MAIN) * TILE);
        const uint32_t d_corr = tmem + (uint32_t)(N_MAIN * TILE);
        umma_tf32(d_main, a_hi + adv, b_hi + adv, step >= N_MAIN);
        umma_tf32(d_corr, a_hi + adv, b_lo + adv, step != 0);
        umma_tf32(d_corr, a_lo + adv, b_hi + adv, 1u);
      }
      umma_commit(&bars[s]);  // arrives when these MMAs (and all earlier ones) completed
    }
  }
  // the last commit covers every MMA of the tile
  const int last = nkb - 1;
  mbar_wait(&bars[last % STAGES], (last / STAGES) & 1);
  fence_after();

  // epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31, columns 64 (w / 4) .. + 63
  const int lrow = (warp & 3) * 32 + lane;
  const int c0 = (warp >> 2) * 64;
  float* out = part + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * (TILE * TILE) + (size_t)lrow * TILE + c0;
  const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    float v[16], w[16];
    tmem_ld16(taddr + 16 * h, v);
#pragma unroll
    for (int a = 1; a <= N_MAIN; ++a) {  // fixed order: ((M0 + M1) + M2) + C
      tmem_ld16(taddr + (uint32_t)(a * TILE) + 16 * h, w);
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] += w[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      reinterpret_cast<float4*>(out + 16 * h)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
  }
}

// G[i][j] = G[j][i] = sum over chunks (fixed order, fp64) of the tile partials, i <= j
__global__ void gram_reduce_kernel(const float* __restrict__ part, int nchunks, int ntiles, int nt, int n,
                                   double* __restrict__ G, long long ldg) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)ntiles * TILE * TILE) return;
  const int tile = (int)(idx / (TILE * TILE)), e = (int)(idx % (TILE * TILE));
  int ti, tj;
  tile_of(tile, nt, &ti, &tj);
  const int i = ti * TILE + e / TILE, j = tj * TILE + e % TILE;
  if (i >= n || j >= n || i > j) return;
  double s = 0.0;
  for (int c = 0; c < nchunks; ++c) s += (double)part[((size_t)c * ntiles + tile) * (TILE * TILE) + e];
  G[(long long)i * ldg + j] = s;
  G[(long long)j * ldg + i] = s;
}

struct Plan {
  int nt, ntiles, chunk_rows, nchunks;
};

static Plan plan(int K, int n) {
  Plan p;
  p.nt = (n + TILE - 1) / TILE;
  p.ntiles = p.nt * (p.nt + 1) / 2;
  // about two CTAs per SM in total (one resident at a time: 128 KB of stages)
  const int want = (2 * sm_count() + p.ntiles - 1) / p.ntiles;
  int rows = (K + want - 1) / want;
  rows = (rows + BK - 1) / BK * BK;
  p.chunk_rows = rows < 4 * BK ? 4 * BK : (rows > MAX_CHUNK ? MAX_CHUNK : rows);
  p.nchunks = K > 0 ? (K + p.chunk_rows - 1) / p.chunk_rows : 0;
  return p;
}

}  // namespace tc
}  // namespace lr

using namespace lr;

extern "C" {

long long lr_gram_tf32x3_workspace_floats(int K, int n) {
  if (K <= 0 || n <= 0) return 0;
  const tc::Plan p = tc::plan(K, n);
  return (long long)p.nchunks * p.ntiles * tc::TILE * tc::TILE;
}

int lr_gram_tf32x3(const float* A, long long lda, int K, int n, double* G, long long ldg, float* work,
                   long long work_floats, void* stream) {
  LR_REQUIRE(K >= 0 && n >= 0, "gram_tf32x3: negative shape %d x %d", K, n);
  if (n == 0) return LR_OK;
  LR_REQUIRE(ldg >= n && lda >= n, "gram_tf32x3: leading dimensions %lld / %lld below n = %d", lda, ldg, n);
  cudaStream_t st = as_stream(stream);
  if (K == 0) {
    LR_CHECK_CUDA(cudaMemset2DAsync(G, (size_t)ldg * 8, 0, (size_t)n * 8, n, st));
    return LR_OK;
  }
  const tc::Plan p = tc::plan(K, n);
  LR_REQUIRE(work_floats >= (long long)p.nchunks * p.ntiles * tc::TILE * tc::TILE,
             "gram_tf32x3: workspace of %lld floats, need %lld", work_floats,
             (long long)p.nchunks * p.ntiles * tc::TILE * tc::TILE);
  static bool attr = false;
  if (!attr) {
    LR_CHECK_CUDA(cudaFuncSetAttribute(tc::gram_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM));
    attr = true;
  }
  tc::gram_tf32x3_kernel<<<dim3(p.ntiles, p.nchunks), tc::THREADS, tc::SMEM, st>>>(A, lda, K, n, p.nt, p.chunk_rows,
                                                                                   work);
  LR_CHECK_LAUNCH();
  const long long total = (long long)p.ntiles * tc::TILE * tc::TILE;
  tc::gram_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(work, p.nchunks, p.ntiles, p.nt, n, G, ldg);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

}  // extern "C"
