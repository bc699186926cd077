// Library plumbing: error strings, device facts, deterministic reductions,
// small utility kernels (copies, fills, column scaling, sign rule).
#include <atomic>
#include <cstdarg>
#include <cstdio>

#include <stdlib.h>

#include "lr_common.cuh"

namespace lr {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::atomic<long long> g_launches{0};
void count_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int env_int_clamped(const char* name, int dflt, int lo, int hi) {
  const char* v = getenv(name);
  int x = v ? atoi(v) : dflt;
  if (x < lo) x = lo;
  if (x > hi) x = hi;
  return x;
}

// The library serves ONE device per process (the framework runs one process
// per GPU; device.require_cuda enforces it), so the SM count and the
// per-kernel shared-memory opt-ins cached in function-local statics hold for
// the process's lifetime.
int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

// ---------------------------------------------------------------- stats
constexpr int kStatsBlocks = 296;
constexpr int kStatsThreads = 256;

__global__ void __launch_bounds__(kStatsThreads) block_stats_kernel(const double* __restrict__ X,
                                                                   long long rows, long long cols,
                                                                   long long ld, double* partial) {
  __shared__ double sh[32];
  double s = 0.0, mx = 0.0, bad = 0.0;
  auto acc = [&](double v) {
    if (!isfinite(v)) {
      bad += 1.0;
    } else {
      s = fma(v, v, s);
      mx = fmax(mx, fabs(v));
    }
  };
  if (ld == cols) {
    // contiguous: one flat grid-stride sweep, 4 independent loads per trip
    const long long total = rows * cols;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; t + 3 * stride < total; t += 4 * stride) {
      const double a = X[t], b = X[t + stride], c = X[t + 2 * stride], d = X[t + 3 * stride];
      acc(a);
      acc(b);
      acc(c);
      acc(d);
    }
    for (; t < total; t += stride) acc(X[t]);
  } else {
    // strided block: a warp per row, lanes across the columns (no 64-bit
    // index division per element)
    const int lane = threadIdx.x & 31;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (; r + 3 * nw < rows; r += 4 * nw) {  // four rows' loads in flight
      const double* r0 = X + r * ld;
      for (long long c = lane; c < cols; c += 32) {
        const double a = r0[c], b = r0[nw * ld + c], d = r0[2 * nw * ld + c], e = r0[3 * nw * ld + c];
        acc(a);
        acc(b);
        acc(d);
        acc(e);
      }
    }
    for (; r < rows; r += nw) {
      const double* row = X + r * ld;
      for (long long c = lane; c < cols; c += 32) acc(row[c]);
    }
  }
  double S = block_sum<kStatsThreads>(s, sh);
  double M = block_max<kStatsThreads>(mx, sh);
  double B = block_sum<kStatsThreads>(bad, sh);
  if (threadIdx.x == 0) {
    partial[3 * blockIdx.x + 0] = S;
    partial[3 * blockIdx.x + 1] = M;
    partial[3 * blockIdx.x + 2] = B;
  }
}

// One warp: lane-strided partial sums then a fixed shuffle tree (deterministic;
// all of a lane's loads are independent, unlike a single-thread serial sum)
__global__ void stats_finish_kernel(const double* partial, int n, double* out) {
  const int lane = threadIdx.x;
  double s = 0, m = 0, b = 0;
  for (int i = lane; i < n; i += 32) {
    s += partial[3 * i];
    m = fmax(m, partial[3 * i + 1]);
    b += partial[3 * i + 2];
  }
  s = warp_sum(s);
  m = warp_max(m);
  b = warp_sum(b);
  if (lane == 0) {
    out[0] = s;
    out[1] = m;
    out[2] = b;
  }
}

__global__ void __launch_bounds__(kStatsThreads) dot_kernel(const double* __restrict__ x,
                                                           const double* __restrict__ y,
                                                           long long n, double* partial) {
  __shared__ double sh[32];
  double s = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    s = fma(x[t], y[t], s);
  double S = block_sum<kStatsThreads>(s, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = S;
}

__global__ void sum_finish_kernel(const double* partial, int n, double* out) {
  const int lane = threadIdx.x;
  double s = 0;
  for (int i = lane; i < n; i += 32) s += partial[i];
  s = warp_sum(s);
  if (lane == 0) out[0] = s;
}

// power iteration: partial[0..B) = x.z partials, partial[B..2B) = z.z partials
__global__ void __launch_bounds__(kStatsThreads) power_dots_kernel(const double* __restrict__ x,
                                                                  const double* __restrict__ z,
                                                                  long long n, const double* state,
                                                                  double* partial) {
  if (state[2] != 0.0) return;  // converged: no-op
  __shared__ double sh[32];
  double a = 0.0, b = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x) {
    double zv = z[t];
    a = fma(x[t], zv, a);
    b = fma(zv, zv, b);
  }
  double A = block_sum<kStatsThreads>(a, sh);
  double B = block_sum<kStatsThreads>(b, sh);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = A;
    partial[gridDim.x + blockIdx.x] = B;
  }
}

// state = {prev, curr, done, iters, zero_hit, zn}
__global__ void power_scalar_kernel(const double* partial, int nb, double tol, double* state) {
  const int lane = threadIdx.x;
  if (lane >= 32 || blockIdx.x != 0) return;
  if (state[2] != 0.0) return;
  double lam = 0, zz = 0;
  for (int i = lane; i < nb; i += 32) {  // one warp, fixed-order folds
    lam += partial[i];
    zz += partial[nb + i];
  }
  lam = warp_sum(lam);
  zz = warp_sum(zz);
  if (lane != 0) return;
  double zn = sqrt(zz);
  state[0] = state[1];
  state[1] = sqrt(fmax(lam, 0.0));
  state[3] += 1.0;
  state[5] = zn;
  if (zn == 0.0) {
    state[4] = 1.0;
    state[2] = 1.0;
    return;
  }
  if (fabs(state[1] - state[0]) <= tol * fmax(state[1], 1e-300)) state[2] = 2.0;  // converged after x update
}

__global__ void power_scale_kernel(double* x, const double* z, long long n, const double* state) {
  // x = z / zn unless zero was hit (state[4]) or we had already converged before this step
  if (state[4] != 0.0) return;
  if (state[2] == 1.0) return;
  const double zn = state[5];
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (long long)gridDim.x * blockDim.x)
    x[t] = z[t] / zn;
}

__global__ void power_latch_kernel(double* state) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && state[2] == 2.0) state[2] = 1.0;
}

// ---------------------------------------------------------------- copies
__global__ void copy2d_kernel(const double* __restrict__ src, long long lds, double* __restrict__ dst,
                              long long ldd, long long rows, long long cols, int reverse) {
  const long long total = rows * cols;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long r = t / cols, c = t - r * cols;
    long long cs = reverse ? (cols - 1 - c) : c;
    dst[r * ldd + c] = src[r * lds + cs];
  }
}

// precision conversion of a strided block: a warp per row, lanes across the
// columns (no per-element index division); fp64 -> fp32 rounds to nearest
template <typename Src, typename Dst>
__global__ void convert2d_kernel(const Src* __restrict__ src, long long lds, Dst* __restrict__ dst, long long ldd,
                                 long long rows, long long cols) {
  if (rows == 1 || (lds == cols && ldd == cols)) {  // contiguous: one flat grid-stride sweep
    const long long total = rows * cols;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x)
      dst[t] = static_cast<Dst>(src[t]);
    return;
  }
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
    const Src* s = src + r * lds;
    Dst* d = dst + r * ldd;
    for (long long c = lane; c < cols; c += 32) d[c] = static_cast<Dst>(s[c]);
  }
}

__global__ void fill_kernel(double* dst, long long ld, long long rows, long long cols, double v) {
  const long long total = rows * cols;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long r = t / cols, c = t - r * cols;
    dst[r * ld + c] = v;
  }
}

__global__ void transpose_kernel(const double* __restrict__ src, long long lds, long long rows, long long cols,
                                 double* __restrict__ dst, long long ldd) {
  __shared__ double tile[32][33];
  const long long r0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    long long r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * lds + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    long long c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][i];
  }
}

__global__ void symmetrize_kernel(const double* __restrict__ src, long long lds, int n, double* __restrict__ dst,
                                  long long ldd) {
  const long long total = (long long)n * n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / n), c = (int)(t - (long long)i * n);
    dst[(long long)i * ldd + c] = 0.5 * (src[(long long)i * lds + c] + src[(long long)c * lds + i]);
  }
}

__global__ void diag_kernel(const double* __restrict__ A, long long lda, int n, double* __restrict__ d) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    d[i] = A[(long long)i * lda + i];
}

// dst[t] = src[perm[t]]: 4 coalesced perm words per thread, then their 4
// random reads in flight together (the random 8-byte reads are the cost:
// each moves a 32-byte sector)
__global__ void gather_kernel(const double* __restrict__ src, const int* __restrict__ perm,
                              double* __restrict__ dst, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; t + 3 * stride < n; t += 4 * stride) {
    int p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = __ldg(perm + t + k * stride);
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldg(src + p[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) dst[t + k * stride] = v[k];
  }
  for (; t < n; t += stride) dst[t] = __ldg(src + __ldg(perm + t));
}

// sign rule: one warp per column
__global__ void fix_signs_kernel(double* V, long long ldv, int rows_v, int cols, double* U,
                                 long long ldu, int rows_u) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= cols) return;
  const int j = warp;
  // first nonzero entry of V[:, j]
  int first = rows_v;
  for (int base = 0; base < rows_v && first == rows_v; base += 32) {
    int i = base + lane;
    bool nz = (i < rows_v) && (V[(long long)i * ldv + j] != 0.0);
    unsigned b = __ballot_sync(0xffffffffu, nz);
    if (b) first = base + __ffs(b) - 1;
  }
  if (first == rows_v) return;
  if (!(V[(long long)first * ldv + j] < 0.0)) return;
  for (int i = lane; i < rows_v; i += 32) V[(long long)i * ldv + j] = -V[(long long)i * ldv + j];
  if (U)
    for (int i = lane; i < rows_u; i += 32) U[(long long)i * ldu + j] = -U[(long long)i * ldu + j];
}

__global__ void scale_columns_kernel(const double* __restrict__ V, long long ldv, int rows,
                                     const int* __restrict__ cidx, int ncols, const double* S,
                                     int invert, double* __restrict__ B, long long ldb) {
  const long long total = (long long)rows * ncols;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    int r = (int)(t / ncols), c = (int)(t - (long long)r * ncols);
    int src = cidx ? cidx[c] : c;
    double s = S ? (invert ? 1.0 / S[src] : S[src]) : 1.0;
    B[(long long)r * ldb + c] = V[(long long)r * ldv + src] * s;
  }
}

__global__ void gram_spectrum_kernel(const double* __restrict__ d, int n, double* __restrict__ S) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) S[i] = sqrt(fmax(d[i], 0.0));
}

static int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  long long cap = (long long)sm_count() * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace lr

using namespace lr;

extern "C" {

int lr_version(void) { return 1; }
const char* lr_last_error(void) { return g_err; }
int lr_sm_count(void) { return sm_count(); }
long long lr_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
int lr_stats_partials(void) { return kStatsBlocks * 3; }
int lr_svt_step_partials_internal(void);

int lr_block_stats_f64(const double* X, long long rows, long long cols, long long ld,
                       double* partial, double* out3, void* stream) {
  LR_REQUIRE(rows >= 0 && cols >= 0 && ld >= cols, "block_stats: bad shape");
  cudaStream_t s = as_stream(stream);
  int nb = kStatsBlocks;
  if (rows * cols == 0) {
    fill_kernel<<<1, 32, 0, s>>>(out3, 3, 1, 3, 0.0);
    LR_CHECK_LAUNCH();
    return LR_OK;
  }
  block_stats_kernel<<<nb, kStatsThreads, 0, s>>>(X, rows, cols, ld, partial);
  LR_CHECK_LAUNCH();
  stats_finish_kernel<<<1, 32, 0, s>>>(partial, nb, out3);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_dot_f64(const double* x, const double* y, long long n, double* partial, double* out,
               void* stream) {
  cudaStream_t s = as_stream(stream);
  dot_kernel<<<kStatsBlocks, kStatsThreads, 0, s>>>(x, y, n, partial);
  LR_CHECK_LAUNCH();
  sum_finish_kernel<<<1, 32, 0, s>>>(partial, kStatsBlocks, out);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_power_update_f64(double* x, const double* z, long long n, double tol, double* state,
                        double* partial, void* stream) {
  cudaStream_t s = as_stream(stream);
  power_dots_kernel<<<kStatsBlocks, kStatsThreads, 0, s>>>(x, z, n, state, partial);
  LR_CHECK_LAUNCH();
  power_scalar_kernel<<<1, 32, 0, s>>>(partial, kStatsBlocks, tol, state);
  LR_CHECK_LAUNCH();
  power_scale_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, z, n, state);
  LR_CHECK_LAUNCH();
  power_latch_kernel<<<1, 32, 0, s>>>(state);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_copy2d_f64(const double* src, long long lds, double* dst, long long ldd, long long rows,
                  long long cols, int reverse_cols, void* stream) {
  if (rows * cols == 0) return LR_OK;
  copy2d_kernel<<<grid_for(rows * cols, 256), 256, 0, as_stream(stream)>>>(src, lds, dst, ldd, rows,
                                                                          cols, reverse_cols);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

static int convert_grid(long long rows, long long cols) {
  long long b = rows == 1 ? (cols + 255) / 256 : (rows + 7) / 8;  // flat, or 8 warps (rows) per block
  const long long cap = (long long)sm_count() * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

int lr_convert_f64_to_f32(const double* src, long long lds, float* dst, long long ldd, long long rows,
                          long long cols, void* stream) {
  LR_REQUIRE(rows >= 0 && cols >= 0 && lds >= cols && ldd >= cols, "convert: bad shape");
  if (rows * cols == 0) return LR_OK;
  convert2d_kernel<double, float><<<convert_grid(rows, cols), 256, 0, as_stream(stream)>>>(src, lds, dst, ldd, rows, cols);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_convert_f32_to_f64(const float* src, long long lds, double* dst, long long ldd, long long rows,
                          long long cols, void* stream) {
  LR_REQUIRE(rows >= 0 && cols >= 0 && lds >= cols && ldd >= cols, "convert: bad shape");
  if (rows * cols == 0) return LR_OK;
  convert2d_kernel<float, double><<<convert_grid(rows, cols), 256, 0, as_stream(stream)>>>(src, lds, dst, ldd, rows, cols);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_fill_f64(double* dst, long long ld, long long rows, long long cols, double v, void* stream) {
  if (rows * cols == 0) return LR_OK;
  fill_kernel<<<grid_for(rows * cols, 256), 256, 0, as_stream(stream)>>>(dst, ld, rows, cols, v);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_gather_f64(const double* src, const int* perm, double* dst, long long n, void* stream) {
  if (n == 0) return LR_OK;
  gather_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(src, perm, dst, n);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_transpose_f64(const double* src, long long lds, long long rows, long long cols, double* dst,
                     long long ldd, void* stream) {
  if (rows * cols == 0) return LR_OK;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(src, lds, rows, cols, dst, ldd);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_symmetrize_f64(const double* src, long long lds, int n, double* dst, long long ldd, void* stream) {
  if (n == 0) return LR_OK;
  symmetrize_kernel<<<grid_for((long long)n * n, 256), 256, 0, as_stream(stream)>>>(src, lds, n, dst, ldd);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_diag_f64(const double* A, long long lda, int n, double* d, void* stream) {
  if (n == 0) return LR_OK;
  diag_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(A, lda, n, d);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_fix_signs_f64(double* V, long long ldv, int rows_v, int cols, double* U, long long ldu,
                     int rows_u, void* stream) {
  if (cols == 0) return LR_OK;
  int threads = 256;
  int blocks = (cols * 32 + threads - 1) / threads;
  fix_signs_kernel<<<blocks, threads, 0, as_stream(stream)>>>(V, ldv, rows_v, cols, U, ldu, rows_u);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_gram_spectrum_f64(const double* d, int n, double* S, void* stream) {
  if (n <= 0) return LR_OK;
  gram_spectrum_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(d, n, S);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

int lr_scale_columns_f64(const double* V, long long ldv, int rows, const int* cols_idx, int ncols,
                         const double* S, int invert, double* B, long long ldb, void* stream) {
  if ((long long)rows * ncols == 0) return LR_OK;
  scale_columns_kernel<<<grid_for((long long)rows * ncols, 256), 256, 0, as_stream(stream)>>>(
      V, ldv, rows, cols_idx, ncols, S, invert, B, ldb);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

}  // extern "C"
