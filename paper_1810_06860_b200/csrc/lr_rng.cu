// Device Gaussian test matrix: gaussian_matrix(RngState(seed), rows, cols) of
// rng.py:77-94 without the host round trip.
//   stream : numpy Philox4x64-10, key = (seed, 0), 256-bit counter starting at
//            1 (numpy increments before generating), 4 uint64 per counter;
//   uniform: (x >> 11) * 2^-53                                  (bit-exact)
//   normals: Box-Muller over the whole request of 2*ceil(k/2) uniforms,
//            u1 = 1 - u[i], u2 = u[P + i]; z[2i] = rho cos, z[2i+1] = rho sin
//            (rng.py:38-55)                       (libdevice log/sincos: <= 2 ulp)
//   layout : column-major fill, row-major storage                (rng.py:93-94)
#include "lr_common.cuh"

namespace lr {

struct U64x4 {
  unsigned long long v[4];
};

__device__ __forceinline__ void mulhilo(unsigned long long a, unsigned long long b, unsigned long long& hi,
                                        unsigned long long& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

__device__ __forceinline__ U64x4 philox4x64_10(U64x4 c, unsigned long long k0, unsigned long long k1) {
  const unsigned long long M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const unsigned long long W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    unsigned long long hi0, lo0, hi1, lo1;
    mulhilo(M0, c.v[0], hi0, lo0);
    mulhilo(M1, c.v[2], hi1, lo1);
    U64x4 o;
    o.v[0] = hi1 ^ c.v[1] ^ k0;
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ k1;
    o.v[3] = lo0;
    c = o;
  }
  return c;
}

// uniform number t of the stream (t = 0, 1, ...): block t/4 uses counter t/4 + 1
__device__ __forceinline__ double philox_uniform(unsigned long long seed, unsigned long long t) {
  U64x4 c;
  const unsigned long long blk = (t >> 2) + 1ULL;
  c.v[0] = blk;
  c.v[1] = 0;
  c.v[2] = 0;
  c.v[3] = 0;
  U64x4 o = philox4x64_10(c, seed, 0ULL);
  const unsigned long long x = o.v[t & 3];
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void gaussian_kernel(unsigned long long seed, int rows, int cols, double* __restrict__ omega,
                                long long ldo) {
  const long long count = (long long)rows * cols;
  const long long pairs = (count + 1) / 2;
  const double two_pi = 2.0 * 3.141592653589793;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < pairs;
       i += (long long)gridDim.x * blockDim.x) {
    const double u1 = 1.0 - philox_uniform(seed, (unsigned long long)i);
    const double u2 = philox_uniform(seed, (unsigned long long)(pairs + i));
    const double rho = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincos(two_pi * u2, &sn, &cs);
    const long long z0 = 2 * i, z1 = 2 * i + 1;
    // z index -> (row, col) of the column-major fill
    omega[(z0 % rows) * ldo + z0 / rows] = rho * cs;
    if (z1 < count) omega[(z1 % rows) * ldo + z1 / rows] = rho * sn;
  }
}

// Omega (rows x cols, row-major) from the host-computed Box-Muller halves of a
// rng.Superset: z[2i] = R[i] * cs[2 (off + i)], z[2i + 1] = R[i] * cs[2 (off + i) + 1]
// (one IEEE multiply each, __dmul_rn: the bits of lr_host_bm_assemble), z filling
// Omega column-major.  A thread per element, column fastest (coalesced stores).
__global__ void omega_assemble_kernel(const double* __restrict__ R, const double* __restrict__ cs, long long off,
                                      int rows, int cols, double* __restrict__ omega, long long ldo) {
  const long long count = (long long)rows * cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(e / cols), col = (int)(e - (long long)row * cols);
    const long long t = (long long)col * rows + row;
    const long long i = t >> 1;
    omega[(long long)row * ldo + col] = __dmul_rn(__ldg(R + i), __ldg(cs + 2 * (off + i) + (t & 1)));
  }
}

}  // namespace lr

using namespace lr;

extern "C" int lr_omega_assemble_f64(const double* R, const double* cs, long long off, int rows, int cols,
                                     double* omega, long long ldo, void* stream) {
  LR_REQUIRE(rows >= 1 && cols >= 1, "omega_assemble needs rows, cols >= 1, got %dx%d", rows, cols);
  LR_REQUIRE(ldo >= cols && off >= 0 && R && cs, "omega_assemble: bad arguments (ldo=%lld off=%lld)", ldo, off);
  const long long count = (long long)rows * cols;
  long long blocks = (count + 255) / 256;
  if (blocks > sm_count() * 16) blocks = sm_count() * 16;
  omega_assemble_kernel<<<(int)blocks, 256, 0, as_stream(stream)>>>(R, cs, off, rows, cols, omega, ldo);
  LR_CHECK_LAUNCH();
  return LR_OK;
}

extern "C" int lr_gaussian_f64(unsigned long long seed, int rows, int cols, double* omega, long long ldo,
                               void* stream) {
  LR_REQUIRE(rows >= 1 && cols >= 1, "gaussian matrix needs rows, cols >= 1, got %dx%d", rows, cols);
  LR_REQUIRE(ldo >= cols, "gaussian: ldo < cols");
  const long long pairs = ((long long)rows * cols + 1) / 2;
  long long blocks = (pairs + 255) / 256;
  if (blocks > sm_count() * 8) blocks = sm_count() * 8;
  gaussian_kernel<<<(int)blocks, 256, 0, as_stream(stream)>>>(seed, rows, cols, omega, ldo);
  LR_CHECK_LAUNCH();
  return LR_OK;
}
