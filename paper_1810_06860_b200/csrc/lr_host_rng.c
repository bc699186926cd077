/* Host side of the parity Omega (rng.py:38-55, 77-94 of the reference): the
 * two pieces of numpy's draw that are plain C -- the Philox4x64-10 uniform
 * stream and the Box-Muller pairing with libm cos/sin -- so a draw costs no
 * numpy temporaries.  The log stays numpy's own (np.log is its SIMD kernel on
 * AVX-512 hosts, not libm); paper_1810_06860_b200/rng.py composes the three
 * and checks the result against the all-numpy draw bit for bit before using
 * it on a host.
 *
 * Compiled by gcc with -fno-fast-math -ffp-contract=off: every operation is
 * the IEEE operation numpy performs, in numpy's order. */
#include <math.h>
#include <stdint.h>

typedef unsigned __int128 u128;

static void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
  const uint64_t W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    const u128 p0 = (u128)M0 * c[0];
    const u128 p1 = (u128)M1 * c[2];
    const uint64_t hi0 = (uint64_t)(p0 >> 64), lo0 = (uint64_t)p0;
    const uint64_t hi1 = (uint64_t)(p1 >> 64), lo1 = (uint64_t)p1;
    const uint64_t o0 = hi1 ^ c[1] ^ k0, o2 = hi0 ^ c[3] ^ k1;
    c[0] = o0;
    c[1] = lo1;
    c[2] = o2;
    c[3] = lo0;
  }
}

/* out[i] = uniform (start + i) of numpy's Philox(key=seed) stream:
 * block b = t / 4 uses counter b + 1 (numpy increments before generating),
 * word t % 4; uniform = (x >> 11) * 2^-53. */
void lr_host_uniforms(unsigned long long seed, long long start, long long count, double* out) {
  long long t = start;
  const long long end = start + count;
  double* o = out;
  while (t < end) {
    uint64_t c[4] = {(uint64_t)(t >> 2) + 1u, 0u, 0u, 0u};
    philox4x64_10(c, (uint64_t)seed, 0u);
    for (int w = (int)(t & 3); w < 4 && t < end; ++w, ++t) *o++ = (double)(c[w] >> 11) * (1.0 / 9007199254740992.0);
  }
}

/* Box-Muller of n pairs: logs[i] = log(1 - u[i]) (numpy's), u2[i] = u[P + i];
 * z[2i] = sqrt(-2 logs[i]) cos(2 pi u2[i]), z[2i+1] = ... sin(...). */
void lr_host_box_muller(const double* logs, const double* u2, long long n, double* z) {
  const double two_pi = 2.0 * 3.141592653589793;
  for (long long i = 0; i < n; ++i) {
    const double radius = sqrt(-2.0 * logs[i]);
    const double angle = two_pi * u2[i];
    z[2 * i] = radius * cos(angle);
    z[2 * i + 1] = radius * sin(angle);
  }
}

/* cs[2j] = cos(2 pi u[j]), cs[2j+1] = sin(2 pi u[j]): the angle halves of
 * Box-Muller for a run of stream positions (shared by several draw widths). */
void lr_host_cossin(const double* u, long long n, double* cs) {
  const double two_pi = 2.0 * 3.141592653589793;
  for (long long j = 0; j < n; ++j) {
    const double angle = two_pi * u[j];
    cs[2 * j] = cos(angle);
    cs[2 * j + 1] = sin(angle);
  }
}

/* z[2i] = R[i] * cs[2i], z[2i+1] = R[i] * cs[2i+1] (R[i] = sqrt(-2 log(1 - u[i])))
 * -- numpy's radius * cos(angle), radius * sin(angle). */
void lr_host_bm_assemble(const double* R, const double* cs, long long n, double* z) {
  for (long long i = 0; i < n; ++i) {
    z[2 * i] = R[i] * cs[2 * i];
    z[2 * i + 1] = R[i] * cs[2 * i + 1];
  }
}
