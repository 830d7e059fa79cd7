/* TEST INFRASTRUCTURE ONLY — host restatement of the DEVICE synthetic-data
 * generator (skr_data_generate, paper_1602_02350_b200/csrc/capi.cu +
 * rng.cuh philox_normal2), so the CPU reference (goldens, bench.py's
 * --impl reference arm) consumes the same instance the GPU generates and times.
 *
 * Not a reference algorithm: BASELINE.json defines the instances
 * (X = G diag(sigma) V^T, w* ~ N(0, I/d), y = X w* + tau z) and SURVEY §8(d)
 * leaves the data RNG to the builder.  The device uses Philox4x32-10 (Salmon et
 * al., SC'11) with one counter stream per quantity:
 *   stream 1: G, element (row, col) of the n x d matrix = normal #(row*d + col)
 *   stream 2: the d x d Gaussian whose QR gives the Haar V
 *   stream 3: |Student-t(3)| row factors (c4), normals 4*row .. 4*row+3
 *   stream 4: w*
 *   stream 5: label noise, normal #row
 * Normal #t of a stream is component (t & 1) of the Box-Muller pair of counter
 * t >> 1.  Integer parts are bit-exact with the device; log / sqrt / sincospi
 * may differ from the device's in the last fp64 bit, so fp64 instances agree to
 * a few ulps and fp32 instances (rounded) agree except for rare ties.
 *
 * The d x d QR and the product G V^T are done by the Python wrapper
 * (oracle/__init__.py: synth_instance) with numpy.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>

typedef struct { uint32_t v[4]; } u32x4;

static u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  for (int i = 0; i < 10; ++i) {
    const uint64_t p0 = (uint64_t)M0 * c.v[0], p1 = (uint64_t)M1 * c.v[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    u32x4 o;
    o.v[0] = hi1 ^ c.v[1] ^ k0;
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ k1;
    o.v[3] = lo0;
    c = o;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

/* raw block for known-answer tests */
void skro_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  u32x4 c;
  for (int i = 0; i < 4; ++i) c.v[i] = ctr[i];
  c = philox4x32_10(c, key[0], key[1]);
  for (int i = 0; i < 4; ++i) out[i] = c.v[i];
}

static void sincospi_host(double x, double* s, double* c) {
  /* x in [0, 2): exact reduction by quarter turns, then sin/cos of pi*r, |r| <= 1/4 */
  double q = nearbyint(2.0 * x);      /* multiples of 1/2 */
  double r = x - 0.5 * q;             /* exact: |r| <= 1/4 */
  long iq = (long)q & 3;
  double sr = sin(M_PI * r), cr = cos(M_PI * r);
  switch (iq) {
    case 0: *s = sr; *c = cr; break;
    case 1: *s = cr; *c = -sr; break;
    case 2: *s = -sr; *c = -cr; break;
    default: *s = -cr; *c = sr; break;
  }
}

/* philox_normal2 (rng.cuh): two standard normals for counter `ctr` of `stream` */
static void normal2(uint64_t seed, uint32_t stream, uint64_t ctr, double* z0, double* z1) {
  u32x4 c = {{(uint32_t)ctr, (uint32_t)(ctr >> 32), stream, 0x5EEDu}};
  c = philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t a = ((uint64_t)c.v[0] << 32) | c.v[1], b = ((uint64_t)c.v[2] << 32) | c.v[3];
  const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = (double)(b >> 11) * 0x1.0p-53;
  const double rr = sqrt(-2.0 * log(u1));
  double s, co;
  sincospi_host(2.0 * u2, &s, &co);
  *z0 = rr * co;
  *z1 = rr * s;
}

/* out[e] = scale * normal #(first + e) of `stream`, e < count */
void skro_philox_normals(uint64_t seed, uint32_t stream, int64_t first, int64_t count, double scale, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < count; ++e) {
    const uint64_t t = (uint64_t)(first + e);
    double z0, z1;
    normal2(seed, stream, t >> 1, &z0, &z1);
    out[e] = scale * ((t & 1) ? z1 : z0);
  }
}

/* synth_g_kernel: G[i, j] = sigma_j * normal #((row0 + i) * d + j) of stream 1 (rows x d) */
void skro_synth_g(uint64_t seed, int64_t row0, int64_t rows, int64_t d, const double* sigma, double* G) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i) {
    for (int64_t j = 0; j < d; ++j) {
      const uint64_t ge = (uint64_t)(row0 + i) * (uint64_t)d + (uint64_t)j;
      double z0, z1;
      normal2(seed, 1u, ge >> 1, &z0, &z1);
      G[i * d + j] = sigma[j] * ((ge & 1) ? z1 : z0);
    }
  }
}

/* synth_tscale_kernel: t_i = |Z0 / sqrt((Z1^2 + Z2^2 + Z3^2) / 3)| from stream 3 */
void skro_synth_tscale(uint64_t seed, int64_t row0, int64_t rows, double* t) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i) {
    double a0, a1, b0, b1;
    normal2(seed, 3u, 2 * (uint64_t)(row0 + i), &a0, &a1);
    normal2(seed, 3u, 2 * (uint64_t)(row0 + i) + 1, &b0, &b1);
    t[i] = fabs(a0 / sqrt((a1 * a1 + b0 * b0 + b1 * b1) / 3.0));
  }
}
