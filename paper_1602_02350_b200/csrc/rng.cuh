// Random streams.
//
// (1) mt19937_64 on the device, bit-exact with std::mt19937_64 as used by the
//     reference's NormalSampler (random.hpp:13-24, random.cpp:10-41): the
//     Gaussian test matrix Pi of block_lanczos (sketch.cpp:52) and the SVRG
//     index stream (svrg.cpp:174,192) must be the reference's own streams
//     (SURVEY §0 fact 10).  The engine is inherently sequential, so one CTA
//     owns the 312-word state in shared memory and regenerates it with a
//     three-phase parallel twist; tempering and the uniform conversion are
//     per-lane.  Box-Muller then runs over all pairs in parallel.
// (2) Philox4x32-10, counter-based, for the synthetic BASELINE data at scale
//     (not a reference stream; DESIGN.md documents the draw order).
#pragma once

#include "common.cuh"

namespace skr {

constexpr int MT_N = 312, MT_M = 156;
constexpr uint64_t MT_UPPER = 0xFFFFFFFF80000000ULL, MT_LOWER = 0x7FFFFFFFULL;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ULL;

struct MtState {
  uint64_t mt[MT_N];
  int32_t mti;  // next output position; MT_N means "twist before the next draw"
  int32_t pad;
};

// std::mt19937_64(seed) seeding (C++ [rand.eng.mers]); done on the host, 312 steps.
inline void mt_seed_host(MtState& s, uint64_t seed) {
  s.mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) s.mt[i] = 6364136223846793005ULL * (s.mt[i - 1] ^ (s.mt[i - 1] >> 62)) + (uint64_t)i;
  s.mti = MT_N;
  s.pad = 0;
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b) {
  const uint64_t x = (a & MT_UPPER) | (b & MT_LOWER);
  return (x >> 1) ^ ((x & 1ULL) ? MT_A : 0ULL);
}

// Parallel regeneration of the state (equivalent to the sequential twist):
//   i in [0,156):   mt[i] = mt[i+156]_old ^ mix(mt[i]_old, mt[i+1]_old)
//   i in [156,311): mt[i] = mt[i-156]_new ^ mix(mt[i]_old, mt[i+1]_old)
//   i = 311:        mt[311] = mt[155]_new ^ mix(mt[311]_old, mt[0]_new)
__device__ __forceinline__ void mt_twist_block(uint64_t* mt) {
  const int t = threadIdx.x;
  uint64_t v = 0;
  if (t < MT_M) v = mt[t + MT_M] ^ mt_mix(mt[t], mt[t + 1]);
  __syncthreads();
  if (t < MT_M) mt[t] = v;
  __syncthreads();
  if (t >= MT_M && t < MT_N - 1) v = mt[t - MT_M] ^ mt_mix(mt[t], mt[t + 1]);
  __syncthreads();
  if (t >= MT_M && t < MT_N - 1) mt[t] = v;
  __syncthreads();
  if (t == 0) mt[MT_N - 1] = mt[MT_M - 1] ^ mt_mix(mt[MT_N - 1], mt[0]);
  __syncthreads();
}

// Draw `count` outputs continuing the stream in *st; writes NormalSampler
// uniforms ((y >> 11) * 2^-53) or raw 64-bit words.  Launch <<<1, 320>>>.
template <bool RAW>
__global__ void __launch_bounds__(320) mt_generate_kernel(MtState* st, void* out, int64_t count) {
  __shared__ uint64_t mt[MT_N];
  __shared__ int pos_s;
  for (int i = threadIdx.x; i < MT_N; i += blockDim.x) mt[i] = st->mt[i];
  if (threadIdx.x == 0) pos_s = st->mti;
  __syncthreads();
  int pos = pos_s;
  int64_t produced = 0;
  while (produced < count) {
    if (pos >= MT_N) {
      mt_twist_block(mt);
      pos = 0;
    }
    const int64_t rem = count - produced;
    const int64_t avail = rem < (int64_t)(MT_N - pos) ? rem : (int64_t)(MT_N - pos);
    if (threadIdx.x < avail) {
      const uint64_t y = mt_temper(mt[pos + threadIdx.x]);
      if (RAW) static_cast<uint64_t*>(out)[produced + threadIdx.x] = y;
      else static_cast<double*>(out)[produced + threadIdx.x] = (double)(y >> 11) * 0x1.0p-53;
    }
    produced += avail;
    pos += (int)avail;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < MT_N; i += blockDim.x) st->mt[i] = mt[i];
  if (threadIdx.x == 0) st->mti = pos;
}

// NormalSampler::normal over a fresh stream (random.cpp:14-26): normal #t uses
// uniform pair p = t/2: u1 = 1 - U[2p], u2 = U[2p+1], r = sqrt(-2 log u1),
// angle = 2 pi u2; even t -> r cos, odd t -> r sin.  Writes the column-major
// rows x cols matrix restricted to rows [row0, row0+rows_local) as a
// cols x rows_local row-major array (Pi^T, one test vector per row).
__global__ void box_muller_kernel(const double* __restrict__ u, int64_t rows, int64_t cols,
                                  int64_t row0, int64_t rows_local, double* __restrict__ out_t) {
  const int64_t total = rows_local * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows_local, il = e % rows_local;
    const int64_t t = j * rows + row0 + il;  // global normal number
    const int64_t p = t >> 1;
    const double u1 = 1.0 - u[2 * p];
    const double u2 = u[2 * p + 1];
    const double r = sqrt(-2.0 * log(u1));
    const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
    double s, c;
    sincos(angle, &s, &c);
    out_t[j * rows_local + il] = (t & 1) ? r * s : r * c;
  }
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. 2011) for synthetic data.
struct Philox {
  __device__ static uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  __device__ static uint4 gen(uint4 c, uint2 k) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

// Two standard normals for counter `ctr` of stream `stream` under `seed`.
__device__ __forceinline__ double2 philox_normal2(uint64_t seed, uint32_t stream, uint64_t ctr) {
  const uint4 r = Philox::gen(make_uint4((uint32_t)ctr, (uint32_t)(ctr >> 32), stream, 0x5EED),
                              make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const uint64_t a = ((uint64_t)r.x << 32) | r.y, b = ((uint64_t)r.z << 32) | r.w;
  const double u1 = ((double)(a >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
  const double u2 = (double)(b >> 11) * 0x1.0p-53;
  const double rr = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  return make_double2(rr * c, rr * s);
}

// out[e] = scale * N(0,1) draw e of `stream` (e < count).
__global__ void philox_normal_kernel(uint64_t seed, uint32_t stream, int64_t count, double scale,
                                     double* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; 2 * p < count;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double2 z = philox_normal2(seed, stream, (uint64_t)p);
    out[2 * p] = scale * z.x;
    if (2 * p + 1 < count) out[2 * p + 1] = scale * z.y;
  }
}

}  // namespace skr
