// K9 — the fused full-gradient + objective pass over the preconditioned rows.
//
// Replaces PreconditionedRidge::full_gradient / ::objective in Dense mode
// (ridge.cpp:174-236), which read X~ twice (dense_tmul_vec then dense_mul_vec)
// and call the objective as a third pass.  Here ONE streaming pass per call
// computes, for every local row i,
//     r_i = x~_i . w - y_i,   g += r_i * x~_i,   loss += r_i^2
// with each row held in registers between its dot and its axpy, so X~ is read
// exactly once (n*d*s bytes) — the HBM roofline of this kernel.
//
// Layout: a CTA owns ALL d columns (thread t holds columns [t*VEC, t*VEC+VEC),
// its w slice and its fp64 partial-gradient slice in registers) and streams
// tiles of TR consecutive rows; grid = a multiple of the SM count, tiles
// grid-strided.  Per tile: TR partial dots -> warp shuffles -> one smem
// exchange + __syncthreads -> residuals -> axpy into the register partials.
// Arithmetic is fp64 (fp32 rows are widened on load; precision
// is free at AI ~ 1 flop/B).  Per-CTA partials are summed in a fixed order
// (deterministic), allreduced across ranks, then scaled and combined with the
// regulariser lambda * P^{-1} w computed through the low-rank form
// P^{-1/2} v = c v + U (D - c) U^T v (precond.cpp:67-80), applied twice as the
// reference does (ridge.cpp:232-235).
#pragma once

#include "common.cuh"

namespace skr {

template <class T, int VEC>
struct RowVec;  // VEC elements of T loaded with 16-byte (or narrower) vector loads

template <class T, int VEC>
__device__ __forceinline__ void load_row(const T* __restrict__ p, double (&v)[VEC]) {
  constexpr int BYTES = VEC * (int)sizeof(T);
  if constexpr (BYTES >= 16) {
    const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
    for (int c = 0; c < BYTES / 16; ++c) {
      const float4 raw = __ldcs(q + c);  // streaming: X~ is read once per pass
      if constexpr (sizeof(T) == 4) {
        v[4 * c + 0] = raw.x; v[4 * c + 1] = raw.y; v[4 * c + 2] = raw.z; v[4 * c + 3] = raw.w;
      } else {
        const double2 d2 = *reinterpret_cast<const double2*>(&raw);
        v[2 * c + 0] = d2.x; v[2 * c + 1] = d2.y;
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < VEC; ++c) v[c] = (double)__ldcs(p + c);
  }
}

template <class T, int VEC, int TR, int NT>
__global__ void __launch_bounds__(NT)
fullgrad_kernel(const T* __restrict__ X, int64_t ld, int64_t n, const double* __restrict__ y,
                const double* __restrict__ w, double* __restrict__ part_g,
                double* __restrict__ part_loss) {
  constexpr int NW = NT / 32;
  __shared__ double red[2][TR][NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)tid * VEC;
  const bool active = c0 < ld;
  double wv[VEC], acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    wv[v] = active ? w[c0 + v] : 0.0;
    acc[v] = 0.0;
  }
  double loss = 0.0;
  const int64_t ntiles = (n + TR - 1) / TR;
  int par = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * TR;
    double xv[TR][VEC];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      if (active && r0 + t < n) {
        load_row<T, VEC>(X + (r0 + t) * ld + c0, xv[t]);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) xv[t][v] = 0.0;
      }
    }
    double p[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      double s = 0.0;
#pragma unroll
      for (int v = 0; v < VEC; ++v) s = fma(xv[t][v], wv[v], s);
      p[t] = s;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int t = 0; t < TR; ++t) p[t] += __shfl_xor_sync(0xffffffffu, p[t], off);
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < TR; ++t) red[par][t][warp] = p[t];
    }
    __syncthreads();
    double r[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) s += red[par][t][q];
      r[t] = (r0 + t < n) ? s - y[r0 + t] : 0.0;
    }
    if (tid == 0) {
#pragma unroll
      for (int t = 0; t < TR; ++t) loss = fma(r[t], r[t], loss);
    }
#pragma unroll
    for (int t = 0; t < TR; ++t)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = fma(r[t], xv[t][v], acc[v]);
    par ^= 1;
  }
  if (active) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) part_g[(int64_t)blockIdx.x * ld + c0 + v] = acc[v];
  }
  if (tid == 0) part_loss[blockIdx.x] = loss;
}

// Sum the per-CTA partials in CTA order: out[j] (j < ld) and out[ld] = loss.
__global__ void fullgrad_reduce_kernel(const double* __restrict__ part_g,
                                       const double* __restrict__ part_loss, int64_t ld, int parts,
                                       double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < ld) {
    double s = 0.0;
    for (int b = 0; b < parts; ++b) s += part_g[(int64_t)b * ld + j];
    out[j] = s;
  } else if (j == ld) {
    double s = 0.0;
    for (int b = 0; b < parts; ++b) s += part_loss[b];
    out[ld] = s;
  }
}

// proj[j] = U_j . v for j < k (one warp per basis vector; Ut is k x ld rows);
// the extra warp j == k computes v . v into proj[k].
__global__ void lowrank_proj_kernel(const double* __restrict__ Ut, int64_t ld, int64_t d,
                                    int64_t k, const double* __restrict__ v,
                                    double* __restrict__ proj) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp > k) return;
  const double* row = warp < k ? Ut + (int64_t)warp * ld : v;
  double s = 0.0;
  for (int64_t i = lane; i < d; i += 32) s = fma(row[i], v[i], s);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) proj[warp] = s;
}

// out_i = c v_i + sum_j U_ij (D_j - c) proj_j   (precond.cpp:67-80); zero pad to ld.
__global__ void lowrank_apply_kernel(const double* __restrict__ Ut, int64_t ld, int64_t d,
                                     int64_t k, const double* __restrict__ D, double c,
                                     const double* __restrict__ v, const double* __restrict__ proj,
                                     double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ld) return;
  if (i >= d) {
    out[i] = 0.0;
    return;
  }
  double s = 0.0;
  for (int64_t j = 0; j < k; ++j) s = fma(Ut[j * ld + i], (D[j] - c) * proj[j], s);
  out[i] = c * v[i] + s;
}

// mu_j = sums[j] / n + lambda * pinv_w[j];  obj = loss/(2n) + (lambda/2) ||P^{-1/2} w||^2
// with ||P^{-1/2} w||^2 = c^2 ||w||^2 + sum_j (D_j^2 - c^2) (U^T w)_j^2 (precond.cpp:110-118).
__global__ void fullgrad_finalize_kernel(const double* __restrict__ sums, int64_t ld, int64_t d,
                                         double n, double lambda,
                                         const double* __restrict__ pinv_w,
                                         const double* __restrict__ uw, int64_t k,
                                         const double* __restrict__ D, double c,
                                         double* __restrict__ mu, double* __restrict__ obj) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < ld) mu[j] = j < d ? sums[j] * (1.0 / n) + lambda * pinv_w[j] : 0.0;
  if (j == 0 && obj) {
    double reg = c * c * uw[k];  // uw[k] = w . w
    for (int64_t l = 0; l < k; ++l) reg += (D[l] * D[l] - c * c) * uw[l] * uw[l];
    *obj = sums[ld] / (2.0 * n) + 0.5 * lambda * reg;
  }
}

}  // namespace skr
