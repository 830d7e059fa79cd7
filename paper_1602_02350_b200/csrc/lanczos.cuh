// Device pieces of block_lanczos (sketch.cpp:18-90) besides the products:
// Krylov-block orthogonalisation with the reference's rank-drop rule, and the
// eigenvector post-processing (descending order, sign rules).
#pragma once

#include "common.cuh"

namespace skr {

constexpr double kRankDropTol = 1e-12;  // factorize.hpp:12

__device__ __forceinline__ double block_sum(double v, double* scratch) {
  // scratch: >= 32 doubles of shared memory; returns the sum to every thread.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int q = 0; q < nw; ++q) s += scratch[q];
  return s;
}

__device__ __forceinline__ double block_max(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double s = scratch[0];
  for (int q = 1; q < nw; ++q) s = fmax(s, scratch[q]);
  return s;
}

// Helpers for MgsBasis::append_block (factorize.cpp:53-71) on the device.
// The block (a rows of length d) is first projected off the accepted basis
// twice with GEMMs (block classical Gram-Schmidt, BCGS2), then factored by a
// Householder QR (cuSOLVER geqrf/orgqr).  |R_jj| is the norm of column j after
// removing every earlier direction — the quantity the reference's two MGS
// passes compare against 1e-12 x the block's largest original column norm —
// so the same rank-drop rule applies; survivors are appended with sign(R_jj)
// so each new basis vector matches the MGS one, not just its span.

// out[0] = max_j ||V_j|| over `rows` rows of length d (row stride ld); one CTA.
// *out = max_j ||V[j, :d]|| (one block per row; *out zeroed by the caller; norms
// are non-negative so their bit patterns order like the values)
__global__ void row_norm_max_kernel(const double* __restrict__ V, int64_t ld, int64_t d, int rows,
                                    double* __restrict__ out) {
  __shared__ double scratch[32];
  const int j = blockIdx.x;
  if (j >= rows) return;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) s = fma(V[j * ld + i], V[j * ld + i], s);
  const double nrm = sqrt(block_sum(s, scratch));
  if (threadIdx.x == 0) atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(nrm));
}

// rdiag[j] = R_jj from geqrf output (column-major, lda = ld): element (j,j) at j*ld + j.
__global__ void qr_diag_kernel(const double* __restrict__ A, int64_t ld, int rows, double* __restrict__ rdiag) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < rows) rdiag[j] = A[(int64_t)j * ld + j];
}

// Append rows j of Q (orgqr output, row j = basis candidate j) whose |R_jj|
// passes the drop rule; count[0] = basis size (in/out), count[1] = appended.
__global__ void qr_select_kernel(double* __restrict__ Qt, int64_t ld, int64_t d, int* __restrict__ count, int cap,
                                 const double* __restrict__ Q, const double* __restrict__ rdiag,
                                 const double* __restrict__ ref, int rows) {
  const double r = *ref;
  int W = count[0], added = 0;
  if (r > 0.0) {
    const double drop = kRankDropTol * r;
    for (int j = 0; j < rows; ++j) {
      const double rj = rdiag[j];
      if (!(fabs(rj) >= drop) || W >= cap) continue;
      const double sgn = rj < 0.0 ? -1.0 : 1.0;
      for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) Qt[(int64_t)W * ld + i] = i < d ? sgn * Q[(int64_t)j * ld + i] : 0.0;
      ++W;
      ++added;
    }
  }
  if (threadIdx.x == 0) {
    count[0] = W;
    count[1] = added;
  }
}

// CholeskyQR acceptance threshold: R_jj >= kCholQrMinRatio * max original norm
constexpr double kCholQrMinRatio = 1e-6;

// out[j] = L_jj of a column-major a x a factor
__global__ void chol_diag_kernel(const double* __restrict__ L, int a, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < a) out[j] = L[(int64_t)j * a + j];
}
// zero the strictly upper triangle of a column-major a x a matrix (element (i,j) at j*a + i, i < j)
__global__ void zero_upper_cm_kernel(double* __restrict__ A, int a) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)a * a) return;
  const int64_t j = e / a, i = e % a;
  if (i < j) A[e] = 0.0;
}
// Accept the CholeskyQR2 block when both factorizations succeeded and every
// R_jj = L1_jj L2_jj clears min_ratio * ref: then append all rows (up to cap).
// count = {W (in/out), appended (out), rejected (out)}.
__global__ void cholqr_select_kernel(double* __restrict__ Qt, int64_t ld, int64_t d, int* __restrict__ count, int cap,
                                     const double* __restrict__ Q, const double* __restrict__ diag, int a,
                                     const double* __restrict__ ref, const int* __restrict__ info, double min_ratio) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = (info[0] != 0 || info[1] != 0 || info[2] != 0 || !(*ref > 0.0)) ? 1 : 0;
  __syncthreads();
  for (int j = threadIdx.x; j < a; j += blockDim.x) {
    const double r = diag[j] * diag[a + j];
    if (!(r >= min_ratio * *ref)) bad = 1;
  }
  __syncthreads();
  const int W = count[0];
  const int take = bad ? 0 : min(a, cap - W);
  for (int64_t e = threadIdx.x; e < (int64_t)take * ld; e += blockDim.x) {
    const int64_t j = e / ld, i = e % ld;
    Qt[(int64_t)(W + j) * ld + i] = i < d ? Q[j * ld + i] : 0.0;
  }
  if (threadIdx.x == 0) {
    count[0] = W + take;
    count[1] = take;
    count[2] = bad;
  }
}

// V[j] *= sign(R_jj)  (Haar fix-up of an orthogonal factor: Q diag(sign diag R))
__global__ void qr_sign_rows_kernel(double* __restrict__ Q, int64_t ld, int64_t d, const double* __restrict__ rdiag,
                                    int rows) {
  const int j = blockIdx.x;
  if (j >= rows || rdiag[j] >= 0.0) return;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) Q[(int64_t)j * ld + i] = -Q[(int64_t)j * ld + i];
}

// syevd returns ascending eigenpairs (column-major evec, W x W).  Produce the
// reference's sym_eigs convention (factorize.cpp:148-164): descending values,
// each eigenvector's largest-|entry| (lowest index on ties) made positive.
// Writes Wt (kk x W, row j = eigenvector j) and vals_desc[j], j < W.
__global__ void eig_post_kernel(const double* __restrict__ evec, const double* __restrict__ eval,
                                int W, int kk, double* __restrict__ Wt,
                                double* __restrict__ vals_desc) {
  __shared__ double smax[32];
  __shared__ int sarg[32];
  const int j = blockIdx.x;  // output column (descending rank)
  const int src = W - 1 - j;
  const double* col = evec + (int64_t)src * W;
  // argmax |col| with lowest index on ties
  double best = -1.0;
  int arg = 0x7fffffff;
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    const double a = fabs(col[i]);
    if (a > best || (a == best && i < arg)) { best = a; arg = i; }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int oa = __shfl_xor_sync(0xffffffffu, arg, off);
    if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { smax[warp] = best; sarg[warp] = arg; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (smax[q] > smax[0] || (smax[q] == smax[0] && sarg[q] < sarg[0])) { smax[0] = smax[q]; sarg[0] = sarg[q]; }
  }
  __syncthreads();
  const double sign = col[sarg[0]] < 0.0 ? -1.0 : 1.0;
  if (j < kk)
    for (int i = threadIdx.x; i < W; i += blockDim.x) Wt[(int64_t)j * W + i] = sign * col[i];
  if (threadIdx.x == 0) vals_desc[j] = eval[src];
}

// normalize_svd_signs (factorize.cpp:167-178): flip row j of Ut (and column j
// of V) when Ut's largest-|entry| (lowest index on ties) is negative.
// One CTA per j; writes flip[j] = +-1.
__global__ void svd_sign_kernel(double* __restrict__ Ut, int64_t ld, int64_t d,
                                double* __restrict__ flip) {
  __shared__ double smax[32];
  __shared__ int64_t sarg[32];
  const int j = blockIdx.x;
  double* row = Ut + (int64_t)j * ld;
  double best = -1.0;
  int64_t arg = INT64_MAX;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
    const double a = fabs(row[i]);
    if (a > best || (a == best && i < arg)) { best = a; arg = i; }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, off);
    const int64_t oa = __shfl_xor_sync(0xffffffffu, arg, off);
    if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { smax[warp] = best; sarg[warp] = arg; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (smax[q] > smax[0] || (smax[q] == smax[0] && sarg[q] < sarg[0])) { smax[0] = smax[q]; sarg[0] = sarg[q]; }
  }
  __syncthreads();
  const double sign = row[sarg[0]] < 0.0 ? -1.0 : 1.0;
  __syncthreads();
  if (sign < 0.0)
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) row[i] = -row[i];
  if (threadIdx.x == 0) flip[j] = sign;
}

// Column norms of a rows x k row-major block (k <= 1024): out[j] += sum_i V[i,j]^2.
// per-block partial column sums of squares (part[b][j]); summed in block order by
// col_sq_reduce_kernel, so the result is run-to-run deterministic
__global__ void col_sq_norms_kernel(const double* __restrict__ V, int64_t rows, int k,
                                    double* __restrict__ part) {
  const int j = threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) s = fma(V[i * k + j], V[i * k + j], s);
  part[(int64_t)blockIdx.x * k + j] = s;
}
__global__ void col_sq_reduce_kernel(const double* __restrict__ part, int blocks, int k, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  double s = 0.0;
  for (int b = 0; b < blocks; ++b) s += part[(int64_t)b * k + j];
  out[j] = s;
}

// V[i,j] *= flip[j] / sqrt(sq[j])  (zero norm -> left unscaled, sketch.cpp:82-83)
__global__ void col_normalize_kernel(double* __restrict__ V, int64_t rows, int k,
                                     const double* __restrict__ sq, const double* __restrict__ flip) {
  const int64_t total = rows * k;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % k);
    const double nrm = sqrt(sq[j]);
    const double s = nrm > 0.0 ? 1.0 / nrm : 1.0;
    V[e] = V[e] * s * flip[j];
  }
}

}  // namespace skr
