// Sparse data (the reference's SparseMatrix: CSC over points, sparse_matrix.hpp;
// kernels.cpp:106-155,216-273) — stored here as CSR over points (= the
// reference's CSC, byte-identical index arrays) plus a host-built CSR over
// features (the transpose), both fp64.  Products are warp-per-row SpMM against
// a dense row-major operand (lanes over its columns: coalesced), so every sum
// runs in a fixed order (deterministic).
#pragma once

#include "common.cuh"

namespace skr {

// out[r][j] = alpha * sum_{(f, v) in row r} v * B[f][j]   (j < ncols)
__global__ void __launch_bounds__(256) csr_spmm_kernel(const int64_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ idx,
                                                       const double* __restrict__ val, int64_t nrows,
                                                       const double* __restrict__ B, int64_t ldb, int64_t ncols,
                                                       double alpha, double* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nrows) return;
  const int64_t b = ptr[r], e = ptr[r + 1];
  for (int64_t j0 = 0; j0 < ncols; j0 += 32) {
    const int64_t j = j0 + lane;
    double acc = 0.0;
    if (j < ncols)
      for (int64_t t = b; t < e; ++t) acc = fma(val[t], B[(int64_t)idx[t] * ldb + j], acc);
    if (j < ncols) out[r * ldo + j] = alpha * acc;
  }
}

// out[r] = alpha * sum_{(f, v) in row r} v * x[f]  (one warp per row, lanes over the nonzeros)
__global__ void __launch_bounds__(256) csr_spmv_kernel(const int64_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ idx,
                                                       const double* __restrict__ val, int64_t nrows,
                                                       const double* __restrict__ x, double alpha,
                                                       double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nrows) return;
  double acc = 0.0;
  for (int64_t t = ptr[r] + lane; t < ptr[r + 1]; t += 32) acc = fma(val[t], x[idx[t]], acc);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) out[r] = alpha * acc;
}

// sq[r] = ||row r||^2
__global__ void __launch_bounds__(256) csr_row_sqnorm_kernel(const int64_t* __restrict__ ptr,
                                                             const double* __restrict__ val, int64_t nrows,
                                                             double* __restrict__ sq) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nrows) return;
  double acc = 0.0;
  for (int64_t t = ptr[r] + lane; t < ptr[r + 1]; t += 32) acc = fma(val[t], val[t], acc);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) sq[r] = acc;
}

// out (cols x ldo) = in^T for in (rows x cols, row stride ldi); out columns >= rows untouched
__global__ void transpose_f64_kernel(const double* __restrict__ in, int64_t rows, int64_t cols, int64_t ldi,
                                     double* __restrict__ out, int64_t ldo) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < rows && j < cols) ? in[i * ldi + j] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (j < cols && i < rows) out[j * ldo + i] = tile[threadIdx.x][r];
  }
}

inline void transpose_f64(Ctx& c, const double* in, int64_t rows, int64_t cols, int64_t ldi, double* out,
                          int64_t ldo) {
  if (rows <= 0 || cols <= 0) return;
  transpose_f64_kernel<<<dim3(ceil_div(rows, 32), ceil_div(cols, 32)), dim3(32, 8), 0, c.stream>>>(in, rows, cols, ldi,
                                                                                                   out, ldo);
  SKR_LAUNCHED(&c);
}

// out (rows x ldo, zeroed here) = the dense rows of a CSR block
__global__ void __launch_bounds__(256) csr_densify_kernel(const int64_t* __restrict__ ptr,
                                                          const int32_t* __restrict__ idx,
                                                          const double* __restrict__ val, int64_t nrows,
                                                          double* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= nrows) return;
  for (int64_t t = ptr[r] + lane; t < ptr[r + 1]; t += 32) out[r * ldo + idx[t]] = val[t];
}

inline void csr_densify(Ctx& c, const int64_t* ptr, const int32_t* idx, const double* val, int64_t nrows,
                        double* out, int64_t ldo) {
  if (nrows <= 0) return;
  SKR_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * nrows * ldo, c.stream));
  csr_densify_kernel<<<ceil_div(nrows * 32, 256), 256, 0, c.stream>>>(ptr, idx, val, nrows, out, ldo);
  SKR_LAUNCHED(&c);
}

inline void csr_spmm(Ctx& c, const int64_t* ptr, const int32_t* idx, const double* val, int64_t nrows,
                     const double* B, int64_t ldb, int64_t ncols, double alpha, double* out, int64_t ldo) {
  if (nrows <= 0 || ncols <= 0) return;
  csr_spmm_kernel<<<ceil_div(nrows * 32, 256), 256, 0, c.stream>>>(ptr, idx, val, nrows, B, ldb, ncols, alpha, out,
                                                                   ldo);
  SKR_LAUNCHED(&c);
}

inline void csr_spmv(Ctx& c, const int64_t* ptr, const int32_t* idx, const double* val, int64_t nrows,
                     const double* x, double alpha, double* out) {
  if (nrows <= 0) return;
  csr_spmv_kernel<<<ceil_div(nrows * 32, 256), 256, 0, c.stream>>>(ptr, idx, val, nrows, x, alpha, out);
  SKR_LAUNCHED(&c);
}

}  // namespace skr
