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

namespace skr {

// ---- Lazy preconditioned problem over sparse rows (ridge.cpp:93-150,174-236 with
// mode Lazy): X~ = c X + (P o (D - c)) U^T is never formed; P = X U^T (n x k). ----

// beta_i = coef (c^2 ||x_i||^2 + sum_l (D_l^2 - c^2) P_il^2)   (ridge.cpp:124-127); rowmax = max ||x~_i||^2
__global__ void __launch_bounds__(256) lazy_betas_kernel(const int64_t* __restrict__ ptr,
                                                         const double* __restrict__ val, int64_t n,
                                                         const double* __restrict__ P, int64_t k,
                                                         const double* __restrict__ D, double c, double coef,
                                                         double* __restrict__ beta, double* __restrict__ rowmax) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t t = ptr[i] + lane; t < ptr[i + 1]; t += 32) s = fma(val[t], val[t], s);
  double q = 0.0;
  for (int64_t l = lane; l < k; l += 32) {
    const double pl = P[i * k + l];
    q = fma((D[l] * D[l] - c * c) * pl, pl, q);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, off);
    q += __shfl_xor_sync(0xffffffffu, q, off);
  }
  const double nrm = c * c * s + q;
  if (lane == 0) {
    beta[i] = coef * nrm;
    atomicMax(reinterpret_cast<unsigned long long*>(rowmax), (unsigned long long)__double_as_longlong(fmax(nrm, 0.0)));
  }
}

// s_i = x~_i . w = c x_i . w + P_i . v  (v = (D - c) o U^T w);  r2_i = (s_i - y_i)^2, r_i = s_i - y_i
__global__ void __launch_bounds__(256) lazy_residual_kernel(const int64_t* __restrict__ ptr,
                                                            const int32_t* __restrict__ idx,
                                                            const double* __restrict__ val, int64_t n,
                                                            const double* __restrict__ w,
                                                            const double* __restrict__ P, int64_t k,
                                                            const double* __restrict__ v, double c,
                                                            const double* __restrict__ y, double* __restrict__ s_out,
                                                            double* __restrict__ r_out, double* __restrict__ r2_out) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  double a = 0.0, b = 0.0;
  for (int64_t t = ptr[i] + lane; t < ptr[i + 1]; t += 32) a = fma(val[t], w[idx[t]], a);
  for (int64_t l = lane; l < k; l += 32) b = fma(P[i * k + l], v[l], b);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, off);
    b += __shfl_xor_sync(0xffffffffu, b, off);
  }
  if (lane == 0) {
    const double s = c * a + b;
    const double r = s - y[i];
    if (s_out) s_out[i] = s;
    r_out[i] = r;
    r2_out[i] = r * r;
  }
}

// v_l = (D_l - c) u_l
__global__ void lazy_scale_kernel(const double* __restrict__ u, const double* __restrict__ D, double c, int64_t k,
                                  double* __restrict__ v) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l < k) v[l] = (D[l] - c) * u[l];
}

// mu_f = (c g1_f + sum_l U_lf (D_l - c) g2_l) / n + lambda (c^2 w_f + sum_l U_lf (D_l^2 - c^2) u_l);
// thread 0 of block 0 also finishes the objective from the loss sum.
__global__ void lazy_finalize_kernel(const double* __restrict__ g1, const double* __restrict__ g2,
                                     const double* __restrict__ Ut, int64_t ld, int64_t d, int64_t k,
                                     const double* __restrict__ D, double c, const double* __restrict__ w,
                                     const double* __restrict__ uw, double inv_n, double lambda,
                                     const double* __restrict__ loss, double* __restrict__ mu,
                                     double* __restrict__ obj) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f < ld) {
    if (f < d) {
      double a = c * g1[f], r = c * c * w[f];
      for (int64_t l = 0; l < k; ++l) {
        const double uf = Ut[l * ld + f];
        a = fma(uf, (D[l] - c) * g2[l], a);
        r = fma(uf, (D[l] * D[l] - c * c) * uw[l], r);
      }
      mu[f] = a * inv_n + lambda * r;
    } else {
      mu[f] = 0.0;
    }
  }
  if (obj && f == 0) {
    double reg = c * c * uw[k];
    for (int64_t l = 0; l < k; ++l) reg += (D[l] * D[l] - c * c) * uw[l] * uw[l];
    *obj = *loss * (0.5 * inv_n) + 0.5 * lambda * reg;
  }
}

// row i of X~ as a dense ld-vector: c x_i + U ((D - c) o P_i)   (zero padded)
__global__ void lazy_row_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                const double* __restrict__ val, int64_t i, const double* __restrict__ P, int64_t k,
                                const double* __restrict__ Ut, int64_t ld, int64_t d, const double* __restrict__ D,
                                double c, double* __restrict__ out) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= ld) return;
  double s = 0.0;
  if (f < d)
    for (int64_t l = 0; l < k; ++l) s = fma(Ut[l * ld + f], (D[l] - c) * P[i * k + l], s);
  out[f] = s;
}
__global__ void lazy_row_scatter_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                        const double* __restrict__ val, int64_t i, double c,
                                        double* __restrict__ out) {
  for (int64_t t = ptr[i] + threadIdx.x; t < ptr[i + 1]; t += blockDim.x) out[idx[t]] += c * val[t];
}

}  // namespace skr

namespace skr {

// ---- Lazy SVRG epoch over sparse rows (LazyEpochState, ridge.cpp:283-400) ------------
// w_t = base_t + U h_t - tau_t mu with tau_t = eta t, z = U^T w tracked like the
// reference (z -= eta (delta D o P_i + U^T mu)), so a data step costs O(nnz_i + k)
// and a regulariser step O(k) — the reference's per-step O(d) axpy of mu into base
// is folded into tau.  The epoch average uses
//   sum_{t=1..m} w_t = m base_0 + sum_s (m-s+1) dbase_s + U sum_s (m-s+1) dh_s - eta m(m+1)/2 mu.
// One CTA runs the sequential chain; all sums are in a fixed order.
struct LazyEpochArgs {
  const int64_t* rptr;
  const int32_t* ridx;
  const double* rval;
  int64_t n, d, ld, k;
  const double* P;      // n x k
  const double* UT;     // d x k (row f = U_f)
  const double* D;      // k
  double c, data_coef, reg_coef;
  const int64_t* idx;   // m
  const double* inv_nq; // N
  int64_t m;
  double eta;
  const double* s_bar;  // n: x~_i . wbar
  const double* half;   // d: (P^{-1/2} wbar)_j
  const double* xmu;    // n: x_i . mu
  const double* mu;     // ld
  const double* bg;     // k: U^T mu
  const double* z0;     // k: U^T wbar
  const double* snap;   // ld: wbar
  double* base;         // ld scratch (starts as wbar)
  double* Sb;           // ld scratch (zero)
  double* w_avg;        // ld out
};

constexpr int kLazyThreads = 256;

__device__ __forceinline__ double lazy_block_sum(double v, double* red, int tid) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((tid & 31) == 0) red[tid >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < kLazyThreads / 32; ++q) s += red[q];
  return s;
}

template <bool SMEM_BASE>
__global__ void __launch_bounds__(kLazyThreads, 1) lazy_epoch_kernel(LazyEpochArgs a) {
  extern __shared__ double lz_sm[];
  const int64_t k = a.k;
  double* h = lz_sm;          // k
  double* z = h + k;          // k
  double* Sh = z + k;         // k
  double* Dm = Sh + k;        // k: D - c
  double* Dd = Dm + k;        // k: D
  double* red = Dd + k;       // 3 x 8
  double* base = SMEM_BASE ? red + 24 : a.base;  // the gathered state, in shared memory when d fits
  const int tid = threadIdx.x;
  if (SMEM_BASE)
    for (int64_t f = tid; f < a.ld; f += kLazyThreads) base[f] = a.base[f];
  for (int64_t l = tid; l < k; l += kLazyThreads) {
    h[l] = 0.0;
    z[l] = a.z0[l];
    Sh[l] = 0.0;
    Dm[l] = a.D[l] - a.c;
    Dd[l] = a.D[l];
  }
  __syncthreads();
  for (int64_t t = 1; t <= a.m; ++t) {
    const int64_t i = a.idx[t - 1];
    const double q = a.inv_nq[i];
    const double tau = a.eta * (double)(t - 1);
    const double wgt = (double)(a.m - t + 1);
    const bool data = i < a.n;
    const double* row = data ? a.P + i * k : a.UT + (i - a.n) * k;
    double A = 0.0, B = 0.0, Cz = 0.0;
    int64_t b0 = 0, b1 = 0;
    if (data) {
      b0 = a.rptr[i];
      b1 = a.rptr[i + 1];
      for (int64_t e = b0 + tid; e < b1; e += kLazyThreads) A = fma(a.rval[e], base[a.ridx[e]], A);
    } else if (tid == 0) {
      A = base[i - a.n];
    }
    for (int64_t l = tid; l < k; l += kLazyThreads) {
      const double r = row[l];
      B = fma(r, h[l], B);
      Cz = fma(Dm[l] * r, z[l], Cz);
    }
    A = lazy_block_sum(A, red, tid);
    B = lazy_block_sum(B, red + 8, tid);
    Cz = lazy_block_sum(Cz, red + 16, tid);
    double delta;
    if (data) {
      const double inner = a.c * (A + B - tau * a.xmu[i]) + Cz;
      delta = a.data_coef * (inner - a.s_bar[i]) * q;
    } else {
      const int64_t j = i - a.n;
      const double inner = a.c * (A + B - tau * a.mu[j]) + Cz;
      delta = a.reg_coef * (inner - a.half[j]) * q;
    }
    __syncthreads();  // every thread has read red/h/z/base before the updates
    const double ed = a.eta * delta;
    if (data) {
      for (int64_t e = b0 + tid; e < b1; e += kLazyThreads) {
        const int64_t f = a.ridx[e];
        const double dv = -ed * a.c * a.rval[e];
        base[f] += dv;
        a.Sb[f] = fma(wgt, dv, a.Sb[f]);
      }
    } else if (tid == 0) {
      const int64_t j = i - a.n;
      const double dv = -ed * a.c;
      base[j] += dv;
      a.Sb[j] = fma(wgt, dv, a.Sb[j]);
    }
    for (int64_t l = tid; l < k; l += kLazyThreads) {
      const double r = row[l];
      const double dh = -ed * Dm[l] * r;
      h[l] += dh;
      Sh[l] = fma(wgt, dh, Sh[l]);
      z[l] -= a.eta * fma(delta, Dd[l] * r, a.bg[l]);
    }
    __syncthreads();
  }
  // w_avg = (m wbar + Sb) / m + U Sh / m - eta (m + 1) / 2 mu
  const double inv_m = 1.0 / (double)a.m, half_tau = 0.5 * a.eta * (double)(a.m + 1);
  for (int64_t f = tid; f < a.ld; f += kLazyThreads) {
    if (f < a.d) {
      double lift = 0.0;
      for (int64_t l = 0; l < k; ++l) lift = fma(a.UT[f * k + l], Sh[l], lift);
      a.w_avg[f] = a.snap[f] + a.Sb[f] * inv_m + lift * inv_m - half_tau * a.mu[f];
    } else {
      a.w_avg[f] = 0.0;
    }
  }
}

inline size_t lazy_epoch_smem(int64_t k, int64_t ld_base) {
  return sizeof(double) * (5 * std::max<int64_t>(k, 1) + 24 + ld_base);
}

}  // namespace skr

namespace skr {

// ---- load balance for skewed rows (power-law feature popularity): rows longer
// than kSplitNnz are cut into consecutive sub-rows; a warp per sub-row writes a
// partial, and a second pass sums each row's partials in sub-row order, so the
// result stays deterministic. ----
constexpr int64_t kSplitNnz = 2048;

struct SplitCSR {
  DBuf<int64_t> ptr;    // S + 1: entry offsets of the sub-rows
  DBuf<int64_t> first;  // rows + 1: first sub-row of each row
  DBuf<int32_t> row;    // S: row of each sub-row
  int64_t S = 0;
};

// host: the split of a CSR with row pointer rp (rows + 1)
inline void build_split(Ctx& c, const int64_t* rp, int64_t rows, SplitCSR& out) {
  std::vector<int64_t> sp{0}, first{0};
  std::vector<int32_t> srow;
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t b = rp[r], e = rp[r + 1];
    int64_t t = b;
    do {
      const int64_t u = std::min(e, t + kSplitNnz);
      sp.push_back(u);
      srow.push_back((int32_t)r);
      t = u;
    } while (t < e);
    first.push_back((int64_t)srow.size());
  }
  out.S = (int64_t)srow.size();
  out.ptr.alloc(out.S + 1, c.stream);
  out.first.alloc(rows + 1, c.stream);
  out.row.alloc(std::max<int64_t>(out.S, 1), c.stream);
  SKR_CUDA(cudaMemcpyAsync(out.ptr.get(), sp.data(), sizeof(int64_t) * sp.size(), cudaMemcpyHostToDevice, c.stream));
  SKR_CUDA(cudaMemcpyAsync(out.first.get(), first.data(), sizeof(int64_t) * first.size(), cudaMemcpyHostToDevice,
                           c.stream));
  if (out.S)
    SKR_CUDA(cudaMemcpyAsync(out.row.get(), srow.data(), sizeof(int32_t) * srow.size(), cudaMemcpyHostToDevice,
                             c.stream));
  c.sync();  // the host vectors go out of scope
}

// part[u] = sum over sub-row u of val * x[idx]   (warp per sub-row)
__global__ void __launch_bounds__(256) split_spmv_kernel(const int64_t* __restrict__ sptr,
                                                         const int32_t* __restrict__ idx,
                                                         const double* __restrict__ val, int64_t S,
                                                         const double* __restrict__ x, double* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (u >= S) return;
  double acc = 0.0;
  for (int64_t t = sptr[u] + lane; t < sptr[u + 1]; t += 32) acc = fma(val[t], x[idx[t]], acc);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) part[u] = acc;
}

// out[r] = alpha * sum_{u in row r's sub-rows} part[u] (ncols-wide rows, part row stride ncols)
__global__ void split_reduce_kernel(const int64_t* __restrict__ first, int64_t rows, const double* __restrict__ part,
                                    int64_t ncols, double alpha, double* __restrict__ out, int64_t ldo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * ncols) return;
  const int64_t r = e / ncols, j = e % ncols;
  double s = 0.0;
  for (int64_t u = first[r]; u < first[r + 1]; ++u) s += part[u * ncols + j];
  out[r * ldo + j] = alpha * s;
}

// part[u][j] = sum over sub-row u of val * B[idx][j]   (warp per sub-row, lanes over j)
__global__ void __launch_bounds__(256) split_spmm_kernel(const int64_t* __restrict__ sptr,
                                                         const int32_t* __restrict__ idx,
                                                         const double* __restrict__ val, int64_t S,
                                                         const double* __restrict__ B, int64_t ldb, int64_t ncols,
                                                         double* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (u >= S) return;
  const int64_t b = sptr[u], e = sptr[u + 1];
  for (int64_t j0 = 0; j0 < ncols; j0 += 32) {
    const int64_t j = j0 + lane;
    double acc = 0.0;
    if (j < ncols)
      for (int64_t t = b; t < e; ++t) acc = fma(val[t], B[(int64_t)idx[t] * ldb + j], acc);
    if (j < ncols) part[u * ncols + j] = acc;
  }
}

// balanced SpMV / SpMM over a split CSR (rows = number of CSR rows)
inline void split_spmv(Ctx& c, const SplitCSR& sp, const int32_t* idx, const double* val, int64_t rows,
                       const double* x, double alpha, double* out) {
  if (rows <= 0) return;
  DBuf<double> part(std::max<int64_t>(sp.S, 1), c.stream);
  split_spmv_kernel<<<ceil_div(sp.S * 32, 256), 256, 0, c.stream>>>(sp.ptr.get(), idx, val, sp.S, x, part.get());
  SKR_LAUNCHED(&c);
  split_reduce_kernel<<<ceil_div(rows, 256), 256, 0, c.stream>>>(sp.first.get(), rows, part.get(), 1, alpha, out, 1);
  SKR_LAUNCHED(&c);
}

inline void split_spmm(Ctx& c, const SplitCSR& sp, const int32_t* idx, const double* val, int64_t rows,
                       const double* B, int64_t ldb, int64_t ncols, double alpha, double* out, int64_t ldo) {
  if (rows <= 0 || ncols <= 0) return;
  DBuf<double> part((size_t)std::max<int64_t>(sp.S, 1) * ncols, c.stream);
  split_spmm_kernel<<<ceil_div(sp.S * 32, 256), 256, 0, c.stream>>>(sp.ptr.get(), idx, val, sp.S, B, ldb, ncols,
                                                                    part.get());
  SKR_LAUNCHED(&c);
  split_reduce_kernel<<<ceil_div(rows * ncols, 256), 256, 0, c.stream>>>(sp.first.get(), rows, part.get(), ncols, alpha,
                                                                         out, ldo);
  SKR_LAUNCHED(&c);
}

}  // namespace skr

namespace skr {

// ---- Lazy epoch v2: the chain only does what depends on the previous step.
// Per-step metadata (row, 1/(N q), row extent, snapshot terms) is gathered on all
// SMs first; the chain prefetches step t+1's metadata, row entries and projection
// row into registers while step t runs; the running sums of the epoch average are
// not accumulated in the chain at all — the chain logs delta_t, and afterwards
// Gamma_i = sum_{t: i_t = i} (m - t) delta_t (rows sorted stably by (i, t)) gives
//   sum_t base_t = m wbar - eta c (X^T Gamma_data + Gamma_reg),
//   sum_t h_t    = -eta (D - c) o (P^T Gamma_data + U_rows^T Gamma_reg).
struct LazyMeta {
  int64_t i, b, e;   // component, row extent (data rows)
  double q, sbar, xm;  // inv_nq, snapshot inner (or (P^{-1/2} wbar)_j), x_i . mu (or mu_j)
};

__global__ void lazy_meta_kernel(const int64_t* __restrict__ idx, int64_t m, int64_t n,
                                 const int64_t* __restrict__ rptr, const double* __restrict__ inv_nq,
                                 const double* __restrict__ s_bar, const double* __restrict__ half,
                                 const double* __restrict__ xmu, const double* __restrict__ mu,
                                 LazyMeta* __restrict__ meta) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const int64_t i = idx[t];
  LazyMeta mt;
  mt.i = i;
  mt.q = inv_nq[i];
  if (i < n) {
    mt.b = rptr[i];
    mt.e = rptr[i + 1];
    mt.sbar = s_bar[i];
    mt.xm = xmu[i];
  } else {
    mt.b = mt.e = 0;
    mt.sbar = half[i - n];
    mt.xm = mu[i - n];
  }
  meta[t] = mt;
}

struct LazyEpoch2Args {
  const int32_t* ridx;
  const double* rval;
  int64_t n, ld, k;
  const double* P;       // n x k
  const double* UT;      // d x k
  const double* D;       // k
  const double* bg;      // k: U^T mu
  const double* z0;      // k: U^T wbar
  double c, data_coef, reg_coef, eta;
  const LazyMeta* meta;  // m
  int64_t m;
  double* base;          // ld: wbar in, final base out (global when not in shared memory)
  double* dlog;          // m: delta_t
};

template <bool SMEM_BASE>
__global__ void __launch_bounds__(kLazyThreads, 1) lazy_epoch2_kernel(LazyEpoch2Args a) {
  extern __shared__ double lz2_sm[];
  const int64_t k = a.k;
  double* h = lz2_sm;      // k
  double* z = h + k;       // k
  double* Dm = z + k;      // k
  double* Dd = Dm + k;     // k
  double* bg = Dd + k;     // k
  double* red = bg + k;    // 3 x 8
  double* base = SMEM_BASE ? red + 24 : a.base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (SMEM_BASE)
    for (int64_t f = tid; f < a.ld; f += kLazyThreads) base[f] = a.base[f];
  for (int64_t l = tid; l < k; l += kLazyThreads) {
    h[l] = 0.0;
    z[l] = a.z0[l];
    Dm[l] = a.D[l] - a.c;
    Dd[l] = a.D[l];
    bg[l] = a.bg[l];
  }
  __syncthreads();
  // registers: the current step (c*), the next one (n*, its row entries in flight
  // during step t) and the metadata two steps ahead (mm, in flight during step t) —
  // every global load has a whole step to land before anything waits on it
  auto load_row = [&](const LazyMeta& mt, int32_t& f, double& v, double& r) {
    f = 0;
    v = 0.0;
    if (mt.i < a.n && mt.b + tid < mt.e) {
      f = a.ridx[mt.b + tid];
      v = a.rval[mt.b + tid];
    }
    const double* row = mt.i < a.n ? a.P + mt.i * k : a.UT + (mt.i - a.n) * k;
    r = tid < k ? row[tid] : 0.0;
  };
  LazyMeta cm, nm, mm;
  int32_t cf = 0, nf = 0;
  double cv = 0.0, cr = 0.0, nv = 0.0, nr = 0.0;
  if (a.m > 0) {
    cm = a.meta[0];
    load_row(cm, cf, cv, cr);
  }
  if (a.m > 1) nm = a.meta[1];
  for (int64_t t = 0; t < a.m; ++t) {
    if (t + 2 < a.m) mm = a.meta[t + 2];
    if (t + 1 < a.m) load_row(nm, nf, nv, nr);
    const bool data = cm.i < a.n;
    const double* row = data ? a.P + cm.i * k : a.UT + (cm.i - a.n) * k;
    double A = 0.0, B = 0.0, Cz = 0.0;
    if (data) {
      if (cm.b + tid < cm.e) A = cv * base[cf];
      for (int64_t e = cm.b + tid + kLazyThreads; e < cm.e; e += kLazyThreads) A = fma(a.rval[e], base[a.ridx[e]], A);
    } else if (tid == 0) {
      A = base[cm.i - a.n];
    }
    if (tid < k) {
      B = cr * h[tid];
      Cz = Dm[tid] * cr * z[tid];
    }
    for (int64_t l = tid + kLazyThreads; l < k; l += kLazyThreads) {
      const double rl = row[l];
      B = fma(rl, h[l], B);
      Cz = fma(Dm[l] * rl, z[l], Cz);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      A += __shfl_xor_sync(0xffffffffu, A, off);
      B += __shfl_xor_sync(0xffffffffu, B, off);
      Cz += __shfl_xor_sync(0xffffffffu, Cz, off);
    }
    if (lane == 0) {
      red[warp] = A;
      red[8 + warp] = B;
      red[16 + warp] = Cz;
    }
    __syncthreads();
    A = B = Cz = 0.0;
#pragma unroll
    for (int q = 0; q < kLazyThreads / 32; ++q) {
      A += red[q];
      B += red[8 + q];
      Cz += red[16 + q];
    }
    const double tau = a.eta * (double)t;
    const double inner = a.c * (A + B - tau * cm.xm) + Cz;
    const double delta = (data ? a.data_coef : a.reg_coef) * (inner - cm.sbar) * cm.q;
    const double ed = a.eta * delta;
    if (data) {
      if (cm.b + tid < cm.e) base[cf] -= ed * a.c * cv;
      for (int64_t e = cm.b + tid + kLazyThreads; e < cm.e; e += kLazyThreads) base[a.ridx[e]] -= ed * a.c * a.rval[e];
    } else if (tid == 0) {
      base[cm.i - a.n] -= ed * a.c;
    }
    if (tid < k) {
      h[tid] -= ed * Dm[tid] * cr;
      z[tid] -= a.eta * fma(delta, Dd[tid] * cr, bg[tid]);
    }
    for (int64_t l = tid + kLazyThreads; l < k; l += kLazyThreads) {
      const double rl = row[l];
      h[l] -= ed * Dm[l] * rl;
      z[l] -= a.eta * fma(delta, Dd[l] * rl, bg[l]);
    }
    if (tid == 0) a.dlog[t] = delta;
    __syncthreads();
    cm = nm;
    cf = nf;
    cv = nv;
    cr = nr;
    nm = mm;
  }
  if (SMEM_BASE)
    for (int64_t f = tid; f < a.ld; f += kLazyThreads) a.base[f] = base[f];
}

inline size_t lazy_epoch2_smem(int64_t k, int64_t ld_base) {
  return sizeof(double) * (5 * std::max<int64_t>(k, 1) + 24 + ld_base);
}

// gamma over rows sorted by (row, step): Gamma[row] = sum (m - t) delta_t in step order
__global__ void lazy_gamma_kernel(const int64_t* __restrict__ rows, const int64_t* __restrict__ steps, int64_t m,
                                  const double* __restrict__ dlog, double* __restrict__ gamma) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= m || (p > 0 && rows[p] == rows[p - 1])) return;
  double s = 0.0;
  for (int64_t u = p; u < m && rows[u] == rows[p]; ++u) s = fma((double)(m - steps[u]), dlog[steps[u]], s);
  gamma[rows[p]] = s;
}

// w_avg_f = wbar_f + (-eta c (g1_f + Gamma_reg_f)) / m + sum_l U_lf Sh_l / m - eta (m+1)/2 mu_f,
// Sh_l = -eta (D_l - c) (gP_l + gU_l)
__global__ void lazy_average_kernel(const double* __restrict__ snap, const double* __restrict__ g1,
                                    const double* __restrict__ gamma_reg, const double* __restrict__ gP,
                                    const double* __restrict__ gU, const double* __restrict__ UT,
                                    const double* __restrict__ D, double c, double eta, int64_t d, int64_t ld,
                                    int64_t k, int64_t m, const double* __restrict__ mu, double* __restrict__ w_avg) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= ld) return;
  if (f >= d) {
    w_avg[f] = 0.0;
    return;
  }
  const double inv_m = 1.0 / (double)m;
  double lift = 0.0;
  for (int64_t l = 0; l < k; ++l) lift = fma(UT[f * k + l], -eta * (D[l] - c) * (gP[l] + gU[l]), lift);
  const double sb = -eta * c * (g1[f] + gamma_reg[f]);
  w_avg[f] = snap[f] + sb * inv_m + lift * inv_m - 0.5 * eta * (double)(m + 1) * mu[f];
}

}  // namespace skr
