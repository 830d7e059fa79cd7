// Tiled FP64-accumulate SIMT GEMM for the tall-skinny products around the hot
// path (Krylov blocks, Rayleigh-Ritz Gram, preconditioner build).
//
//   C[M x N] (+)= alpha * op(A)[M x K] * op(B)[K x N]
//
// A/B element types are float or double (fp32 data is widened to fp64 in the
// shared-memory stage, so every product and sum is fp64 — the precision the
// reference computes in).  op() is selected at compile time:
//   A_T = false: A(m,k) = A[m*lda + k]     A_T = true: A(m,k) = A[k*lda + m]
//   B_T = false: B(k,n) = B[k*ldb + n]     B_T = true: B(k,n) = B[n*ldb + k]
// Split-K (gridDim.z) writes per-split partials that a second kernel sums in a
// fixed order, so results are run-to-run deterministic.
#pragma once

#include "common.cuh"

namespace skr {

constexpr int GEMM_BM = 64, GEMM_BN = 64, GEMM_BK = 16, GEMM_THREADS = 256;
constexpr int GEMM_PAD = 2;

template <class T>
__device__ __forceinline__ double ld_as_double(const T* p) { return static_cast<double>(__ldg(p)); }

// Epilogue receives the fp64 accumulator of one output element.
struct EpiStore {  // C = alpha*acc + beta*C  (beta ignored when 0)
  double* C;
  int64_t ldc;
  double alpha, beta;
  __device__ void operator()(int64_t m, int64_t n, double acc) const {
    double* c = C + m * ldc + n;
    *c = beta == 0.0 ? alpha * acc : alpha * acc + beta * *c;
  }
};

struct EpiPartial {  // split-K partial: ws[z][m][n]
  double* ws;
  int64_t M, N;
  __device__ void operator()(int64_t m, int64_t n, double acc, int z) const {
    ws[(int64_t)z * M * N + m * N + n] = acc;
  }
};

template <class TA, class TB, bool A_T, bool B_T, class Epi, bool PARTIAL>
__global__ void __launch_bounds__(GEMM_THREADS)
gemm_kernel(int64_t M, int64_t N, int64_t K, const TA* __restrict__ A, int64_t lda,
            const TB* __restrict__ B, int64_t ldb, int64_t kchunk, Epi epi) {
  __shared__ __align__(16) double As[2][GEMM_BK][GEMM_BM + GEMM_PAD];
  __shared__ __align__(16) double Bs[2][GEMM_BK][GEMM_BN + GEMM_PAD];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.x * GEMM_BM;
  const int64_t n0 = (int64_t)blockIdx.y * GEMM_BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);

  double acc[4][4] = {};
  double ra[4], rb[4];

  auto load_a = [&](int64_t k0) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      int mm, kk;
      if (!A_T) { kk = tid % 16; mm = tid / 16 + 16 * p; }
      else      { mm = tid % 64; kk = tid / 64 + 4 * p; }
      const int64_t m = m0 + mm, k = k0 + kk;
      ra[p] = (m < M && k < kend) ? ld_as_double(A_T ? A + k * lda + m : A + m * lda + k) : 0.0;
    }
  };
  auto load_b = [&](int64_t k0) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      int nn, kk;
      if (!B_T) { nn = tid % 64; kk = tid / 64 + 4 * p; }
      else      { kk = tid % 16; nn = tid / 16 + 16 * p; }
      const int64_t n = n0 + nn, k = k0 + kk;
      rb[p] = (n < N && k < kend) ? ld_as_double(B_T ? B + n * ldb + k : B + k * ldb + n) : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      int mm, kk;
      if (!A_T) { kk = tid % 16; mm = tid / 16 + 16 * p; }
      else      { mm = tid % 64; kk = tid / 64 + 4 * p; }
      As[buf][kk][mm] = ra[p];
      int nn;
      if (!B_T) { nn = tid % 64; kk = tid / 64 + 4 * p; }
      else      { kk = tid % 16; nn = tid / 16 + 16 * p; }
      Bs[buf][kk][nn] = rb[p];
    }
  };

  if (kbeg < kend) {
    load_a(kbeg);
    load_b(kbeg);
    store(0);
    __syncthreads();
    int buf = 0;
    for (int64_t k0 = kbeg; k0 < kend; k0 += GEMM_BK) {
      const bool more = k0 + GEMM_BK < kend;
      if (more) {
        load_a(k0 + GEMM_BK);
        load_b(k0 + GEMM_BK);
      }
#pragma unroll
      for (int kk = 0; kk < GEMM_BK; ++kk) {
        const double2 a01 = *reinterpret_cast<const double2*>(&As[buf][kk][ty * 4]);
        const double2 a23 = *reinterpret_cast<const double2*>(&As[buf][kk][ty * 4 + 2]);
        const double2 b01 = *reinterpret_cast<const double2*>(&Bs[buf][kk][tx * 4]);
        const double2 b23 = *reinterpret_cast<const double2*>(&Bs[buf][kk][tx * 4 + 2]);
        const double a[4] = {a01.x, a01.y, a23.x, a23.y};
        const double b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      if (more) {
        store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n >= N) continue;
      if constexpr (PARTIAL) epi(m, n, acc[i][j], (int)blockIdx.z);
      else epi(m, n, acc[i][j]);
    }
  }
}

// Sum split-K partials in split order, then apply the final epilogue.
template <class Epi>
__global__ void splitk_reduce_kernel(const double* __restrict__ ws, int64_t M, int64_t N,
                                     int splits, Epi epi) {
  const int64_t total = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += ws[(int64_t)z * total + e];
    epi(e / N, e % N, s);
  }
}

// Host driver.  `splits` <= 0 picks a split count that fills ~2 waves.
template <class TA, class TB, bool A_T, bool B_T, class Epi>
void gemm(Ctx* ctx, int64_t M, int64_t N, int64_t K, const TA* A, int64_t lda, const TB* B,
          int64_t ldb, Epi epi, int splits = 0) {
  if (M <= 0 || N <= 0) return;
  const int64_t tiles = (int64_t)ceil_div(M, GEMM_BM) * ceil_div(N, GEMM_BN);
  if (splits <= 0) {
    const int64_t want = 2LL * ctx->sm_count;
    splits = tiles >= want ? 1 : (int)std::min<int64_t>((want + tiles - 1) / tiles,
                                                         std::max<int64_t>(1, K / (4 * GEMM_BK)));
    splits = std::max(1, std::min(splits, 1024));
  }
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = (kchunk + GEMM_BK - 1) / GEMM_BK * GEMM_BK;
  if (kchunk == 0) kchunk = GEMM_BK;
  splits = (int)std::max<int64_t>(1, (K + kchunk - 1) / kchunk);
  dim3 grid(ceil_div(M, GEMM_BM), ceil_div(N, GEMM_BN), splits);
  if (splits == 1) {
    gemm_kernel<TA, TB, A_T, B_T, Epi, false><<<grid, GEMM_THREADS, 0, ctx->stream>>>(
        M, N, K, A, lda, B, ldb, kchunk, epi);
    SKR_LAUNCHED(ctx);
    return;
  }
  DBuf<double> ws((size_t)splits * M * N, ctx->stream);
  EpiPartial part{ws.get(), M, N};
  gemm_kernel<TA, TB, A_T, B_T, EpiPartial, true><<<grid, GEMM_THREADS, 0, ctx->stream>>>(
      M, N, K, A, lda, B, ldb, kchunk, part);
  SKR_LAUNCHED(ctx);
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(M * N, 256), 4LL * ctx->sm_count);
  splitk_reduce_kernel<Epi><<<blocks, 256, 0, ctx->stream>>>(ws.get(), M, N, splits, epi);
  SKR_LAUNCHED(ctx);
}

}  // namespace skr
