// FP64 tensor-core (DMMA) GEMM for the tall-skinny products around the hot path
// (fp64 Krylov blocks, Rayleigh-Ritz Gram, preconditioner build).
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
#include "tma.cuh"

namespace skr {

constexpr int GEMM_BK = 16, GEMM_THREADS = 256;

template <class T>
__device__ __forceinline__ double ld_as_double(const T* p) { return static_cast<double>(__ldg(p)); }

// Epilogue receives the fp64 accumulator of one output element.  An epilogue with
// `static constexpr bool kPair = true` also takes two adjacent columns (n even,
// n + 1 < N) in one call, so it can use 2-element vector loads and stores.
template <class E, class = void>
struct epi_has_pair { static constexpr bool value = false; };
template <class E>
struct epi_has_pair<E, decltype((void)E::kPair)> { static constexpr bool value = E::kPair; };
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

// FP64 tensor-core GEMM (DMMA, mma.sync m8n8k4 f64): CTA tile BM x BN x 16,
// 8 warps of 32 x 32, register-staged double-buffered shared tiles (k-major, so
// the m8n8k4 fragment loads are two conflict-free wavefronts).
constexpr int GEMM_SP = 4;  // row pad (doubles): k-rows 0..3 start 8 banks apart
constexpr size_t gemm_smem(int bm, int bn) { return sizeof(double) * 2 * GEMM_BK * (bm + bn + 2 * GEMM_SP); }

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <class TA, class TB, bool A_T, bool B_T, class Epi, bool PARTIAL, int BM, int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 2)
gemm_kernel(int64_t M, int64_t N, int64_t K, const TA* __restrict__ A, int64_t lda,
            const TB* __restrict__ B, int64_t ldb, int64_t kchunk, Epi epi) {
  static_assert((BM / 32) * (BN / 32) == GEMM_THREADS / 32, "8 warps of 32x32");
  constexpr int PA = (BM * GEMM_BK) / GEMM_THREADS, PB = (BN * GEMM_BK) / GEMM_THREADS;
  constexpr int SP = GEMM_SP;
  extern __shared__ __align__(16) double gemm_sm[];
  auto As = reinterpret_cast<double(*)[GEMM_BK][BM + SP]>(gemm_sm);
  auto Bs = reinterpret_cast<double(*)[GEMM_BK][BN + SP]>(gemm_sm + 2 * GEMM_BK * (BM + SP));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp % (BM / 32)) * 32, wn = (warp / (BM / 32)) * 32;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);

  double acc[4][4][2] = {};
  double ra[PA], rb[PB];

  // element p of this thread's share of the A tile: (mm, kk)
  auto a_idx = [&](int p, int& mm, int& kk) {
    const int e = tid + p * GEMM_THREADS;
    if (!A_T) { kk = e % GEMM_BK; mm = e / GEMM_BK; }   // k fastest: row-contiguous A
    else      { mm = e % BM; kk = e / BM; }             // m fastest: column-contiguous A
  };
  auto b_idx = [&](int p, int& nn, int& kk) {
    const int e = tid + p * GEMM_THREADS;
    if (!B_T) { nn = e % BN; kk = e / BN; }
    else      { kk = e % GEMM_BK; nn = e / GEMM_BK; }
  };
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int p = 0; p < PA; ++p) {
      int mm, kk;
      a_idx(p, mm, kk);
      const int64_t m = m0 + mm, k = k0 + kk;
      ra[p] = (m < M && k < kend) ? ld_as_double(A_T ? A + k * lda + m : A + m * lda + k) : 0.0;
    }
#pragma unroll
    for (int p = 0; p < PB; ++p) {
      int nn, kk;
      b_idx(p, nn, kk);
      const int64_t n = n0 + nn, k = k0 + kk;
      rb[p] = (n < N && k < kend) ? ld_as_double(B_T ? B + n * ldb + k : B + k * ldb + n) : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int p = 0; p < PA; ++p) {
      int mm, kk;
      a_idx(p, mm, kk);
      As[buf][kk][mm] = ra[p];
    }
#pragma unroll
    for (int p = 0; p < PB; ++p) {
      int nn, kk;
      b_idx(p, nn, kk);
      Bs[buf][kk][nn] = rb[p];
    }
  };

  if (kbeg < kend) {
    load(kbeg);
    store(0);
    __syncthreads();
    int buf = 0;
    const int fr = lane >> 2, fk = lane & 3;
    for (int64_t k0 = kbeg; k0 < kend; k0 += GEMM_BK) {
      const bool more = k0 + GEMM_BK < kend;
      if (more) load(k0 + GEMM_BK);
#pragma unroll
      for (int k4 = 0; k4 < GEMM_BK; k4 += 4) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[buf][k4 + fk][wm + 8 * i + fr];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[buf][k4 + fk][wn + 8 * j + fr];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
      if (more) {
        store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
    }
  }
  // C fragment: row lane/4, columns 2 (lane%4) + {0, 1}
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + wm + 8 * i + (lane >> 2);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t n = n0 + wn + 8 * j + 2 * (lane & 3) + h;
        if (n >= N) continue;
        if constexpr (PARTIAL) epi(m, n, acc[i][j][h], (int)blockIdx.z);
        else epi(m, n, acc[i][j][h]);
      }
    }
  }
}

}  // namespace skr
#include "gemm_tma.cuh"
namespace skr {

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
template <class TA, class TB, bool A_T, bool B_T, class Epi, int BM, int BN>
void gemm_tiled(Ctx* ctx, int64_t M, int64_t N, int64_t K, const TA* A, int64_t lda, const TB* B,
                int64_t ldb, Epi epi, int splits) {
  const int64_t tiles = (int64_t)ceil_div(M, BM) * ceil_div(N, BN);
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
  dim3 grid(ceil_div(M, BM), ceil_div(N, BN), splits);
  constexpr size_t smem = gemm_smem(BM, BN);
  if (splits == 1) {
    configure_once((const void*)gemm_kernel<TA, TB, A_T, B_T, Epi, false, BM, BN>, [&] {
      SKR_CUDA(cudaFuncSetAttribute(gemm_kernel<TA, TB, A_T, B_T, Epi, false, BM, BN>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    gemm_kernel<TA, TB, A_T, B_T, Epi, false, BM, BN><<<grid, GEMM_THREADS, smem, ctx->stream>>>(
        M, N, K, A, lda, B, ldb, kchunk, epi);
    SKR_LAUNCHED(ctx);
    return;
  }
  DBuf<double> ws((size_t)splits * M * N, ctx->stream);
  EpiPartial part{ws.get(), M, N};
  configure_once((const void*)gemm_kernel<TA, TB, A_T, B_T, EpiPartial, true, BM, BN>, [&] {
    SKR_CUDA(cudaFuncSetAttribute(gemm_kernel<TA, TB, A_T, B_T, EpiPartial, true, BM, BN>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  gemm_kernel<TA, TB, A_T, B_T, EpiPartial, true, BM, BN><<<grid, GEMM_THREADS, smem, ctx->stream>>>(
      M, N, K, A, lda, B, ldb, kchunk, part);
  SKR_LAUNCHED(ctx);
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(M * N, 256), 4LL * ctx->sm_count);
  splitk_reduce_kernel<Epi><<<blocks, 256, 0, ctx->stream>>>(ws.get(), M, N, splits, epi);
  SKR_LAUNCHED(ctx);
}

// TMA-staged DMMA GEMM (gemm_tma.cuh) for the large products: needs 16-byte aligned
// bases and row strides (TMA), int32 coordinates.  Returns false when not eligible.
template <class TA, class TB, bool A_T, bool B_T, class Epi>
bool gemm_tma(Ctx* ctx, int64_t M, int64_t N, int64_t K, const TA* A, int64_t lda, const TB* B, int64_t ldb, Epi epi,
              int splits) {
  static const bool off = getenv("SKR_GEMM_LEGACY") != nullptr;
  if (off) return false;
  constexpr bool AK = !A_T, BK_ = B_T;  // K-major operands
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) return false;
  if ((lda * (int64_t)sizeof(TA)) % 16 || (ldb * (int64_t)sizeof(TB)) % 16) return false;
  if (M >= (1LL << 31) || N >= (1LL << 31) || K >= (1LL << 31)) return false;
  // small products, and products narrower than the 128 x 128 tile in M or N (the
  // register-staged kernel's 64 x 128 / 128 x 64 tiles waste less there)
  // and short K (the rank-k X~ product: with 1 CTA per SM the 3-4 stage ring never fills,
  // while the register-staged kernel runs 2 CTAs per SM)
  if ((double)M * (double)N * (double)K < 3e8 || M < TG_BM || N < TG_BN || K < 512) return false;
  constexpr int EA = 128 / (int)sizeof(TA), EB = 128 / (int)sizeof(TB);
  const CUtensorMap ma = AK ? make_tmap_2d(A, sizeof(TA), M, K, lda, TG_BM, EA, CU_TENSOR_MAP_SWIZZLE_128B)
                            : make_tmap_2d(A, sizeof(TA), K, M, lda, TG_BK, EA, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap mb = BK_ ? make_tmap_2d(B, sizeof(TB), N, K, ldb, TG_BN, EB, CU_TENSOR_MAP_SWIZZLE_128B)
                             : make_tmap_2d(B, sizeof(TB), K, N, ldb, TG_BK, EB, CU_TENSOR_MAP_SWIZZLE_128B);
  const int64_t tiles = (int64_t)ceil_div(M, TG_BM) * ceil_div(N, TG_BN);
  if (splits <= 0) {
    // one CTA per SM: pick the split count whose last wave is fullest (fewest splits on ties)
    const int64_t kmax = std::max<int64_t>(1, std::min<int64_t>(256, K / (8 * TG_BK)));
    double best = -1.0;
    splits = 1;
    for (int64_t sp = 1; sp <= kmax; ++sp) {
      const int64_t ctas = tiles * sp, waves = (ctas + ctx->sm_count - 1) / ctx->sm_count;
      if (waves > 8 && sp > 1) break;
      const double eff = (double)ctas / (double)(waves * ctx->sm_count);
      if (eff > best + 0.02) {
        best = eff;
        splits = (int)sp;
      }
    }
  }
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = std::max<int64_t>(TG_BK, (kchunk + TG_BK - 1) / TG_BK * TG_BK);
  splits = (int)std::max<int64_t>(1, (K + kchunk - 1) / kchunk);
  const dim3 grid(ceil_div(M, TG_BM), ceil_div(N, TG_BN), splits);
  constexpr size_t smem = tg_smem<TA, TB>();
  if (splits == 1) {
    auto k = dgemm_tma_kernel<TA, TB, AK, BK_, Epi, false>;
    configure_once((const void*)k, [&] {
      SKR_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    });
    k<<<grid, TG_THREADS, smem, ctx->stream>>>(ma, mb, M, N, K, kchunk, epi);
    SKR_LAUNCHED(ctx);
    return true;
  }
  DBuf<double> ws((size_t)splits * M * N, ctx->stream);
  EpiPartial part{ws.get(), M, N};
  auto k = dgemm_tma_kernel<TA, TB, AK, BK_, EpiPartial, true>;
  configure_once((const void*)k, [&] {
    SKR_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  });
  k<<<grid, TG_THREADS, smem, ctx->stream>>>(ma, mb, M, N, K, kchunk, part);
  SKR_LAUNCHED(ctx);
  const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(M * N, 256), 4LL * ctx->sm_count);
  splitk_reduce_kernel<Epi><<<blocks, 256, 0, ctx->stream>>>(ws.get(), M, N, splits, epi);
  SKR_LAUNCHED(ctx);
  return true;
}

template <class TA, class TB, bool A_T, bool B_T, class Epi>
void gemm(Ctx* ctx, int64_t M, int64_t N, int64_t K, const TA* A, int64_t lda, const TB* B,
          int64_t ldb, Epi epi, int splits = 0) {
  if (M <= 0 || N <= 0) return;
  if (gemm_tma<TA, TB, A_T, B_T, Epi>(ctx, M, N, K, A, lda, B, ldb, epi, splits)) return;
  if (M <= 64 && N > 64)
    gemm_tiled<TA, TB, A_T, B_T, Epi, 64, 128>(ctx, M, N, K, A, lda, B, ldb, epi, splits);
  else
    gemm_tiled<TA, TB, A_T, B_T, Epi, 128, 64>(ctx, M, N, K, A, lda, B, ldb, epi, splits);
}

}  // namespace skr
