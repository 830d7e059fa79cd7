// FP64 tensor-core (DMMA) GEMM with TMA-staged tiles (the Lanczos products of
// the fp64 path: X Q^T, T^T X, Pi^T X).
//
//   C[M x N] = epi( sum_k A(m, k) B(k, n) )
//
// Each operand is either K-major (stored M x K / N x K row-major, K contiguous)
// or MN-major (stored K x M / K x N row-major), fp32 (widened on the fragment
// load) or fp64.  Tiles: CTA 128 x 128, K step 32 per stage; thread 0 issues
// 2-D TMA loads (cp.async.bulk.tensor, 128-byte rows, SWIZZLE_128B) into an
// S-stage ring (full / empty mbarriers), refilling a stage once all 8 warps
// released it (a dedicated producer warp would cap the registers at 168 and
// spill the accumulators); 8 warps each own a 32 x 64
// tile = 4 x 8 DMMA m8n8k4 fragments (64 fp64 accumulators per thread) and read
// conflict-free (K-major) or 2-way (MN-major) swizzled fragments.  Out-of-range
// rows / columns / K read as zero (TMA OOB fill), so the inner loop has no bounds
// checks.  Split-K over gridDim.z writes per-split partials summed in split order
// (deterministic), exactly like gemm_kernel.
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace skr {

constexpr int TG_BM = 128, TG_BN = 128, TG_BK = 32, TG_THREADS = 256;  // 8 warps; thread 0 also issues the TMA loads

template <class T>
constexpr int tg_tile_bytes(int rows) { return rows * TG_BK * (int)sizeof(T); }
template <class TA, class TB>
constexpr int tg_stage_bytes() { return tg_tile_bytes<TA>(TG_BM) + tg_tile_bytes<TB>(TG_BN); }
template <class TA, class TB>
constexpr int tg_stages() { return (200 * 1024) / tg_stage_bytes<TA, TB>() > 4 ? 4 : (200 * 1024) / tg_stage_bytes<TA, TB>(); }
template <class TA, class TB>
constexpr size_t tg_smem() { return (size_t)tg_stages<TA, TB>() * tg_stage_bytes<TA, TB>() + 1024 + 256; }

// Element (row index `outer` of the tile dimension that is NOT contiguous in
// memory, index `inner` of the contiguous one) of one operand tile in shared
// memory: the tile is a row of boxes, each box 128-byte rows x `rows` rows.
//   K-major tile (R = 128 M/N rows, K contiguous): boxes split K into 128-byte pieces.
//   MN-major tile (R = 32 K rows, M/N contiguous): boxes split M/N into 128-byte pieces.
template <class T>
__device__ __forceinline__ T tg_elem(const unsigned char* tile, int box_rows, int outer, int inner) {
  constexpr int E = 128 / (int)sizeof(T);  // elements per 128-byte box row
  const int box = inner / E, c = inner % E;
  return *reinterpret_cast<const T*>(tile + box * box_rows * 128 + swz128((uint32_t)outer, (uint32_t)(c * sizeof(T))));
}

template <class TA, class TB, bool A_KMAJOR, bool B_KMAJOR, class Epi, bool PARTIAL>
__global__ void __launch_bounds__(TG_THREADS, 1)
dgemm_tma_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int64_t M, int64_t N,
                 int64_t K, int64_t kchunk, Epi epi) {
  constexpr int S = tg_stages<TA, TB>();
  constexpr int A_BYTES = tg_tile_bytes<TA>(TG_BM), B_BYTES = tg_tile_bytes<TB>(TG_BN);
  constexpr int EA = 128 / (int)sizeof(TA), EB = 128 / (int)sizeof(TB);
  extern __shared__ unsigned char tg_raw[];
  // 1024-byte alignment for SWIZZLE_128B boxes
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tg_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)S * (A_BYTES + B_BYTES));
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.x * TG_BM, n0 = (int64_t)blockIdx.y * TG_BN;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk, kend = min(K, kbeg + kchunk);
  const int nk = kbeg < kend ? (int)((kend - kbeg + TG_BK - 1) / TG_BK) : 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // TMA loads of K tile `it` into stage it % S (thread 0)
  auto issue = [&](int it) {
    const int s = it % S;
    unsigned char* sa = base + (size_t)s * (A_BYTES + B_BYTES);
    unsigned char* sb = sa + A_BYTES;
    mbar_expect_tx(&full[s], (uint32_t)(A_BYTES + B_BYTES));
    // the last tile of a split is partial only when kend == K (kchunk is a multiple
    // of TG_BK), where the tensor map's own bound zero-fills it
    const int k0 = (int)(kbeg + (int64_t)it * TG_BK);
    if (A_KMAJOR) {  // tensor (K inner, M outer): boxes of EA K-columns x 128 rows
#pragma unroll
      for (int b = 0; b < TG_BK / EA; ++b) tma_load_2d(sa + b * TG_BM * 128, &ma, &full[s], k0 + b * EA, (int)m0);
    } else {         // tensor (M inner, K outer): boxes of EA M-columns x 32 K rows
#pragma unroll
      for (int b = 0; b < TG_BM / EA; ++b) tma_load_2d(sa + b * TG_BK * 128, &ma, &full[s], (int)m0 + b * EA, k0);
    }
    if (B_KMAJOR) {
#pragma unroll
      for (int b = 0; b < TG_BK / EB; ++b) tma_load_2d(sb + b * TG_BN * 128, &mb, &full[s], k0 + b * EB, (int)n0);
    } else {
#pragma unroll
      for (int b = 0; b < TG_BN / EB; ++b) tma_load_2d(sb + b * TG_BK * 128, &mb, &full[s], (int)n0 + b * EB, k0);
    }
  };
  if (tid == 0)
    for (int it = 0; it < S && it < nk; ++it) issue(it);
  {
    // ---------------- 8 warps: 4 (M) x 2 (N) warp tiles of 32 x 64 ----------------
    const int wm = (warp & 3) * 32, wn = (warp >> 2) * 64;
    const int fr = lane >> 2, fk = lane & 3;
    double acc[4][8][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int it = 0; it < nk; ++it) {
      const int s = it % S;
      mbar_wait(&full[s], (uint32_t)((it / S) & 1));
      const unsigned char* sa = base + (size_t)s * (A_BYTES + B_BYTES);
      const unsigned char* sb = sa + A_BYTES;
#pragma unroll
      for (int k4 = 0; k4 < TG_BK; k4 += 4) {
        double a[4], b[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int m = wm + 8 * i + fr, k = k4 + fk;
          a[i] = A_KMAJOR ? (double)tg_elem<TA>(sa, TG_BM, m, k) : (double)tg_elem<TA>(sa, TG_BK, k, m);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int n = wn + 8 * j + fr, k = k4 + fk;
          b[j] = B_KMAJOR ? (double)tg_elem<TB>(sb, TG_BN, n, k) : (double)tg_elem<TB>(sb, TG_BK, k, n);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
      if (tid == 0 && it + S < nk) {
        mbar_wait(&empty[s], (uint32_t)((it / S) & 1));  // every warp is done with stage s
        issue(it + S);
      }
    }
    // C fragment: row lane/4, columns 2 (lane%4) + {0, 1}
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t m = m0 + wm + 8 * i + fr;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t n = n0 + wn + 8 * j + 2 * fk;
        if constexpr (!PARTIAL && epi_has_pair<Epi>::value) {
          if (n + 1 < N) {  // n is even: one 2-element access for both columns
            epi.pair(m, n, acc[i][j][0], acc[i][j][1]);
            continue;
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (n + h >= N) continue;
          if constexpr (PARTIAL) epi(m, n + h, acc[i][j][h], (int)blockIdx.z);
          else epi(m, n + h, acc[i][j][h]);
        }
      }
    }
  }
}

}  // namespace skr
