// tcgen05 (5th-gen tensor core) GEMM for the fp32-storage Lanczos products.
//
//   C[M x N] = alpha * A[M x K] . B[N x K]^T      (A, B fp32, both K-major)
//
// computed as 3xTF32:  a_hi b_hi + a_hi b_lo + a_lo b_hi  with a_hi = a
// truncated to TF32 by the tensor core and a_lo = a - trunc_tf32(a) (exact in
// fp32), accumulated in FP32 in tensor memory (SURVEY §7 hard part 2: single
// TF32 misses the 1e-3 Ritz gate on the c4 spectrum, 3xTF32 gives ~1e-6).
//
// One CTA = one 128 x BN output tile over a K-range (split-K over gridDim.z):
//   warp 0   TMA producer: 2-D tensor-map loads of 128x32 (A) and BNx32 (B)
//            fp32 tiles, 128-byte swizzle, into an NST-stage ring;
//   warp 1   MMA issuer: allocates TMEM, one elected lane issues
//            tcgen05.mma.cta_group::1.kind::tf32 (4 K-steps x 3 products per
//            stage), tcgen05.commit frees the stage / signals the epilogue;
//   warps 2-5 split the landed tiles into lo parts (same swizzled layout,
//            element-wise), fence to the async proxy, then run the epilogue:
//            tcgen05.ld of their TMEM lane quarter -> fp64 partials (split-K)
//            or a transposed fp32 output.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "fullgrad.cuh"  // mbarrier / bulk-copy helpers

namespace skr {

constexpr int TC_BM = 128, TC_BK = 32, TC_THREADS = 192;
// pipeline depth by tile width (stage = hi+lo of A and B: 32 KB + BN*256 B)
template <int BN>
constexpr int tc_stages() { return BN <= 64 ? 4 : BN <= 128 ? 3 : 2; }

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major operand tile in shared memory with the 128-byte swizzle: rows of
// 32 fp32 (128 B), 8-row core groups 1024 B apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_k_sw128(const void* smem) {
  const uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;           // start address
  d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

template <int BN>
__device__ __forceinline__ uint32_t tc_idesc_tf32() {
  uint32_t d = 0;
  d |= 1u << 4;                 // D format F32
  d |= 2u << 7;                 // A format TF32
  d |= 2u << 10;                // B format TF32
  d |= (uint32_t)(BN >> 3) << 17;
  d |= (uint32_t)(TC_BM >> 4) << 24;
  return d;
}

__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0));
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

struct TcGemmArgs {
  int64_t M, N, K;
  int64_t kchunk;      // K per split (multiple of TC_BK)
  double alpha;
  int mode;            // 0: fp64 partials out64[z][m][n] (ld N); 1: fp32 transposed out32[n][m] (ld ldt)
  double* out64;
  float* out32;
  int64_t ldt;
};

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
tc_gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      TcGemmArgs g) {
  constexpr int A_BYTES = TC_BM * TC_BK * 4, B_BYTES = BN * TC_BK * 4;
  constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // hi + lo of A and B
  constexpr int TC_NST = tc_stages<BN>();
  constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar_tma[TC_NST], bar_conv[TC_NST], bar_empty[TC_NST], bar_done;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.x * TC_BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk;
  const int64_t kend = min(g.K, kbeg + g.kchunk);
  const int nk = kend > kbeg ? (int)((kend - kbeg + TC_BK - 1) / TC_BK) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < TC_NST; ++s) {
      mbar_init(&bar_tma[s], 1);
      mbar_init(&bar_conv[s], 128);
      mbar_init(&bar_empty[s], 1);
    }
    mbar_init(&bar_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % TC_NST;
        if (kb >= TC_NST) mbar_wait(&bar_empty[s], (uint32_t)(((kb / TC_NST) - 1) & 1));
        unsigned char* st = smem + (size_t)s * STAGE;
        mbar_expect_tx(&bar_tma[s], A_BYTES + B_BYTES);
        const int kc = (int)(kbeg + (int64_t)kb * TC_BK);
        tma_load_2d(st, &mapA, &bar_tma[s], kc, (int)m0);
        tma_load_2d(st + 2 * A_BYTES, &mapB, &bar_tma[s], kc, (int)n0);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = tc_idesc_tf32<BN>();
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % TC_NST;
      mbar_wait(&bar_conv[s], (uint32_t)((kb / TC_NST) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        unsigned char* st = smem + (size_t)s * STAGE;
        const unsigned char* ahi = st;
        const unsigned char* alo = st + A_BYTES;
        const unsigned char* bhi = st + 2 * A_BYTES;
        const unsigned char* blo = st + 2 * A_BYTES + B_BYTES;
#pragma unroll
        for (int k = 0; k < TC_BK / 8; ++k) {  // UMMA_K = 8 tf32 = 32 bytes
          const uint64_t dah = umma_desc_k_sw128(ahi + 32 * k), dal = umma_desc_k_sw128(alo + 32 * k);
          const uint64_t dbh = umma_desc_k_sw128(bhi + 32 * k), dbl = umma_desc_k_sw128(blo + 32 * k);
          const uint32_t acc0 = (kb > 0 || k > 0) ? 1u : 0u;
          tc_mma_tf32(tmem, dal, dbh, idesc, acc0);  // small terms first
          tc_mma_tf32(tmem, dah, dbl, idesc, 1u);
          tc_mma_tf32(tmem, dah, dbh, idesc, 1u);
        }
        tc_commit(&bar_empty[s]);            // smem stage reusable once these MMAs retire
        if (kb == nk - 1) tc_commit(&bar_done);  // accumulator complete
      }
      __syncwarp();
    }
    if (nk == 0 && lane == 0) mbar_arrive_local(&bar_done);
  } else {
    // converters + epilogue: 128 threads (warps 2..5)
    const int ct = threadIdx.x - 64;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % TC_NST;
      mbar_wait(&bar_tma[s], (uint32_t)((kb / TC_NST) & 1));
      unsigned char* st = smem + (size_t)s * STAGE;
      // lo = a - trunc_tf32(a), element-wise over the (swizzled) raw tiles
      const float4* ah = reinterpret_cast<const float4*>(st);
      float4* al = reinterpret_cast<float4*>(st + A_BYTES);
      for (int e = ct; e < A_BYTES / 16; e += 128) {
        float4 v = ah[e], r;
        r.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
        r.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
        r.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
        r.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        al[e] = r;
      }
      const float4* bh = reinterpret_cast<const float4*>(st + 2 * A_BYTES);
      float4* bl = reinterpret_cast<float4*>(st + 2 * A_BYTES + B_BYTES);
      for (int e = ct; e < B_BYTES / 16; e += 128) {
        float4 v = bh[e], r;
        r.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
        r.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
        r.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
        r.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
        bl[e] = r;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core reads
      mbar_arrive_local(&bar_conv[s]);
    }
    // epilogue: TMEM lane quarter (warp % 4) -> rows m0 + 32*(warp%4) + lane
    mbar_wait(&bar_done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int quarter = warp & 3;
    const int64_t row = m0 + 32 * quarter + lane;
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t r[16];
      const uint32_t taddr = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < g.M) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t col = n0 + c0 + j;
          if (col >= g.N) continue;
          const double v = g.alpha * (double)__uint_as_float(r[j]);
          if (g.mode == 0) g.out64[((int64_t)blockIdx.z * g.M + row) * g.N + col] = v;
          else g.out32[col * g.ldt + row] = (float)v;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

template <int BN>
constexpr size_t tc_gemm_smem() {
  return (size_t)tc_stages<BN>() * (2 * TC_BM * TC_BK * 4 + 2 * BN * TC_BK * 4) + 1024;
}

}  // namespace skr
