// tcgen05 (5th-gen tensor core) GEMM for the fp32-storage Lanczos products.
//
//   C[M x N] = alpha * A . B^T      A: M x K (K-major rows, or MN-major = the
//                                   data matrix read as its transpose)
//                                   B: N x K K-major, given as hi + lo arrays
//
// computed as 3xTF32:  a_hi b_hi + a_hi b_lo + a_lo b_hi, where x_hi is x
// truncated to TF32 by the tensor core and x_lo = x - trunc_tf32(x) (exact in
// fp32), accumulated in FP32 in tensor memory (SURVEY §7 hard part 2: single
// TF32 misses the 1e-3 Ritz gate on the c4 spectrum, 3xTF32 gives ~1e-6).
//
// Shared-memory traffic is the limit for skinny products (N = k = 64..256),
// so the kernel keeps it minimal:
//   * B's lo part comes from global memory (produced once by whoever wrote B);
//   * A's lo part is computed by the converter warps straight into TENSOR
//     memory (tcgen05.st) and consumed from there (A-from-TMEM MMA), so it is
//     never written to or re-read from shared memory;
//   * for N <= 128 the hi.hi and hi.lo products are ONE MMA of width 2N over
//     the stacked [B_hi; B_lo] tile, so A_hi is read once per K step; the two
//     accumulator halves are summed in fp64 by the epilogue.
// MN-major A (the X^T products) lets X serve both orientations from one copy:
// no transposed duplicate of the data matrix is ever built.  Its converter warps
// read the unswizzled 32 x 128 tile and put both A_hi and A_lo into TMEM, so every
// MMA reads A as a K-major TMEM operand; clusters of 4 M tiles share the B tile
// by TMA multicast (tc_launch).
//
// One CTA = one 128 x BN output tile over a K-range (split-K over gridDim.z);
// N > 128 runs as several 128-wide tiles (stacked hi/lo needs 2N <= 256):
//   warp 0    TMA producer: A tile (128 x 32: one 2-D box K-major with the
//             128-byte swizzle, or four 32 x 32 boxes MN-major with the 128-byte/
//             32-byte-atom swizzle), B_hi and B_lo tiles (BN x 32), NST-stage ring;
//   warp 1    TMEM allocator + MMA issuer (one elected lane);
//   warps 2-9 A_lo converters (smem -> registers -> TMEM, one row per thread):
//             two groups of four warps (one per TMEM lane quarter) taking
//             alternate K blocks, so each scheduler has a second converter warp
//             to issue while the other waits on its shared-memory loads or on
//             tcgen05.wait::st (with one group the skinny products ran at 55 % of
//             the DRAM peak, half their stall samples on the loads' scoreboard);
//             then the epilogue: tcgen05.ld of their TMEM lane quarter ->
//             fp64 partials (transposed, split-K) or fp32 hi/lo transposed out,
//             the 16-column chunks dealt over the groups.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "tma.cuh"  // tensor maps, TMA tile loads (mbarrier / bulk-copy helpers: common.cuh)

namespace skr {

constexpr int TC_BM = 128, TC_BK = 32;
// warp 0 producer, warp 1 MMA issuer, then TC_CG groups of 4 converter warps (one per TMEM lane quarter)
// OCC = 2 (K-major A, BN = 64): two co-resident CTAs per SM, each with half the tensor
// memory, 3 stages and one converter group, so one CTA's prologue / pipeline fill /
// epilogue overlaps the other's steady state (the X Q^T products run one short-lived CTA
// per 128-row tile: 32 K blocks of work against ~10 us of un-overlapped set-up and drain).
template <bool A_MN, int BN>
constexpr int tc_occ() { return (!A_MN && BN <= 64) ? 2 : 1; }
template <bool A_MN, int BN>
constexpr int tc_cg() { return tc_occ<A_MN, BN>() == 2 ? 1 : 2; }
template <bool A_MN, int BN>
constexpr int tc_threads() { return 64 + 128 * tc_cg<A_MN, BN>(); }
constexpr int TC_A_BYTES = TC_BM * TC_BK * 4;  // 16 KB

template <bool A_MN, int BN>
constexpr int tc_stages() { return tc_occ<A_MN, BN>() == 2 ? 3 : BN <= 64 ? 6 : BN <= 128 ? 4 : 2; }
template <int BN>
constexpr bool tc_concat() { return BN <= 128; }
template <int BN>
constexpr uint32_t tc_acc_cols() { return tc_concat<BN>() ? 2 * BN : BN; }
template <int BN>
constexpr size_t tc_stage_bytes() { return (size_t)TC_A_BYTES + 2 * (size_t)BN * TC_BK * 4; }
template <bool A_MN, int BN>
constexpr size_t tc_gemm_smem() { return (size_t)tc_stages<A_MN, BN>() * tc_stage_bytes<BN>() + 1024; }


// the same box, written to the same shared offset of every CTA in ctaMask, each
// CTA's mbarrier at `bar`'s offset receiving the bytes it got
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// K-major operand tile with the 128-byte swizzle: rows of 32 fp32 (128 B),
// 8-row core groups 1024 B apart (SBO), descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_k_sw128(const void* smem) {
  const uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;      // start address
  d |= (uint64_t)1 << 16;            // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

// MN-major tf32 operand tile: the only MN-major layout the tensor core takes for
// 32-bit types is SWIZZLE_128B_BASE32B (32-byte chunks swizzled within each
// 128-byte line, pattern repeating every 4 lines; TMA's SWIZZLE_128B_ATOM_32B
// writes exactly this). Atoms of 32 M-elements (128 B) x 4 K-rows (512 B); atoms
// along M are LBO = 4 KB apart (each TMA box is 32 M x 32 K), 4-row K groups SBO =
// 512 B apart.
__device__ __forceinline__ uint64_t umma_desc_mn_sw128_32b(const void* smem) {
  const uint64_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)(4096 >> 4) << 16;  // LBO: next 32-wide M atom
  d |= (uint64_t)(512 >> 4) << 32;   // SBO: next 4-row K group
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;            // SWIZZLE_128B_BASE32B
  return d;
}

// instruction descriptor: D f32, A/B tf32, N, M = 128, A major (0 = K, 1 = MN)
__device__ __forceinline__ uint32_t tc_idesc_tf32(int n, bool a_mn) {
  uint32_t d = 0;
  d |= 1u << 4;   // D format F32
  d |= 2u << 7;   // A format TF32
  d |= 2u << 10;  // B format TF32
  if (a_mn) d |= 1u << 15;
  d |= (uint32_t)(n >> 3) << 17;
  d |= (uint32_t)(TC_BM >> 4) << 24;
  return d;
}

// A and B from shared memory
__device__ __forceinline__ void tc_mma_ss(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}
// A from tensor memory, B from shared memory
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0));
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// arrive on the barrier at `bar`'s offset in every CTA of ctaMask once the MMAs complete
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"(mask)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ float tf32_lo(float v) { return v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

struct TcGemmArgs {
  int64_t M, N, K;
  int64_t kchunk;  // K per split (multiple of TC_BK)
  double alpha;
  int mode;        // 0: fp64 partials out64[z][n][m];  1: fp32 out32[n][m] (+ lo part into out32lo)
  double* out64;
  float* out32;
  float* out32lo;
  int64_t ldt;     // row stride of out32 / out32lo
};

// CS > 1: a cluster of CS CTAs with consecutive M tiles and the same N tile / K range
// shares the B tiles — each CTA loads 1/CS of the rows and multicasts them to all, so
// L2 -> SM traffic for B drops CS-fold (B was 2/3 of each stage's bytes, re-read by
// every M tile); a stage is refilled once the MMAs of every CTA in the cluster are done
// with it (the MMA commit arrives on all CTAs' empty barriers).
template <bool A_MN, int BN, int CS>
__global__ void __launch_bounds__((tc_threads<A_MN, BN>()), (tc_occ<A_MN, BN>()))
tc_gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapBh,
                      const __grid_constant__ CUtensorMap mapBl, TcGemmArgs g) {
  constexpr int B_BYTES = BN * TC_BK * 4;
  constexpr int STAGE = (int)tc_stage_bytes<BN>();
  constexpr int NST = tc_stages<A_MN, BN>();
  constexpr int TC_CG = tc_cg<A_MN, BN>();
  constexpr uint32_t ACC = tc_acc_cols<BN>();
  // TMEM columns per stage: A_lo (32); MN-major A also keeps A_hi in TMEM (32 more):
  // every MMA then reads A as a K-major TMEM operand — the MN-major shared-memory
  // A operand ran the tensor pipe at 45 % vs 61 % for K-major (ncu, c3)
  constexpr uint32_t SLOT = A_MN ? 64u : 32u;
  constexpr uint32_t TMEM_COLS = 512 / tc_occ<A_MN, BN>();
  static_assert(tc_acc_cols<BN>() + SLOT * NST <= TMEM_COLS, "TMEM budget");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align by offsetting the shared array itself so the compiler keeps the shared address space (LDS, not LD)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // bar_tma: the A tile landed (the converters need only A); bar_tb: the B tiles landed
  __shared__ __align__(8) uint64_t bar_tma[NST], bar_tb[NST], bar_conv[NST], bar_empty[NST], bar_done;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tiles linearised N-fastest: the CTAs sharing an A tile run side by side, so A
  // comes from HBM once and from L2 for the other N tiles.  Clusters (CS > 1): groups
  // of CS consecutive M tiles, N tile next, then the next group — a cluster shares its
  // B tile, consecutive clusters share their A tiles
  const int64_t ntn = (g.N + BN - 1) / BN;
  int64_t mt, nt;
  if (CS > 1) {
    const int64_t t = blockIdx.x / CS;
    nt = t % ntn;
    mt = (t / ntn) * CS + blockIdx.x % CS;
  } else {
    mt = blockIdx.x / ntn;
    nt = blockIdx.x % ntn;
  }
  const int64_t m0 = mt * TC_BM, n0 = nt * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk;
  const int64_t kend = min(g.K, kbeg + g.kchunk);
  const int nk = kend > kbeg ? (int)((kend - kbeg + TC_BK - 1) / TC_BK) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&bar_tma[s], 1);
      mbar_init(&bar_tb[s], 1);
      mbar_init(&bar_conv[s], 128);
      mbar_init(&bar_empty[s], CS);  // one MMA-commit arrival per CTA of the cluster
    }
    mbar_init(&bar_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBl)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CS > 1) cluster_sync_all();  // every CTA's barriers exist before any multicast lands
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  uint32_t crank = 0;
  if (CS > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  constexpr uint16_t CMASK = (uint16_t)((1u << CS) - 1u);

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % NST;
        if (kb >= NST) mbar_wait(&bar_empty[s], (uint32_t)(((kb / NST) - 1) & 1));
        unsigned char* st = smem + (size_t)s * STAGE;
        mbar_expect_tx(&bar_tma[s], TC_A_BYTES);
        mbar_expect_tx(&bar_tb[s], 2 * B_BYTES);
        const int kc = (int)(kbeg + (int64_t)kb * TC_BK);
        if (A_MN) {
          // A^T stored K x M row-major (the data matrix): one unswizzled 128 (M) x 32 (K) box
          tma_load_2d(st, &mapA, &bar_tma[s], (int)m0, kc);
        } else {
          tma_load_2d(st, &mapA, &bar_tma[s], kc, (int)m0);
        }
        if (CS > 1) {
          // this CTA's BN/CS rows of B_hi and B_lo, to every CTA of the cluster
          constexpr int SR = BN / CS;
          const int off = (int)crank * SR;
          tma_load_2d_mc(st + TC_A_BYTES + off * 128, &mapBh, &bar_tb[s], kc, (int)n0 + off, CMASK);
          tma_load_2d_mc(st + TC_A_BYTES + B_BYTES + off * 128, &mapBl, &bar_tb[s], kc, (int)n0 + off, CMASK);
        } else {
          tma_load_2d(st + TC_A_BYTES, &mapBh, &bar_tb[s], kc, (int)n0);
          tma_load_2d(st + TC_A_BYTES + B_BYTES, &mapBl, &bar_tb[s], kc, (int)n0);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t id_w = tc_idesc_tf32(tc_concat<BN>() ? 2 * BN : BN, A_MN);  // A_hi x B (stacked when concat)
    const uint32_t id_n = tc_idesc_tf32(BN, A_MN);
    const uint32_t id_t = tc_idesc_tf32(BN, false);  // A from TMEM is K-major by construction
    const uint32_t id_wt = tc_idesc_tf32(tc_concat<BN>() ? 2 * BN : BN, false);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % NST;
      mbar_wait(&bar_tma[s], (uint32_t)((kb / NST) & 1));
      mbar_wait(&bar_tb[s], (uint32_t)((kb / NST) & 1));
      mbar_wait(&bar_conv[s], (uint32_t)((kb / NST) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (lane == 0) {
        const unsigned char* st = smem + (size_t)s * STAGE;
        const unsigned char* bhi = st + TC_A_BYTES;
        const unsigned char* blo = st + TC_A_BYTES + B_BYTES;
        const uint32_t alo = tmem + ACC + SLOT * (uint32_t)s;
        const uint32_t ahi = alo + 32u;  // A_MN only
#pragma unroll
        for (int k = 0; k < TC_BK / 8; ++k) {  // UMMA_K = 8 tf32
          const uint64_t dah = umma_desc_k_sw128(st + 32 * k);  // K-major A (A_MN: unused)
          const uint64_t dbh = umma_desc_k_sw128(bhi + 32 * k);
          const uint32_t acc0 = (kb > 0 || k > 0) ? 1u : 0u;
          if (A_MN) {
            if (tc_concat<BN>()) {
              tc_mma_ts(tmem, ahi + 8 * k, dbh, id_wt, acc0);  // [hi.hi | hi.lo] in columns [0, 2 BN)
              tc_mma_ts(tmem, alo + 8 * k, dbh, id_t, 1u);     // + lo.hi into [0, BN)
            } else {
              const uint64_t dbl = umma_desc_k_sw128(blo + 32 * k);
              tc_mma_ts(tmem, alo + 8 * k, dbh, id_t, acc0);
              tc_mma_ts(tmem, ahi + 8 * k, dbl, id_t, 1u);
              tc_mma_ts(tmem, ahi + 8 * k, dbh, id_t, 1u);
            }
          } else if (tc_concat<BN>()) {
            tc_mma_ss(tmem, dah, dbh, id_w, acc0);         // [hi.hi | hi.lo] in columns [0, 2 BN)
            tc_mma_ts(tmem, alo + 8 * k, dbh, id_t, 1u);   // + lo.hi into [0, BN)
          } else {
            const uint64_t dbl = umma_desc_k_sw128(blo + 32 * k);
            tc_mma_ts(tmem, alo + 8 * k, dbh, id_t, acc0);  // small terms first
            tc_mma_ss(tmem, dah, dbl, id_n, 1u);
            tc_mma_ss(tmem, dah, dbh, id_n, 1u);
          }
        }
        if (CS > 1) tc_commit_mc(&bar_empty[s], CMASK);  // every CTA may refill this stage (its B slice lands everywhere)
        else tc_commit(&bar_empty[s]);                 // smem stage + TMEM A_lo slot reusable
        if (kb == nk - 1) tc_commit(&bar_done);   // accumulator complete
      }
      __syncwarp();
    }
    if (nk == 0 && lane == 0) mbar_arrive_local(&bar_done);
  } else {
    // A_lo converters: thread owns A row (lane quarter of its warp) -> TMEM lane
    const int quarter = warp & 3;
    const int grp = (warp - 2) >> 2;    // converter group: K blocks grp, grp + TC_CG, ...
    const int r = 32 * quarter + lane;  // M index within the tile = TMEM lane
    for (int kb = grp; kb < nk; kb += TC_CG) {
      const int s = kb % NST;
      mbar_wait(&bar_tma[s], (uint32_t)((kb / NST) & 1));
      const unsigned char* st = smem + (size_t)s * STAGE;
      uint32_t v[32], h[32];
      if (A_MN) {
        // element (r, k) at line k, word r (unswizzled 32 x 128 box): conflict-free per k
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float a = *reinterpret_cast<const float*>(st + 512 * k + 4 * r);
          h[k] = __float_as_uint(a);  // read as TF32 by the MMA, like the shared-memory operand
          v[k] = __float_as_uint(tf32_lo(a));
        }
      } else {
        // row r = 128 contiguous bytes, 16-byte chunk j stored at slot j ^ (r%8)
        const unsigned char* row = st + 128 * r;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 q = *reinterpret_cast<const float4*>(row + 16 * (j ^ (r & 7)));
          v[4 * j + 0] = __float_as_uint(tf32_lo(q.x));
          v[4 * j + 1] = __float_as_uint(tf32_lo(q.y));
          v[4 * j + 2] = __float_as_uint(tf32_lo(q.z));
          v[4 * j + 3] = __float_as_uint(tf32_lo(q.w));
        }
      }
      const uint32_t taddr = tmem + ((uint32_t)(32 * quarter) << 16) + ACC + SLOT * (uint32_t)s;
      if (A_MN)
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr + 32u),
            "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]), "r"(h[8]),
            "r"(h[9]), "r"(h[10]), "r"(h[11]), "r"(h[12]), "r"(h[13]), "r"(h[14]), "r"(h[15]), "r"(h[16]),
            "r"(h[17]), "r"(h[18]), "r"(h[19]), "r"(h[20]), "r"(h[21]), "r"(h[22]), "r"(h[23]), "r"(h[24]),
            "r"(h[25]), "r"(h[26]), "r"(h[27]), "r"(h[28]), "r"(h[29]), "r"(h[30]), "r"(h[31])
            : "memory");
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
          "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
          "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
          "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive_local(&bar_conv[s]);
    }
    // epilogue: TMEM lane quarter -> rows m0 + r
    mbar_wait(&bar_done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int64_t row = m0 + r;
    for (int c0 = 16 * grp; c0 < BN; c0 += 16 * TC_CG) {
      uint32_t a[16], b[16];
      const uint32_t taddr = tmem + ((uint32_t)(32 * quarter) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]),
            "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15])
          : "r"(taddr));
      if (tc_concat<BN>()) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]),
              "=r"(b[8]), "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15])
            : "r"(taddr + (uint32_t)BN));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < g.M) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t col = n0 + c0 + j;
          if (col >= g.N) continue;
          double v = (double)__uint_as_float(a[j]);
          if (tc_concat<BN>()) v += (double)__uint_as_float(b[j]);
          v *= g.alpha;
          if (g.mode == 0) {
            g.out64[((int64_t)blockIdx.z * g.N + col) * g.M + row] = v;
          } else {
            const float f = (float)v;
            g.out32[col * g.ldt + row] = f;
            if (g.out32lo) g.out32lo[col * g.ldt + row] = tf32_lo(f);
          }
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
  if (CS > 1) cluster_sync_all();  // no CTA exits while peers may still multicast into it / arrive on it
}

// lo = x - trunc_tf32(x) of an fp32 matrix (the B operands' lo arrays)
__global__ void tf32_lo_kernel(const float* __restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                               float* __restrict__ dst, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, cc = e % cols;
    dst[r * ldd + cc] = tf32_lo(src[r * lds + cc]);
  }
}

// fp64 -> fp32 hi (round to nearest) + lo (tf32 residual of the fp32 value), rows x cols
__global__ void f64_to_tf32x2_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                                     float* __restrict__ hi, float* __restrict__ lo, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, cc = e % cols;
    const float f = (float)src[r * lds + cc];
    hi[r * ldd + cc] = f;
    lo[r * ldd + cc] = tf32_lo(f);
  }
}

// C^T-oriented split-K sum: part[z][n][m] (fp64) -> out[n * ldo + m] = sum_z in split order
__global__ void tc_splitk_reduce_kernel(const double* __restrict__ part, int64_t M, int64_t N, int splits,
                                        double* __restrict__ out, int64_t ldo) {
  const int64_t total = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[(int64_t)z * total + e];
    const int64_t nn = e / M, mm = e % M;
    out[nn * ldo + mm] = s;
  }
}

}  // namespace skr
