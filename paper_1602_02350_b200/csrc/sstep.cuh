// K10 s-step: the SVRG inner loop (svrg.cpp:18-54, :188-195) reformulated over
// blocks of L steps (SURVEY §7 hard part 1).  Exact in real arithmetic.
//
// Within a block starting from w0 = w_{t0}, with rows r_l (l = 1..L) of the
// stacked [X~; B], c_l = coef_{i_l} * inv_nq_{i_l}, G = R R^T, e = R mu,
// b = R wbar (the epoch snapshot), a = R w0:
//   r_l . w_{t0+l-1} = a_l - eta sum_{l'<l} G_{ll'} delta_{l'} - eta (l-1) e_l
//   delta_l = c_l (r_l . w_{t0+l-1} - b_l)        (labels cancel, svrg.cpp:142-150)
//   => (I + eta C G_strict) delta = C (a - p),  p_l = eta (l-1) e_l + b_l
//   => delta = M (a - p),  M = (I + eta C G_strict)^{-1} C
//   w_{t0+L} = w0 - eta R^T delta - eta L mu
//   sum_l w_{t0+l} = L w0 - eta R^T ((L-l+1) delta_l) - eta mu L(L+1)/2.
// M and p depend only on the (pre-drawn) indices, mu and wbar, so the PREP
// kernel computes them for every block on all SMs; the CHAIN kernel (one
// thread-block cluster, each CTA owning a column slice) only does the
// dependent part per block.
//
// Look-ahead: with X_b = R_b R_{b-1}^T and e_b = R_b mu (also from PREP),
//   a_b = R_b w_b = R_b w_{b-1} - eta X_b delta_{b-1} - eta L e_b,
// so the partial dots a~_b = R_b w_{b-1} are computed (and their cluster
// reduction started) while block b-1 is still being resolved; the exchange
// latency leaves the dependent chain.  PREP folds eta L e_b into
// p'_b = p_b + eta L e_b for every block but the first of a launch, whose a_0 is
// computed directly.
//
// Row staging (v2): PREP, which reads every sampled row anyway, also writes the
// block's rows widened to fp64 into a PACKED buffer laid out per CTA slice,
// pk[block][cta][l][SW], so each chain CTA receives its L x SW slice of a block
// with ONE bulk copy (v1 issued one bulk copy per row slice from two producer
// warps plus two fp32 -> fp64 widener warps).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "svrg.cuh"
#include "fullgrad.cuh"
#include "gemm.cuh"

namespace skr {
namespace cg = cooperative_groups;

struct SstepRows {
  const void* Xt;      // data components (dtype T), row stride ld
  const double* B;     // regulariser components (fp64), row stride ld
  int64_t ld, d, n;    // n = number of data components
};

template <class T>
__device__ __forceinline__ double row_elem(const SstepRows& R, int64_t i, int64_t j) {
  return i < R.n ? (double)static_cast<const T*>(R.Xt)[i * R.ld + j] : R.B[(i - R.n) * R.ld + j];
}

// Packed-row geometry of the chain: CS CTAs, SW columns each (CS * SW >= ld).
struct PackGeom {
  int cs, sw;
};
// Element (row l, column j) of a CTA's L x SW slice sits at l * SW + pk_swz(j, l).
// The XOR swizzle makes both chain access patterns conflict-free: the dots
// (lanes = rows, one column at a time) and the update (lanes = columns, one row
// at a time); 8-byte accesses are served per half-warp, so 16 distinct bank
// pairs suffice.
__host__ __device__ __forceinline__ int pk_swz(int j, int l) { return j ^ (l & 15); }

// ---------------------------------------------------------------------------
// PREP: one CTA (256 threads, 8 warps) per block of L (16 or 32) steps.  One
// FP64 tensor-core (DMMA m8n8k4) product of the block's rows against the staged
// rows [R_b; R_{b-1}; mu; wbar] gives G = R_b R_b^T, X = R_b R_{b-1}^T
// (look-ahead), e = R_b mu and b = R_b wbar in one pass over the rows (column
// chunks of 32, register-prefetched one chunk ahead); the same pass writes the
// block's rows (fp64) to the packed buffer.  Then M = (I + eta C G_strict)^{-1} C
// by forward substitution.  Outputs: Mout[b] (L x L, stored TRANSPOSED:
// Mout[b][j*L + i] = M[i][j]), pout[b] (L), Xout[b] (transposed, blocks > 0 of
// the launch), pk.  Padded steps (beyond `steps`) get c_l = 0, so delta_l = 0
// there, and zero rows.
template <class T, int L>
__global__ void __launch_bounds__(256)
sstep_prep_kernel(SstepRows R, const int64_t* __restrict__ idx, int64_t steps, const double* __restrict__ inv_nq,
                  double data_coef, double reg_coef, const double* __restrict__ mu,
                  const double* __restrict__ wbar, double eta, double* __restrict__ Mout,
                  double* __restrict__ pout, double* __restrict__ Xout, double* __restrict__ pk, PackGeom pg) {
  static_assert(L == 16 || L == 32, "L = 16 or 32");
  constexpr int KC = 32, SP = KC + 4;         // staged columns per chunk, padded row stride (conflict-free frags)
  constexpr int NR = 2 * L + 8;               // staged rows: block b, block b-1, mu, wbar, zero pad
  constexpr int NTN = NR / 8;                 // n-tiles
  constexpr int MT = L / 8;                   // m-tiles
  constexpr int STEP = 8 / MT;                // warps per m-tile
  constexpr int NJ = (NTN + STEP - 1) / STEP; // n-tiles per warp
  constexpr int PER = NR * KC / 256;          // staged elements per thread per chunk
  static_assert(NR * KC % 256 == 0, "staging split");
  constexpr int RS = NR + 1;                  // result row stride
  extern __shared__ double dyn[];
  double* st = dyn;                           // [NR][SP] staging, then [L][RS] results
  double (*Xs)[L + 1] = reinterpret_cast<double (*)[L + 1]>(dyn + NR * SP);  // column j of T^{-1}
  __shared__ double cvec[L];
  __shared__ int64_t ridx[2 * L];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // grid-strided over the chunk's blocks: a capped grid (skr_ctx_set_prep_cap) leaves
  // SMs to concurrent chains (eta-grid lanes)
  const int64_t nblk = (steps + L - 1) / L;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t t0 = (int64_t)blk * L;
    const bool look = blk > 0;  // the previous block of this launch exists (and is full)
    if (tid < L) {
      const int64_t t = t0 + tid;
      const int64_t i = t < steps ? idx[t] : -1;
      ridx[tid] = i;
      ridx[L + tid] = look ? idx[t0 - L + tid] : -1;
      cvec[tid] = i < 0 ? 0.0 : (i < R.n ? data_coef : reg_coef) * inv_nq[i];
    }
    __syncthreads();
    auto fetch = [&](int64_t c0, double (&v)[PER]) {
  #pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int e = tid + q * 256, r = e / KC;
        const int64_t col = c0 + e % KC;
        double x = 0.0;
        if (col < R.d) {
          if (r < 2 * L) {
            const int64_t i = ridx[r];
            if (i >= 0) x = row_elem<T>(R, i, col);
          } else if (r == 2 * L) {
            x = mu[col];
          } else if (r == 2 * L + 1) {
            x = wbar[col];
          }
        }
        v[q] = x;
      }
    };
    const int mt = warp % MT, nb = warp / MT;  // m-tile; n-tiles nb, nb + STEP, ...
    double acc[NJ][2] = {};
    double v[PER];
    fetch(0, v);
    double* pkb = pk + (size_t)blk * pg.cs * L * pg.sw;
    for (int64_t c0 = 0; c0 < R.d; c0 += KC) {
      __syncthreads();
  #pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int e = tid + q * 256, r = e / KC;
        st[r * SP + e % KC] = v[q];
        const int64_t col = c0 + e % KC;
        if (r < L && col < R.d)  // the block's rows, packed per chain-CTA slice (swizzled, see pk_swz)
          pkb[((col / pg.sw) * L + r) * pg.sw + pk_swz((int)(col % pg.sw), r)] = v[q];
      }
      __syncthreads();
      if (c0 + KC < R.d) fetch(c0 + KC, v);  // next chunk in flight during the products
  #pragma unroll
      for (int k4 = 0; k4 < KC; k4 += 4) {
        const double a = st[(8 * mt + (lane >> 2)) * SP + k4 + (lane & 3)];
  #pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int nt = nb + STEP * j;
          if (nt < NTN) dmma_884(acc[j][0], acc[j][1], a, st[(8 * nt + (lane >> 2)) * SP + k4 + (lane & 3)]);
        }
      }
    }
    __syncthreads();
    double* res = st;  // res[i*RS + n]: n < L: G, L..2L-1: X, 2L: e, 2L+1: b
  #pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int nt = nb + STEP * j;
      if (nt < NTN) {
        const int i = 8 * mt + (lane >> 2), n = 8 * nt + 2 * (lane & 3);
        res[i * RS + n] = acc[j][0];
        res[i * RS + n + 1] = acc[j][1];
      }
    }
    __syncthreads();
    if (look) {  // X = R_b R_{b-1}^T stored transposed: Xt[j*L + i] = X[i][j]
      double* Xb = Xout + (int64_t)blk * L * L;
      for (int e = tid; e < L * L; e += blockDim.x) Xb[e] = res[(e % L) * RS + L + e / L];
    }
    // T = I + eta C G_strict (unit lower).  Column j of T^{-1} by forward
    // substitution (thread j), then M = T^{-1} C  (M[i][j] = Tinv[i][j] c_j).
    double* Mb = Mout + (int64_t)blk * L * L;
    if (tid < L) {
      const int j = tid;
      for (int i = 0; i < L; ++i) Xs[i][j] = i == j ? 1.0 : 0.0;
      for (int i = j + 1; i < L; ++i) {
        double s = 0.0;
        for (int k2 = j; k2 < i; ++k2) s = fma(res[i * RS + k2], Xs[k2][j], s);
        Xs[i][j] = -eta * cvec[i] * s;
      }
      // p_j = eta (j-1) e_j + b_j (1-based), + eta L e_j when a_b is formed by look-ahead
      pout[(int64_t)blk * L + j] = eta * (double)(look ? j + L : j) * res[j * RS + 2 * L] + res[j * RS + 2 * L + 1];
    }
    __syncthreads();
    for (int e = tid; e < L * L; e += blockDim.x) {  // stored transposed: Mt[j][i] = M[i][j]
      const int j = e / L, i = e % L;
      Mb[e] = Xs[i][j] * cvec[j];
    }
    __syncthreads();  // shared staging / results are reused by the next block
  }
}

template <int L>
constexpr size_t sstep_prep_smem() {
  return sizeof(double) * ((2 * L + 8) * (32 + 4) + L * (L + 1));
}

// ---------------------------------------------------------------------------
// CHAIN (v3): one cluster of CS CTAs; CTA r owns columns [r*SW, r*SW + SW).
// Roles per CTA (warps): NDW dot warps | NUW = SW/32 update warps | one delta
// warp | one producer warp.
//  * producer (lane 0): per block, ONE bulk copy of the block's packed L x SW
//    slice into an NB-deep ring (full/empty mbarriers), and M_b^T, X_b^T, p'_b
//    into a 2-deep ring;
//  * dot warps, iteration b: the look-ahead partials a~_{b+1} = R_{b+1} w_b over
//    the slice, lanes = rows (no cross-lane reduction), dot warp k covering
//    columns [k*SW/NDW, ...) — combined in shared memory when NDW = 2 — then
//    every row total goes to every rank of the cluster by st.async (8-byte
//    remote stores that complete_tx the receiver's part[(b+1) % 4] mbarrier);
//    w_b comes from the update warps (wready[b & 1]);
//  * update warps, iteration b: thread t owns column t (w_t and the running sum
//    S_t in registers): wait delta_b, the two rank-L updates with the block's
//    rows, w_{b+1} to the shared slice buffer of parity b+1 (wready), rows slot
//    released (empty);
//  * delta warp, block b: X term (X_b delta_{b-1}) while the partials travel,
//    wait part[b % 4] (acquire, cluster scope), z = sum of the CS partials in
//    rank order - eta X term - p'_b, delta_b = M_b z, then re-arm part[b % 4]
//    for block b+4.
// The dependent cycle spans two blocks: update(b-1) -> dots(b+1) -> exchange ->
// delta_{b+1} -> update(b+1), with the dots and the update of consecutive
// blocks running concurrently on different warps.
// Exchange ordering: st.async's complete_tx is the only publication: a phase of
// part[s] completes when its receiver has armed it (arrive.expect_tx of
// CS*L*8 bytes) AND every byte of the phase has landed, so a delta warp that
// observes completion reads complete partials.  Slot reuse needs no
// back-pressure: a rank pushes block b+4 into slot (b % 4) only after its
// dots(b+4), which need w_{b+3}, hence delta_{b+2}, hence THIS rank's partials
// of block b+2, which need this rank's w_{b+1}, i.e. its update(b), which
// follows its delta warp's read of slot b % 4 and the re-arming.
// Shared w buffers: dots(b+1) read buffer b & 1 (w_b); update(b+1) rewrites it
// only after delta_{b+1}, which needs this CTA's own partials of block b+1.
// w and the running sum persist in global state[0..ld) / [ld..2 ld) between
// launches (one launch per chunk of blocks).
struct ChainArgs {
  const double* pk;     // this chunk's packed rows [nblk][CS][L][SW] (swizzled)
  int64_t steps;        // steps in this chunk
  const double* M;      // nblk x L x L (transposed)
  const double* p;      // nblk x L  (p'_b: look-ahead correction folded in for b >= 1)
  const double* X;      // nblk x L x L (transposed): R_b R_{b-1}^T, b >= 1
  const double* mu;     // ld
  int64_t ld;
  double eta;
  double* state;        // [0, ld) w ; [ld, 2 ld) sum
  unsigned long long* prof;  // optional: per-phase cycle totals of CTA 0 (debug)
};

template <int SW, int L>
struct ChainCfg {
  static constexpr int NUW = SW / 32;                   // update warps (one column per thread)
  static constexpr int NDW = SW * L / 1024;             // dot warps: 32 columns per dot lane
  static constexpr int NT = 32 * (NDW + NUW) + 64;      // + delta warp + producer warp
  static constexpr int NB = SW * L * 8 <= 16384 ? 4 : SW * L * 8 <= 32768 ? 3 : 2;  // row ring depth (smem budget)
  static constexpr int NMX = 2;                         // M/X/p ring depth
  static constexpr int MXW = 2 * L * L + L;             // doubles per M/X/p slot
  static constexpr int NPS = 4;                         // partials slots (see the ordering argument)
  static constexpr size_t smem() {
    return sizeof(double) * ((size_t)NB * L * SW + (size_t)NMX * MXW + (size_t)NPS * 16 * L + 4 * L + L +
                             2 * NDW * L + 2 * SW) +
           sizeof(uint64_t) * (2 * NB + 2 * NMX + NPS + 2 + 2) + 128;
  }
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
// 8-byte asynchronous store to the cluster shared address `rdst`, completing 8
// bytes on the mbarrier at cluster shared address `rbar` (same CTA as rdst)
__device__ __forceinline__ void st_async_f64(uint32_t rdst, uint32_t rbar, double v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rdst),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}

// debug event trace (SKR_DEBUG_CHAIN): clock64 of CTA 0 per event for blocks
// [kTraceB0, kTraceB0 + kTraceN) of the first launch: prof[16 + 8 * k + e]
constexpr int kTraceB0 = 200, kTraceN = 8;
__device__ __forceinline__ void chain_trace(unsigned long long* prof, int cr, int64_t b, int e) {
  if (prof && cr == 0 && b >= kTraceB0 && b < kTraceB0 + kTraceN && prof[15] == 0)
    prof[16 + 8 * (b - kTraceB0) + e] = clock64();
}

template <int SW, int L>
__global__ void __launch_bounds__(ChainCfg<SW, L>::NT, 1) sstep_chain_kernel(ChainArgs a) {
  using Cf = ChainCfg<SW, L>;
  constexpr int NUW = Cf::NUW, NDW = Cf::NDW, NB = Cf::NB, NMX = Cf::NMX, MXW = Cf::MXW, NPS = Cf::NPS;
  constexpr int WU0 = NDW, WDL = NDW + NUW, WPR = NDW + NUW + 1;  // first update warp, delta warp, producer
  static_assert(L == 16 || L == 32, "lanes = rows in the dots");
  static_assert(SW >= 32 && SW % 32 == 0, "slice width");
  extern __shared__ __align__(128) unsigned char sm[];
  double* rows = reinterpret_cast<double*>(sm);                 // [NB][L][SW] (swizzled)
  double* mx = rows + (size_t)NB * L * SW;                      // [NMX][MXW]: M_b^T, X_b^T, p'_b
  double* apub = mx + NMX * MXW;                                // [NPS][16][L] partials by sender rank
  double* dl = apub + NPS * 16 * L;                             // [2][L] delta_b by parity
  double* d2 = dl + 2 * L;                                      // [2][L] (Lb - l) delta_b by parity
  double* zbuf = d2 + 2 * L;                                    // [L]
  double* dpart = zbuf + L;                                     // [2][NDW][L] dot warps' partials by parity
  double* wsm = dpart + 2 * NDW * L;                            // [2][SW] w slice by block parity
  uint64_t* full = reinterpret_cast<uint64_t*>(wsm + 2 * SW);   // [NB]
  uint64_t* empty = full + NB;                                  // [NB]
  uint64_t* mx_full = empty + NB;                               // [NMX]
  uint64_t* mx_empty = mx_full + NMX;                           // [NMX]
  uint64_t* part = mx_empty + NMX;                              // [NPS] partials (complete_tx)
  uint64_t* dready = part + NPS;                                // [2] delta_b published (local)
  uint64_t* wready = dready + 2;                                // [2] w_b written, by parity

  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t slice0 = (int64_t)cr * SW;
  const int64_t nblk = (a.steps + L - 1) / L;
  const uint32_t part_bytes = (uint32_t)(CS * L * 8);
  if (tid == 0) {
    for (int q = 0; q < NB; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NUW);
    }
    for (int q = 0; q < NMX; ++q) {
      mbar_init(&mx_full[q], 1);
      mbar_init(&mx_empty[q], 1);
    }
    for (int q = 0; q < NPS; ++q) mbar_init(&part[q], 1);  // the receiver's own arming arrive
    mbar_init(&dready[0], 1);
    mbar_init(&dready[1], 1);
    mbar_init(&wready[0], NUW);
    mbar_init(&wready[1], NUW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // arm the first NPS phases; bytes that land earlier count negative until then
    for (int q = 0; q < NPS && q < nblk; ++q) mbar_expect_tx(&part[q], part_bytes);
  }
  // w_0 in both parity buffers (dots(0) reads buffer 1, dots(1) buffer 0)
  for (int t = tid; t < SW; t += blockDim.x) {
    const int64_t col = slice0 + t;
    const double w0 = col < a.ld ? a.state[col] : 0.0;
    wsm[t] = w0;
    wsm[SW + t] = w0;
  }
  cluster.sync();  // every CTA's barriers exist before any remote complete_tx; w_0 visible

  if (warp == WPR) {
    // ---------------- producer: packed rows and M/X/p by bulk copy ----------------
    if (lane == 0) {
      const uint32_t slice_bytes = (uint32_t)(L * SW * 8);
      for (int64_t b = 0; b < nblk; ++b) {
        const int s = (int)(b % NB);
        if (b >= NB) mbar_wait(&empty[s], (uint32_t)(((b / NB) - 1) & 1));
        mbar_expect_tx(&full[s], slice_bytes);
        bulk_g2s(rows + (size_t)s * L * SW, a.pk + ((size_t)b * CS + cr) * L * SW, slice_bytes, &full[s]);
        const int ms = (int)(b % NMX);
        if (b >= NMX) mbar_wait(&mx_empty[ms], (uint32_t)(((b / NMX) - 1) & 1));
        double* dst = mx + ms * MXW;
        mbar_expect_tx(&mx_full[ms], (uint32_t)(MXW * 8));
        bulk_g2s(dst, a.M + b * L * L, (uint32_t)(L * L * 8), &mx_full[ms]);
        bulk_g2s(dst + L * L, a.X + b * L * L, (uint32_t)(L * L * 8), &mx_full[ms]);  // b = 0: unused
        bulk_g2s(dst + 2 * L * L, a.p + b * L, (uint32_t)(L * 8), &mx_full[ms]);
      }
    }
  } else if (warp == WDL) {
    // ---------------- delta warp: lane i resolves row i of each block ----------------
    const int i = lane;
    const bool prof = a.prof && cr == 0 && lane == 0;
    unsigned long long t_wait = 0;
    for (int64_t b = 0; b < nblk; ++b) {
      const int Lb = (int)min((int64_t)L, a.steps - b * L);
      const int ms = (int)(b % NMX);
      const double* Ms = mx + ms * MXW;
      const double* Xs = Ms + L * L;
      const double* ps = Ms + 2 * L * L;
      mbar_wait(&mx_full[ms], (uint32_t)((b / NMX) & 1));
      // off the critical path (delta_{b-1} is known, the partials of b are in
      // flight): c_i = eta (X_b delta_{b-1})_i + p'_i and row i of M_b in registers
      double ci = 0.0, mrow[L];
      if (i < L) {
        double xt = 0.0;
        if (b > 0) {
          const double* dp = dl + ((b - 1) & 1) * L;
          double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
#pragma unroll
          for (int k = 0; k < L; k += 4) {
            const double4 dq = *reinterpret_cast<const double4*>(dp + k);
            x0 = fma(Xs[k * L + i], dq.x, x0);
            x1 = fma(Xs[(k + 1) * L + i], dq.y, x1);
            x2 = fma(Xs[(k + 2) * L + i], dq.z, x2);
            x3 = fma(Xs[(k + 3) * L + i], dq.w, x3);
          }
          xt = (x0 + x1) + (x2 + x3);
        }
        ci = a.eta * xt + ps[i];
#pragma unroll
        for (int k = 0; k < L; ++k) mrow[k] = Ms[k * L + i];
      }
      const int ps4 = (int)(b % NPS);
      const unsigned long long w0 = prof ? clock64() : 0;
      mbar_wait_cluster(&part[ps4], (uint32_t)((b / NPS) & 1));
      if (prof) t_wait += clock64() - w0;
      if (lane == 0) chain_trace(a.prof, cr, b, 2);
      if (i < L) {
        // the CS partials of row i, summed by a fixed tree (deterministic)
        const double* ap = apub + (size_t)ps4 * 16 * L + i;
        double pq[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) pq[q] = q < CS ? ap[q * L] : 0.0;
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
          for (int q = 0; q < h; ++q) pq[q] += pq[q + h];
        zbuf[i] = pq[0] - ci;
      }
      __syncwarp();
      if (i < L) {
        double d0 = 0.0, d1 = 0.0, d2v = 0.0, d3 = 0.0;
#pragma unroll
        for (int k = 0; k < L; k += 4) {
          const double4 zq = *reinterpret_cast<const double4*>(zbuf + k);
          d0 = fma(mrow[k], zq.x, d0);
          d1 = fma(mrow[k + 1], zq.y, d1);
          d2v = fma(mrow[k + 2], zq.z, d2v);
          d3 = fma(mrow[k + 3], zq.w, d3);
        }
        const double dv = (d0 + d1) + (d2v + d3);
        dl[(b & 1) * L + i] = dv;
        d2[(b & 1) * L + i] = (double)(Lb - i) * dv;  // (Lb - l + 1) weight, 1-based l
      }
      __syncwarp();
      if (lane == 0) {
        chain_trace(a.prof, cr, b, 3);
        mbar_arrive_local(&dready[b & 1]);  // delta_b visible to the update warps (release.cta)
        mbar_arrive_local(&mx_empty[ms]);   // M/X slot consumed
        if (b + NPS < nblk) mbar_expect_tx(&part[ps4], part_bytes);  // slot read: arm block b + NPS
      }
    }
    if (prof) atomicAdd(a.prof + 4, t_wait);
  } else if (warp < NDW) {
    // ---------------- dot warps: lanes = rows ----------------
    // L = 32: lane l = row l; L = 16: lanes l and l+16 take row l, each half of
    // the warp's columns.  Every dot lane covers 32 consecutive (logical) columns
    // starting at c0; with the swizzle, column c0 + 16m + jj of row l sits at
    // c0 + 16m + (jj ^ (l & 15)): 16 per-lane offsets, the rest immediates.
    constexpr int HALVES = 32 / L;
    constexpr int NCOL = 32;
    static_assert(NDW * HALVES * NCOL == SW, "dot warps cover the slice");
    const int l = lane % L;
    const int c0 = (warp * HALVES + lane / L) * NCOL;
    int off[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) off[jj] = jj ^ (l & 15);
    // remote addresses of this lane's partial in every rank (slot 0), and of part[0]
    uint32_t rdst[16], rbar[16];
    const uint32_t ldst = smem_u32(apub + (size_t)cr * L + l), lbar = smem_u32(&part[0]);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      rdst[q] = q < CS ? mapa_u32(ldst, (uint32_t)q) : 0u;
      rbar[q] = q < CS ? mapa_u32(lbar, (uint32_t)q) : 0u;
    }
    const bool prof = a.prof && cr == 0 && tid == 0;
    unsigned long long tw = 0, td = 0;
    for (int64_t bb = 0; bb < nblk; ++bb) {  // dots(bb) against w_{bb-1} (w_0 for bb = 0)
      const int s = (int)(bb % NB);
      const unsigned long long q0 = prof ? clock64() : 0;
      if (bb >= 2) mbar_wait(&wready[(bb - 1) & 1], (uint32_t)(((bb - 2) >> 1) & 1));  // w_{bb-1} written
      mbar_wait(&full[s], (uint32_t)((bb / NB) & 1));
      const unsigned long long q1 = prof ? clock64() : 0;
      if (warp == 0 && lane == 0) chain_trace(a.prof, cr, bb, 0);
      const double* x = rows + (size_t)s * L * SW + (size_t)l * SW + c0;
      const double* wb = wsm + (size_t)((bb + 1) & 1) * SW + c0;  // w_{bb-1}: buffer of parity bb - 1
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int m = 0; m < NCOL / 16; ++m) {
#pragma unroll
        for (int jj = 0; jj < 16; jj += 2) {
          const double2 wq = *reinterpret_cast<const double2*>(wb + 16 * m + jj);
          acc[(jj >> 1) & 3] = fma(x[16 * m + off[jj]], wq.x, acc[(jj >> 1) & 3]);
          acc[((jj >> 1) + 1) & 3] = fma(x[16 * m + off[jj + 1]], wq.y, acc[((jj >> 1) + 1) & 3]);
        }
      }
      double v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      if constexpr (HALVES == 2) v += __shfl_xor_sync(0xffffffffu, v, 16);
      if constexpr (NDW > 1) {
        // the dot warps' partials of the same rows meet in shared memory (by parity)
        double* dp = dpart + (size_t)(bb & 1) * NDW * L;
        if (lane < L) dp[warp * L + l] = v;
        named_bar(2, 32 * NDW);
        if (warp == 0 && lane < L) {
          v = dp[l];
#pragma unroll
          for (int k = 1; k < NDW; ++k) v += dp[k * L + l];
        }
      }
      if (warp == 0 && lane < L) {
        const uint32_t off_s = (uint32_t)((bb % NPS) * 16 * L * 8), boff = (uint32_t)((bb % NPS) * 8);
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (q < CS) st_async_f64(rdst[q] + off_s, rbar[q] + boff, v);
        if (lane == 0) chain_trace(a.prof, cr, bb, 1);
      }
      if (prof) {
        const unsigned long long q2 = clock64();
        tw += q1 - q0;
        td += q2 - q1;
      }
    }
    if (prof) {
      atomicAdd(a.prof + 0, td);
      atomicAdd(a.prof + 5, tw);
    }
  } else {
    // ---------------- update warps: thread t owns column slice0 + t ----------------
    const int t = tid - 32 * WU0;
    const int64_t col = slice0 + t;
    const bool act = col < a.ld;
    double w = act ? a.state[col] : 0.0;
    double S = act ? a.state[a.ld + col] : 0.0;
    const double muc = act ? a.mu[col] : 0.0;
    int off[16];  // column t of row l sits at l * SW + off[l & 15]
#pragma unroll
    for (int k = 0; k < 16; ++k) off[k] = pk_swz(t, k);
    const bool prof = a.prof && cr == 0 && t == 0;
    unsigned long long tp[3] = {};
    for (int64_t b = 0; b < nblk; ++b) {
      const int s = (int)(b % NB);
      const int Lb = (int)min((int64_t)L, a.steps - b * L);
      const unsigned long long c0 = prof ? clock64() : 0;
      mbar_wait(&dready[b & 1], (uint32_t)((b >> 1) & 1));
      const unsigned long long c1 = prof ? clock64() : 0;
      if (t == 0) chain_trace(a.prof, cr, b, 4);
      // w <- w0 - eta R^T delta - eta Lb mu ; S += Lb w0 - eta R^T((Lb-l+1) delta) - eta mu Lb(Lb+1)/2
      const double* rb = rows + (size_t)s * L * SW;
      const double* dd = dl + (b & 1) * L;
      const double* ee = d2 + (b & 1) * L;
      double u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0, v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
      if (Lb == L) {
#pragma unroll
        for (int l = 0; l < L; l += 4) {
          const double x0 = rb[l * SW + off[l & 15]], x1 = rb[(l + 1) * SW + off[(l + 1) & 15]];
          const double x2 = rb[(l + 2) * SW + off[(l + 2) & 15]], x3 = rb[(l + 3) * SW + off[(l + 3) & 15]];
          const double4 dq = *reinterpret_cast<const double4*>(dd + l);
          const double4 eq = *reinterpret_cast<const double4*>(ee + l);
          u0 = fma(dq.x, x0, u0); u1 = fma(dq.y, x1, u1); u2 = fma(dq.z, x2, u2); u3 = fma(dq.w, x3, u3);
          v0 = fma(eq.x, x0, v0); v1 = fma(eq.y, x1, v1); v2 = fma(eq.z, x2, v2); v3 = fma(eq.w, x3, v3);
        }
      } else {
        for (int l = 0; l < Lb; ++l) {
          const double x = rb[l * SW + pk_swz(t, l)];
          u0 = fma(dd[l], x, u0);
          v0 = fma(ee[l], x, v0);
        }
      }
      const double u = (u0 + u1) + (u2 + u3), vv = (v0 + v1) + (v2 + v3);
      const double w0 = w;
      S += (double)Lb * w0 - a.eta * vv - a.eta * muc * (0.5 * (double)Lb * (double)(Lb + 1));
      w = w0 - a.eta * u - a.eta * (double)Lb * muc;
      wsm[((b + 1) & 1) * SW + t] = w;  // w_{b+1}
      __syncwarp();
      if (t == 0) chain_trace(a.prof, cr, b, 5);
      if (lane == 0) {
        mbar_arrive_local(&wready[(b + 1) & 1]);  // this warp's columns of w_{b+1} written (release.cta)
        mbar_arrive_local(&empty[s]);             // this warp is done with rows[s]
      }
      if (prof) {
        const unsigned long long c2 = clock64();
        tp[0] += c1 - c0;
        tp[1] += c2 - c1;
        tp[2] += 1;
      }
    }
    if (prof) {
      atomicAdd(a.prof + 1, tp[0]);
      atomicAdd(a.prof + 2, tp[1]);
      atomicAdd(a.prof + 3, tp[2]);
    }
    if (act) {
      a.state[col] = w;
      a.state[a.ld + col] = S;
    }
  }
  cluster.sync();  // no CTA exits while others may still write its smem / signal its barriers
}

// w_avg = S / m ; zero padding.
__global__ void sstep_finish_kernel(const double* __restrict__ state, int64_t ld, int64_t d, double m,
                                    double* __restrict__ w_avg) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < ld) w_avg[j] = j < d ? state[ld + j] * (1.0 / m) : 0.0;
}

// state = (snapshot, 0)
__global__ void sstep_init_kernel(const double* __restrict__ snap, int64_t ld, double* __restrict__ state) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < ld) {
    state[j] = snap[j];
    state[ld + j] = 0.0;
  }
}

}  // namespace skr
