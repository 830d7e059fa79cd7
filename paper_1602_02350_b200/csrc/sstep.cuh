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
// File map:
//   PACK + GRAM   the per-block quantities for a chunk of blocks, on all SMs, one chunk ahead of
//                 the chain: PACK gathers the sampled rows once (widened to fp64) into the packed
//                 buffer pk[block][cta][l][SW]; GRAM forms R_b [R_b; R_{b-1}; (R_{b-2};) mu; wbar]^T
//                 on DMMA from the packed tiles and solves for M (and Y_q = eta M X_q, p'');
//   chain v7      look-ahead depth 3 (the default): see its header below;
//   chain v3      look-ahead depth 2 (SKR_CHAIN_V3=1, kept for A/B).
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
// PREP = PACK + GRAM (round 2).  Round 1's one-kernel PREP issued one dependent
// gather per 32-column chunk (64-128 global round trips per block, ~5 B/clk/SM in
// flight): 0.81 ms per 1024 blocks at c3, as long as the chain it is supposed to
// hide behind.  Now:
//  * PACK (all SMs, many independent 16-byte loads in flight): gathers every
//    sampled row ONCE, widens it to fp64 and writes it to the packed buffer
//    pk[block][chain CTA][l][SW] (the layout the chain's bulk copies want);
//  * GRAM: one CTA per block reads the packed tiles of blocks b, b-1 (, b-2)
//    back with bulk copies (an NSTG-stage ring over the CS column slices, no
//    register staging) and runs the DMMA products R_b [R_b; R_{b-1}; ..; mu;
//    wbar]^T from shared memory, then the small triangular solve and products.
// Fragment loads straight from the XOR-swizzled tiles are conflict-free when a
// k-step of the m8n8k4 product takes the four columns {c, c+4, c+8, c+12} of a
// 16-column group (any fixed order of the columns gives the same dot products).
template <class E>
__device__ __forceinline__ void pack_row(const E* __restrict__ src, int l, double* __restrict__ pkb, PackGeom pg,
                                         int L, int64_t d, int64_t ld, int lane) {
  constexpr int VE = 16 / (int)sizeof(E);  // elements per 16-byte load
  const int x = l & 15;
  constexpr int UN = 4;
  for (int64_t c0 = (int64_t)lane * VE; c0 < ld; c0 += 32 * VE * UN) {
    int4 raw[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int64_t c = c0 + (int64_t)u * 32 * VE;
      raw[u] = make_int4(0, 0, 0, 0);
      if (src && c < ld) raw[u] = __ldg(reinterpret_cast<const int4*>(src + c));
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int64_t c = c0 + (int64_t)u * 32 * VE;
      if (c >= ld) continue;
      double v[VE], o[VE];
      const E* e = reinterpret_cast<const E*>(&raw[u]);
#pragma unroll
      for (int q = 0; q < VE; ++q) v[q] = c + q < d ? (double)e[q] : 0.0;
#pragma unroll
      for (int q = 0; q < VE; ++q) o[q] = v[q ^ (x & (VE - 1))];  // o[q ^ m] = v[q]
      const int64_t slice = c / pg.sw;
      const int j0 = (int)(c % pg.sw) ^ (x & ~(VE - 1));
      double* dst = pkb + ((size_t)slice * L + l) * pg.sw + j0;
#pragma unroll
      for (int q = 0; q < VE; q += 2) *reinterpret_cast<double2*>(dst + q) = make_double2(o[q], o[q + 1]);
    }
  }
}

template <class T, int L>
__global__ void __launch_bounds__(256)
sstep_pack_kernel(SstepRows R, const int64_t* __restrict__ idx, int64_t steps, double* __restrict__ pk, PackGeom pg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nblk = (steps + L - 1) / L;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    double* pkb = pk + (size_t)blk * pg.cs * L * pg.sw;
    for (int l = warp; l < L; l += 8) {
      const int64_t t = blk * L + l;
      const int64_t i = t < steps ? idx[t] : -1;
      if (i >= 0 && i < R.n)
        pack_row<T>(static_cast<const T*>(R.Xt) + i * R.ld, l, pkb, pg, L, R.d, R.ld, lane);
      else  // regulariser component, or a padded step (zero row)
        pack_row<double>(i < 0 ? nullptr : R.B + (i - R.n) * R.ld, l, pkb, pg, L, R.d, R.ld, lane);
    }
  }
}

// Output layout of DEPTH = 3 (chain v7), per block MX7<L>::W doubles:
//   [M | Y1 | Y2] each L x L "lane-major pairs": A[i][k] at (k >> 1) * 2L + 2i + (k & 1), so lane i
//   reads its row with 16-byte loads, conflict-free; then p'' (L).
template <int L>
struct MX7 {
  static constexpr int W = 3 * L * L + L;
};
__host__ __device__ __forceinline__ int lm_pair(int L, int i, int k) { return (k >> 1) * 2 * L + 2 * i + (k & 1); }

template <int L, int DEPTH>
struct GramCfg {
  static constexpr int NRB = DEPTH * L;          // staged block rows
  static constexpr int NTN = NRB / 8 + 1;        // n-tiles: block rows, then [mu; wbar; 0...]
  static constexpr int MT = L / 8;               // m-tiles
  static constexpr int STEP = 8 / MT;            // warps per m-tile: they split the k-steps, each takes every n-tile
  static constexpr int NJ = NTN;
  static constexpr int RS = NRB + 3;             // result row stride (odd: conflict-free column reads)
  static constexpr size_t stage_bytes(int sw) { return sizeof(double) * ((size_t)NRB * sw + 2 * sw); }
  static constexpr size_t epi_bytes() { return sizeof(double) * ((size_t)L * RS + 3 * (size_t)L * (L + 1) + L); }
};

// idx: this chunk's step indices; pk: this chunk's packed rows; outputs as the chain of the same DEPTH reads
// them (DEPTH 2: Mout/pout/Xout as PREP v1; DEPTH 3: MXout, MX7 layout).
template <int L, int DEPTH>
__global__ void __launch_bounds__(256, 1)
sstep_gram_kernel(const double* __restrict__ pk, PackGeom pg, int nstg, const int64_t* __restrict__ idx, int64_t steps,
                  int64_t n_data, const double* __restrict__ inv_nq, double data_coef, double reg_coef,
                  const double* __restrict__ mu, const double* __restrict__ wbar, int64_t ld, double eta,
                  double* __restrict__ Mout, double* __restrict__ pout, double* __restrict__ Xout,
                  double* __restrict__ MXout) {
  using G = GramCfg<L, DEPTH>;
  constexpr int NRB = G::NRB, NTN = G::NTN, MT = G::MT, STEP = G::STEP, NJ = G::NJ, RS = G::RS;
  static_assert(L == 16 || L == 32, "L = 16 or 32");
  static_assert(DEPTH == 2 || DEPTH == 3, "look-ahead depth");
  extern __shared__ __align__(128) unsigned char gsm[];
  __shared__ __align__(8) uint64_t full[4];
  __shared__ double cvec[L];
  const int SW = pg.sw, CS = pg.cs;
  const size_t stage_d = (size_t)NRB * SW + 2 * SW;  // doubles per stage
  double* stg = reinterpret_cast<double*>(gsm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mt = warp % MT, kpart = warp / MT;  // m-tile; this warp's share of the k-steps (k-step c of a 16-column group)
  const int64_t nblk = (steps + L - 1) / L;
  if (tid == 0) {
    for (int s = 0; s < 4; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t issued = 0, waited = 0;  // stage uses so far (ring position and phase parity)
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int nprev = (int)min((int64_t)(DEPTH - 1), blk);  // previous blocks of this launch that exist
    if (tid < L) {
      const int64_t t = blk * L + tid;
      const int64_t i = t < steps ? idx[t] : -1;
      cvec[tid] = i < 0 ? 0.0 : (i < n_data ? data_coef : reg_coef) * inv_nq[i];
    }
    auto issue = [&](int s) {  // slice s of blocks blk, blk-1, .. and of mu, wbar -> ring slot
      const int slot = (int)(issued % (uint32_t)nstg);
      double* dst = stg + (size_t)slot * stage_d;
      const uint32_t tile_bytes = (uint32_t)(L * SW * 8), vec_bytes = (uint32_t)(SW * 8);
      mbar_expect_tx(&full[slot], (uint32_t)(1 + nprev) * tile_bytes + 2 * vec_bytes);
      for (int q = 0; q <= nprev; ++q)
        bulk_g2s(dst + (size_t)q * L * SW, pk + ((size_t)(blk - q) * CS + s) * L * SW, tile_bytes, &full[slot]);
      bulk_g2s(dst + (size_t)NRB * SW, mu + (size_t)s * SW, vec_bytes, &full[slot]);
      bulk_g2s(dst + (size_t)NRB * SW + SW, wbar + (size_t)s * SW, vec_bytes, &full[slot]);
      ++issued;
    };
    if (tid == 0) {
      // the ring was last touched through the generic proxy (the previous block's results)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int s = 0; s < nstg - 1 && s < CS; ++s) issue(s);
    }
    double acc[NJ][2] = {};
    // per-lane fragment geometry: row r8 = lane >> 2 of an 8-row tile, k index t4 = lane & 3
    const int r8 = lane >> 2, t4 = lane & 3;
    const int la = 8 * mt + r8;  // A row (block b)
    // B operand of n-tile q: element (row, column j) at boff[q] + (j ^ bxor[q]); lanes with
    // bok[q] false feed zeros.  No branch inside the product loop: a conditional mma.sync
    // costs a WARPSYNC and serialises the tiles (the first version ran the FP64 pipe at a third
    // of this).  Tiles of blocks that are not in this launch (nprev < q) multiply stale but
    // finite-or-not data into accumulators the epilogue never reads.
    int boff[NJ], bxor[NJ];
    bool bok[NJ];
#pragma unroll
    for (int q = 0; q < NJ; ++q) {
      if (q < NTN - 1) {
        const int rr = 8 * q + r8;
        boff[q] = rr * SW;
        bxor[q] = (rr % L) & 15;
        bok[q] = true;
      } else {  // [mu; wbar; zero rows]
        boff[q] = NRB * SW + (r8 < 2 ? r8 : 0) * SW;
        bxor[q] = 0;
        bok[q] = r8 < 2;
      }
    }
    for (int s = 0; s < CS; ++s) {
      if (tid == 0 && s + nstg - 1 < CS) issue(s + nstg - 1);
      const int slot = (int)(waited % (uint32_t)nstg);
      mbar_wait(&full[slot], (waited / (uint32_t)nstg) & 1u);
      ++waited;
      const double* st = stg + (size_t)slot * stage_d;
      const double* arow = st + (size_t)la * SW;
      const int ax = la & 15;
      // the STEP warps of an m-tile take the k-steps c = kpart, kpart + STEP, .. of every 16-column
      // group and every n-tile (one A fragment per NTN products; no padding tile); their partial
      // accumulators are summed in warp order below
#pragma unroll 2
      for (int g16 = 0; g16 < SW; g16 += 16) {
#pragma unroll
        for (int cc = 0; cc < 4 / STEP; ++cc) {
          const int c = kpart + STEP * cc;
          const int j = g16 + c + 4 * t4;  // this lane's column of the k-step {c, c+4, c+8, c+12}
          const double a = arow[j ^ ax];
          double bv[NJ];
#pragma unroll
          for (int q = 0; q < NJ; ++q) {
            bv[q] = 0.0;
            if (bok[q]) bv[q] = st[boff[q] + (j ^ bxor[q])];
          }
#pragma unroll
          for (int q = 0; q < NJ; ++q) dmma_884(acc[q][0], acc[q][1], a, bv[q]);
        }
      }
      __syncthreads();  // the slot may be refilled
    }
    // ---- results: res[i * RS + n], n < L: G; L..2L: X1; (2L..3L: X2); NRB: e; NRB + 1: b ----
    double* res = stg;                                   // aliases ring slot 0.. (all stages consumed)
    double* Ti = res + (size_t)L * RS;                   // [L][L+1] T^{-1}, then M
    double* W1 = Ti + (size_t)L * (L + 1);               // [L][L+1] scratch (Y1)
    double* W2 = W1 + (size_t)L * (L + 1);               // [L][L+1] scratch (Y2)
    double* pv = W2 + (size_t)L * (L + 1);               // [L]
    for (int kp = 0; kp < STEP; ++kp) {  // fixed order: deterministic
      if (kpart == kp) {
#pragma unroll
        for (int q = 0; q < NJ; ++q) {
          const int i = 8 * mt + r8, n = 8 * q + 2 * t4;
          if (n < RS - 1) {
            if (kp == 0) {
              res[i * RS + n] = acc[q][0];
              res[i * RS + n + 1] = acc[q][1];
            } else {
              res[i * RS + n] += acc[q][0];
              res[i * RS + n + 1] += acc[q][1];
            }
          }
        }
      }
      __syncthreads();
    }
    // T = I + eta C G_strict (unit lower).  Column j of T^{-1} by forward substitution; a column
    // only depends on itself, so PARTS = 256 / L lanes of one warp share column j (each sums the
    // k2 = j + part (mod PARTS) terms of a row, xor-shuffle reduction) and no block barrier is
    // needed between rows (one thread per column took ~15 K cycles per block with 7 warps idle).
    {
      constexpr int PARTS = 256 / L;
      const int j = tid / PARTS, part = tid % PARTS;
      for (int i = part; i < L; i += PARTS) Ti[i * (L + 1) + j] = i == j ? 1.0 : 0.0;
      __syncwarp();
      const int jmin = (tid & ~31) / PARTS;  // lowest column of this warp
      for (int i = jmin + 1; i < L; ++i) {
        double sacc = 0.0;
        if (i > j)
          for (int k2 = j + part; k2 < i; k2 += PARTS) sacc = fma(res[i * RS + k2], Ti[k2 * (L + 1) + j], sacc);
#pragma unroll
        for (int o = PARTS / 2; o >= 1; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        if (i > j && part == 0) Ti[i * (L + 1) + j] = -eta * cvec[i] * sacc;
        __syncwarp();
      }
    }
    if (tid < L) {
      const int j = tid;
      // p_j = eta j e_j + b_j (0-based j), + eta L nprev e_j: the dots of this block were taken nprev blocks early
      pv[j] = eta * (double)(j + L * nprev) * res[j * RS + NRB] + res[j * RS + NRB + 1];
    }
    __syncthreads();
    for (int e = tid; e < L * L; e += 256) {  // M = T^{-1} C in place
      const int i = e / L, j = e % L;
      Ti[i * (L + 1) + j] *= cvec[j];
    }
    __syncthreads();
    if (DEPTH == 2) {
      double* Mb = Mout + (int64_t)blk * L * L;
      for (int e = tid; e < L * L; e += 256) Mb[e] = Ti[(e % L) * (L + 1) + e / L];  // transposed
      if (nprev >= 1) {
        double* Xb = Xout + (int64_t)blk * L * L;
        for (int e = tid; e < L * L; e += 256) Xb[e] = res[(e % L) * RS + L + e / L];
      }
      if (tid < L) pout[(int64_t)blk * L + tid] = pv[tid];
    } else {
      double* out = MXout + (int64_t)blk * MX7<L>::W;
      // Y_q = eta M X_q (zero when block b - q is not in this launch), p'' = M p
      for (int e = tid; e < 2 * L * L; e += 256) {
        const int q = e / (L * L), i = (e / L) % L, k = e % L;
        double y = 0.0;
        if (q < nprev) {
          const double* xq = res + (size_t)(q + 1) * L + k;
          for (int j = 0; j <= i; ++j) y = fma(Ti[i * (L + 1) + j], xq[j * RS], y);
          y *= eta;
        }
        out[(size_t)(q + 1) * L * L + lm_pair(L, i, k)] = y;
      }
      for (int e = tid; e < L * L; e += 256) out[lm_pair(L, e / L, e % L)] = Ti[(e / L) * (L + 1) + e % L];
      if (tid < L) {
        double y = 0.0;
        for (int j = 0; j <= tid; ++j) y = fma(Ti[tid * (L + 1) + j], pv[j], y);
        out[3 * L * L + tid] = y;
      }
    }
    __syncthreads();  // results alias the ring: done before the next block's copies land
  }
}

// mu and wbar zero-padded to the chain's CS * SW columns (GRAM bulk-copies whole slices)
__global__ void sstep_padvec_kernel(const double* __restrict__ mu, const double* __restrict__ wbar, int64_t d,
                                    int64_t width, double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < width) {
    out[j] = j < d ? mu[j] : 0.0;
    out[width + j] = j < d ? wbar[j] : 0.0;
  }
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
  static constexpr int NT = 32 * (NDW + NUW) + 96;      // + delta warp + producer warp + sender warp
  static constexpr int NB = SW * L * 8 <= 16384 ? 4 : SW * L * 8 <= 32768 ? 3 : 2;  // row ring depth (smem budget)
  static constexpr int NMX = 2;                         // M/X/p ring depth
  static constexpr int MXW = 2 * L * L + L;             // doubles per M/X/p slot
  static constexpr int NPS = 4;                         // partials slots (see the ordering argument)
  static constexpr size_t smem() {
    return sizeof(double) * ((size_t)NB * L * SW + (size_t)NMX * MXW + (size_t)NPS * 16 * L + 4 * L + L +
                             2 * NDW * L + 2 * SW) +
           sizeof(uint64_t) * (2 * NB + 2 * NMX + NPS + 2 + 2 + 2) + 128;
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
// Non-suspending waits for the hand-offs on the chain's dependent cycle (try_wait may park
// the warp; a parked warp resumes some hundred cycles after the phase completes).
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "SPIN_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 0x989680;\n"
      "@!P1 bra SPIN_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// one non-blocking test: issue it early and look at the answer after independent work (a
// phase check answers through the long scoreboard, some hundred cycles even when the phase is
// complete; the answer "complete" stays valid while the ring arguments exclude a second flip)
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_spin_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "SPINC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, 0x989680;\n"
      "@!P1 bra SPINC_%=;\n"
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

// 16-byte form: two doubles per store, one complete_tx of 16 bytes (the receiver's mbarrier
// serialises its complete_tx updates: half as many per block)
__device__ __forceinline__ void st_async_f64x2(uint32_t rdst, uint32_t rbar, double v0, double v1) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(rdst),
               "l"(__double_as_longlong(v0)), "l"(__double_as_longlong(v1)), "r"(rbar)
               : "memory");
}

// debug event trace (SKR_DEBUG_CHAIN): clock64 of CTA 0 per event for blocks
// [kTraceB0, kTraceB0 + kTraceN) of the first launch: prof[16 + 8 * k + e]
constexpr int kTraceB0 = 200, kTraceN = 8;
__device__ __forceinline__ void chain_trace(unsigned long long* prof, int cr, int64_t b, int e) {
  const unsigned long long t = clock64();
  if (prof && cr == 0 && b >= kTraceB0 && b < kTraceB0 + kTraceN) prof[16 + 8 * (b - kTraceB0) + e] = t;
}

// four more events per traced block: prof[80 + 4 * k + e]
__device__ __forceinline__ void chain_trace2(unsigned long long* prof, int cr, int64_t b, int e) {
  const unsigned long long t = clock64();
  if (prof && cr == 0 && b >= kTraceB0 && b < kTraceB0 + kTraceN) prof[80 + 4 * (b - kTraceB0) + e] = t;
}

template <int SW, int L>
__global__ void __launch_bounds__(ChainCfg<SW, L>::NT, 1) sstep_chain_kernel(ChainArgs a) {
  using Cf = ChainCfg<SW, L>;
  constexpr int NUW = Cf::NUW, NDW = Cf::NDW, NB = Cf::NB, NMX = Cf::NMX, MXW = Cf::MXW, NPS = Cf::NPS;
  constexpr int WU0 = NDW, WDL = NDW + NUW, WPR = NDW + NUW + 1, WSN = NDW + NUW + 2;  // update, delta, producer, sender
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
  uint64_t* dotdone = part + NPS;                               // [2] the dot warps' partials of a block are in dpart
  uint64_t* dready = dotdone + 2;                               // [2] delta_b published (local)
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
      mbar_init(&empty[q], NUW + NDW);  // update warps (column in registers) and dot warps (dots done)
    }
    for (int q = 0; q < NMX; ++q) {
      mbar_init(&mx_full[q], 1);
      mbar_init(&mx_empty[q], 1);
    }
    for (int q = 0; q < NPS; ++q) mbar_init(&part[q], 1);  // the receiver's own arming arrive
    mbar_init(&dotdone[0], NDW);
    mbar_init(&dotdone[1], NDW);
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
      mbar_spin_cluster(&part[ps4], (uint32_t)((b / NPS) & 1));
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
    const bool prof = a.prof && cr == 0 && tid == 0;
    unsigned long long tw = 0, td = 0;
    for (int64_t bb = 0; bb < nblk; ++bb) {  // dots(bb) against w_{bb-1} (w_0 for bb = 0)
      const int s = (int)(bb % NB);
      const unsigned long long q0 = prof ? clock64() : 0;
      if (bb >= 2) mbar_spin(&wready[(bb - 1) & 1], (uint32_t)(((bb - 2) >> 1) & 1));  // w_{bb-1} written
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
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&empty[s]);  // this warp's reads of rows[s] are done
      if constexpr (HALVES == 2) v += __shfl_xor_sync(0xffffffffu, v, 16);
      // hand the warp's row partials to the sender warp (by block parity): dots(bb + 2) needs
      // delta_bb, hence this rank's partials of block bb on every rank, so the sender has read
      // dpart[bb & 1] before it is rewritten
      if (lane < L) dpart[(size_t)(bb & 1) * NDW * L + warp * L + l] = v;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_local(&dotdone[bb & 1]);
        if (warp == 0) chain_trace(a.prof, cr, bb, 1);
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
  } else if (warp == WSN) {
    // ---------------- sender warp: lane l pushes row l's partial to every rank ----------------
    // (its own warp: the 16 L remote stores of a block keep their issuer ~1 K cycles in the
    // outbound queue, time the dot warps now spend on the next block)
    uint32_t rdst[16], rbar[16];
    const int l = lane % L;
    const uint32_t ldst = smem_u32(apub + (size_t)cr * L + l), lbar = smem_u32(&part[0]);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      rdst[q] = q < CS ? mapa_u32(ldst, (uint32_t)q) : 0u;
      rbar[q] = q < CS ? mapa_u32(lbar, (uint32_t)q) : 0u;
    }
    for (int64_t bb = 0; bb < nblk; ++bb) {
      mbar_spin(&dotdone[bb & 1], (uint32_t)((bb >> 1) & 1));
      if (lane < L) {
        const double* dp = dpart + (size_t)(bb & 1) * NDW * L + l;
        double v = dp[0];
#pragma unroll
        for (int k = 1; k < NDW; ++k) v += dp[k * L];
        const uint32_t off_s = (uint32_t)((bb % NPS) * 16 * L * 8), boff = (uint32_t)((bb % NPS) * 8);
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (q < CS) st_async_f64(rdst[q] + off_s, rbar[q] + boff, v);
      }
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
      // w <- w0 - eta R^T delta - eta Lb mu ; S += Lb w0 - eta R^T((Lb-l+1) delta) - eta mu Lb(Lb+1)/2
      // The column of the block's rows goes to registers BEFORE delta_b is known (the rows
      // landed for dots(b)), the slot is released at once, and only the w half of the update
      // sits between delta_b and w_{b+1}; the running sum follows off the dependent cycle.
      const double* rb = rows + (size_t)s * L * SW;
      const double* dd = dl + (b & 1) * L;
      const double* ee = d2 + (b & 1) * L;
      double u, vv;
      unsigned long long c1 = 0;
      if (Lb == L) {
        double xr[L];
        mbar_wait(&full[s], (uint32_t)((b / NB) & 1));
#pragma unroll
        for (int l = 0; l < L; ++l) xr[l] = rb[l * SW + off[l & 15]];
        __syncwarp();
        if (lane == 0) mbar_arrive_local(&empty[s]);  // this warp is done with rows[s]
        mbar_spin(&dready[b & 1], (uint32_t)((b >> 1) & 1));
        c1 = prof ? clock64() : 0;
        if (t == 0) chain_trace(a.prof, cr, b, 4);
        double u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0;
#pragma unroll
        for (int l = 0; l < L; l += 4) {
          const double4 dq = *reinterpret_cast<const double4*>(dd + l);
          u0 = fma(dq.x, xr[l], u0); u1 = fma(dq.y, xr[l + 1], u1);
          u2 = fma(dq.z, xr[l + 2], u2); u3 = fma(dq.w, xr[l + 3], u3);
        }
        u = (u0 + u1) + (u2 + u3);
        const double wn = w - a.eta * u - a.eta * (double)Lb * muc;
        wsm[((b + 1) & 1) * SW + t] = wn;  // w_{b+1}
        __syncwarp();
        if (t == 0) chain_trace(a.prof, cr, b, 5);
        if (lane == 0) mbar_arrive_local(&wready[(b + 1) & 1]);  // this warp's columns of w_{b+1} written
        double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
#pragma unroll
        for (int l = 0; l < L; l += 4) {
          const double4 eq = *reinterpret_cast<const double4*>(ee + l);
          v0 = fma(eq.x, xr[l], v0); v1 = fma(eq.y, xr[l + 1], v1);
          v2 = fma(eq.z, xr[l + 2], v2); v3 = fma(eq.w, xr[l + 3], v3);
        }
        vv = (v0 + v1) + (v2 + v3);
        S += (double)Lb * w - a.eta * vv - a.eta * muc * (0.5 * (double)Lb * (double)(Lb + 1));
        w = wn;
      } else {
        mbar_wait(&dready[b & 1], (uint32_t)((b >> 1) & 1));
        c1 = prof ? clock64() : 0;
        double u0 = 0.0, v0 = 0.0;
        for (int l = 0; l < Lb; ++l) {
          const double x = rb[l * SW + pk_swz(t, l)];
          u0 = fma(dd[l], x, u0);
          v0 = fma(ee[l], x, v0);
        }
        u = u0;
        vv = v0;
        const double w0 = w;
        S += (double)Lb * w0 - a.eta * vv - a.eta * muc * (0.5 * (double)Lb * (double)(Lb + 1));
        w = w0 - a.eta * u - a.eta * (double)Lb * muc;
        wsm[((b + 1) & 1) * SW + t] = w;  // w_{b+1}
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_local(&wready[(b + 1) & 1]);
          mbar_arrive_local(&empty[s]);
        }
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

// ---------------------------------------------------------------------------
// CHAIN v7 (round 2): look-ahead depth 3.  The partial dots of block b are taken
// against w_{b-2}, two blocks early:
//   a_b = R_b w_b = a~_b - eta X2_b delta_{b-2} - eta X1_b delta_{b-1} - 2 eta L e_b,
//   delta_b = M_b (a_b - p_b) = [M_b a~_b - p''_b - Y2_b delta_{b-2}] - Y1_b delta_{b-1},
// with Y_q = eta M_b X_q and p''_b = M_b (p_b + nprev eta L e_b) from GRAM (DEPTH = 3).
// v3's dependent cycle (update -> dots -> all-to-all -> delta -> update, two blocks
// long, ~1.1 K cycles of it the DSMEM exchange) now spans three blocks, and the
// delta recurrence itself is one L x L product per block on its own warp:
//   dot warps     a~_b against w_{b-2} (lanes = rows), partials to dpart
//   sender warp   sums the dot warps' partials, st.async to every rank (complete_tx)
//   postA warp    t_b = p''_b + Y2_b delta_{b-2}             (two blocks of slack)
//   postB warp    waits the partials of b, tree-sums the CS ranks, s_b = M_b a~_b - t_b
//   chain warp    delta_b = s_b - Y1_b delta_{b-1}           (Y1 delta_{b-1} before s_b lands)
//   update warps  column in registers; w_{b+1} published first, running sum after
//   two producer lanes (own warps): packed rows ring; [M | Y1 | Y2 | p''] ring.
// Ring depths (each argued from the dependency chain dots(b) <- w_{b-2} <-
// update(b-3) <- delta_{b-3} <- partials(b-3) of every rank):
//   w slices 3, delta 4, t / s 4, dot partials 4, exchange slots 6 (a rank pushes
//   block b+6 only after its w_{b+4}, i.e. delta_{b+3}, i.e. every rank's partials
//   of b+3, whose sender needed its own w_{b+1} = update(b), after its postB(b)).
template <int SW, int L>
struct Chain7Cfg {
  static constexpr int NUW = SW / 32;
  // dot lanes take 32 / DSPLIT columns: 2 at SW = 256 (c4 53.7 -> 52.4 ns); at SW = 64 it was slower
  // (c5 20.4 -> 21.8 ns: more warps on the same shared-memory pipe), at SW = 128 no change
  static constexpr int DSPLIT = SW >= 256 ? 2 : 1;
  static constexpr int NDW = SW * L / 1024 * DSPLIT;
  // each 32-column group of the update is shared by two warps (half the block's rows each): the
  // update warps' occupancy per block (~130 instructions at ~6-8 cycles each on a lone warp) set
  // the chain's period
  static constexpr int NT = 32 * (NDW + 2 * NUW + 6);  // + sender, postA, postB, chain, rows producer, matrix producer
  // ring depths are powers of two and block counters 32-bit: the 64-bit % 3, % 6 of the first
  // version cost every role ~300 cycles of dependent integer arithmetic per block
  static constexpr int NB = SW * L * 8 <= 16384 ? 8 : 4;
  static constexpr int NMX = 2;
  static constexpr int MXW = MX7<L>::W;
  static constexpr int NPS = 8;   // >= 6 (see above)
  static constexpr int NW = 4;    // w slices: w_b in slot b % 4 (>= 3)
  static constexpr size_t smem() {
    return sizeof(double) * ((size_t)NB * L * SW + (size_t)NMX * MXW + (size_t)NPS * 16 * L + 17 * L +
                             4 * NDW * L + NW * SW + 2 * SW) +
           sizeof(uint64_t) * (2 * NB + 2 * NMX + NPS + 4 + 4 + NW + 4 + 4) + 128;
  }
};

// lane's share of row i of an L x L matrix in the lane-major pair layout (MX7): KPL consecutive k from k0
template <int L>
struct LaneRow {
  static constexpr int HALVES = 32 / L, KPL = L / HALVES;
  double m[KPL];
  __device__ __forceinline__ void load(const double* At, int i, int k0) {
#pragma unroll
    for (int kk = 0; kk < KPL; kk += 2) {
      const double2 q = *reinterpret_cast<const double2*>(At + ((k0 + kk) >> 1) * 2 * L + 2 * i);
      m[kk] = q.x;
      m[kk + 1] = q.y;
    }
  }
  // (row i) . vec, vec in shared memory; every lane of a row gets the full sum
  __device__ __forceinline__ double dot(const double* vec, int k0) const {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0, a5 = 0.0, a6 = 0.0, a7 = 0.0;
#pragma unroll
    for (int kk = 0; kk < KPL; kk += 8) {
      const double2 v0 = *reinterpret_cast<const double2*>(vec + k0 + kk);
      const double2 v1 = *reinterpret_cast<const double2*>(vec + k0 + kk + 2);
      const double2 v2 = *reinterpret_cast<const double2*>(vec + k0 + kk + 4);
      const double2 v3 = *reinterpret_cast<const double2*>(vec + k0 + kk + 6);
      a0 = fma(m[kk], v0.x, a0); a1 = fma(m[kk + 1], v0.y, a1);
      a2 = fma(m[kk + 2], v1.x, a2); a3 = fma(m[kk + 3], v1.y, a3);
      a4 = fma(m[kk + 4], v2.x, a4); a5 = fma(m[kk + 5], v2.y, a5);
      a6 = fma(m[kk + 6], v3.x, a6); a7 = fma(m[kk + 7], v3.y, a7);
    }
    double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if constexpr (HALVES == 2) r += __shfl_xor_sync(0xffffffffu, r, 16);
    return r;
  }
};

struct Chain7Args {
  const double* pk;     // this chunk's packed rows [nblk][CS][L][SW] (swizzled)
  int64_t steps;        // steps in this chunk
  const double* MX;     // nblk x MX7<L>::W
  const double* mu;     // ld
  int64_t ld;
  double eta;
  double* state;        // [0, ld) w ; [ld, 2 ld) sum
  unsigned long long* prof;  // optional event trace of CTA 0 (debug)
};

template <int SW, int L>
__global__ void __launch_bounds__(Chain7Cfg<SW, L>::NT, 1) sstep_chain7_kernel(Chain7Args a) {
  using Cf = Chain7Cfg<SW, L>;
  constexpr int NUW = Cf::NUW, NDW = Cf::NDW, NB = Cf::NB, NMX = Cf::NMX, MXW = Cf::MXW, NPS = Cf::NPS;
  constexpr int NW = Cf::NW;
  constexpr int WU0 = NDW, WSN = NDW + 2 * NUW, WPA = WSN + 1, WPB = WSN + 2, WCH = WSN + 3, WPR = WSN + 4, WPM = WSN + 5;
  constexpr int HALVES = 32 / L, KPL = L / HALVES;
  static_assert(L == 16 || L == 32, "lanes = rows in the dots");
  static_assert(SW >= 32 && SW % 32 == 0, "slice width");
  extern __shared__ __align__(128) unsigned char sm[];
  double* rows = reinterpret_cast<double*>(sm);                 // [NB][L][SW] (swizzled)
  double* mx = rows + (size_t)NB * L * SW;                      // [NMX][MXW]: M | Y1 | Y2 | p''
  double* apub = mx + NMX * MXW;                                // [NPS][16][L] partials by sender rank
  double* dl = apub + NPS * 16 * L;                             // [4][L] delta_b
  double* d2 = dl + 4 * L;                                      // [4][L] (Lb - l) delta_b
  double* tbuf = d2 + 4 * L;                                    // [4][L] t_b
  double* sbuf = tbuf + 4 * L;                                  // [4][L] s_b
  double* abuf = sbuf + 4 * L;                                  // [L] a~_b (postB)
  double* dpart = abuf + L;                                     // [4][NDW][L] dot warps' partials
  double* wsm = dpart + 4 * NDW * L;                            // [NW][SW] w slice: w_b in slot b % NW
  double* ubuf = wsm + NW * SW;                                 // [SW][2] second half's partial (u, v)
  uint64_t* full = reinterpret_cast<uint64_t*>(ubuf + 2 * SW);  // [NB]
  uint64_t* empty = full + NB;                                  // [NB]
  uint64_t* mx_full = empty + NB;                               // [NMX]
  uint64_t* mx_empty = mx_full + NMX;                           // [NMX]
  uint64_t* part = mx_empty + NMX;                              // [NPS] partials (complete_tx)
  uint64_t* dotdone = part + NPS;                               // [4]
  uint64_t* dready = dotdone + 4;                               // [4] delta_b published
  uint64_t* wready = dready + 4;                                // [NW] w_b written
  uint64_t* tready = wready + NW;                               // [4]
  uint64_t* sready = tready + 4;                                // [4]

  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t slice0 = (int64_t)cr * SW;
  const int nblk = (int)((a.steps + L - 1) / L);
  const uint32_t part_bytes = (uint32_t)(CS * L * 8);
  if (tid == 0) {
    for (int q = 0; q < NB; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 2 * NUW + NDW);
    }
    for (int q = 0; q < NMX; ++q) {
      mbar_init(&mx_full[q], 1);
      mbar_init(&mx_empty[q], 3);  // postA, postB and chain each hold their matrix row in registers
    }
    for (int q = 0; q < NPS; ++q) mbar_init(&part[q], 1);
    for (int q = 0; q < 4; ++q) {
      mbar_init(&dotdone[q], NDW);
      mbar_init(&dready[q], 1);
      mbar_init(&tready[q], 1);
      mbar_init(&sready[q], 1);
    }
    for (int q = 0; q < NW; ++q) mbar_init(&wready[q], NUW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < NPS && q < nblk; ++q) mbar_expect_tx(&part[q], part_bytes);
  }
  for (int t = tid; t < SW; t += blockDim.x) {
    const int64_t col = slice0 + t;
    wsm[t] = col < a.ld ? a.state[col] : 0.0;  // w_0
  }
  for (int t = tid; t < 8 * L; t += blockDim.x) dl[t] = 0.0;  // dl and d2
  cluster.sync();

  const int gi = lane % L, gk0 = (lane / L) * KPL;  // matrix-row lanes: row, first k
  if (warp == WPR) {
    if (lane == 0) {
      const uint32_t slice_bytes = (uint32_t)(L * SW * 8);
      for (int b = 0; b < nblk; ++b) {
        const int s = b & (NB - 1);
        if (b >= NB) mbar_spin(&empty[s], (uint32_t)(((b / NB) - 1) & 1));
        mbar_expect_tx(&full[s], slice_bytes);
        bulk_g2s(rows + (size_t)s * L * SW, a.pk + ((size_t)b * CS + cr) * L * SW, slice_bytes, &full[s]);
      }
    }
  } else if (warp == WPM) {
    if (lane == 0) {
      for (int b = 0; b < nblk; ++b) {
        const int ms = b & (NMX - 1);
        if (b >= NMX) mbar_spin(&mx_empty[ms], (uint32_t)(((b / NMX) - 1) & 1));
        mbar_expect_tx(&mx_full[ms], (uint32_t)(MXW * 8));
        bulk_g2s(mx + ms * MXW, a.MX + (size_t)b * MXW, (uint32_t)(MXW * 8), &mx_full[ms]);
      }
    }
  } else if (warp == WPA) {
    // ---------------- postA: t_b = p''_b + Y2_b delta_{b-2} ----------------
    LaneRow<L> y2;
    for (int b = 0; b < nblk; ++b) {
      const int ms = b & (NMX - 1);
      const double* Ms = mx + ms * MXW;
      mbar_spin(&mx_full[ms], (uint32_t)((b / NMX) & 1));
      y2.load(Ms + 2 * L * L, gi, gk0);
      const double pp = Ms[3 * L * L + gi];
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&mx_empty[ms]);
      double t = pp;
      if (b >= 2) {
        mbar_spin(&dready[(b - 2) & 3], (uint32_t)(((b - 2) >> 2) & 1));
        t += y2.dot(dl + ((b - 2) & 3) * L, gk0);
      }
      if (lane < L) tbuf[(b & 3) * L + gi] = t;
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&tready[b & 3]);
    }
  } else if (warp == WPB) {
    // ---------------- postB: s_b = M_b a~_b - t_b ----------------
    LaneRow<L> mr;
    for (int b = 0; b < nblk; ++b) {
      const int ms = b & (NMX - 1);
      if (!mbar_test(&mx_full[ms], (uint32_t)((b / NMX) & 1))) mbar_spin(&mx_full[ms], (uint32_t)((b / NMX) & 1));
      mr.load(mx + ms * MXW, gi, gk0);
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&mx_empty[ms]);
      const int ps = b & (NPS - 1);
      mbar_spin_cluster(&part[ps], (uint32_t)((b / NPS) & 1));
      if (lane == 0) chain_trace(a.prof, cr, b, 2);
      if (lane < L) {
        // the CS partials of row i, summed by a fixed tree (deterministic)
        const double* ap = apub + (size_t)ps * 16 * L + gi;
        double pq[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) pq[q] = q < CS ? ap[q * L] : 0.0;
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1)
#pragma unroll
          for (int q = 0; q < h; ++q) pq[q] += pq[q + h];
        abuf[gi] = pq[0];
      }
      __syncwarp();
      if (lane == 0 && b + NPS < nblk) mbar_expect_tx(&part[ps], part_bytes);  // slot read: arm block b + NPS
      const bool tok = mbar_test(&tready[b & 3], (uint32_t)((b >> 2) & 1));  // t_b is two blocks early: normally there
      const double ma = mr.dot(abuf, gk0);
      if (!tok) mbar_spin(&tready[b & 3], (uint32_t)((b >> 2) & 1));
      if (lane < L) sbuf[(b & 3) * L + gi] = ma - tbuf[(b & 3) * L + gi];
      __syncwarp();  // also: every lane is done with abuf before the next block rewrites it
      if (lane == 0) mbar_arrive_local(&sready[b & 3]);
    }
  } else if (warp == WCH) {
    // ---------------- chain: delta_b = s_b - Y1_b delta_{b-1} ----------------
    LaneRow<L> y1;
    for (int b = 0; b < nblk; ++b) {
      const int Lb = (int)min((int64_t)L, a.steps - (int64_t)b * L);
      const int ms = b & (NMX - 1);
      mbar_spin(&mx_full[ms], (uint32_t)((b / NMX) & 1));
      y1.load(mx + ms * MXW + L * L, gi, gk0);
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&mx_empty[ms]);
      const double yd = b >= 1 ? y1.dot(dl + ((b - 1) & 3) * L, gk0) : 0.0;  // before s_b is known
      mbar_spin(&sready[b & 3], (uint32_t)((b >> 2) & 1));
      const double dv = sbuf[(b & 3) * L + gi] - yd;
      if (lane < L) {
        dl[(b & 3) * L + gi] = dv;
        d2[(b & 3) * L + gi] = (double)(Lb - gi) * dv;  // (Lb - l + 1) weight, 1-based l
      }
      __syncwarp();
      if (lane == 0) {
        chain_trace(a.prof, cr, b, 3);
        mbar_arrive_local(&dready[b & 3]);
      }
    }
  } else if (warp == WSN) {
    // ---------------- sender: row l's partial to every rank ----------------
    // lane j < L / 2 sends rows 2j, 2j + 1 as one 16-byte store per rank
    uint32_t rdst[16], rbar[16];
    const uint32_t ldst = smem_u32(apub + (size_t)cr * L + 2 * (lane % (L / 2))), lbar = smem_u32(&part[0]);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      rdst[q] = q < CS ? mapa_u32(ldst, (uint32_t)q) : 0u;
      rbar[q] = q < CS ? mapa_u32(lbar, (uint32_t)q) : 0u;
    }
    for (int bb = 0; bb < nblk; ++bb) {
      mbar_spin(&dotdone[bb & 3], (uint32_t)((bb >> 2) & 1));
      const double* dp = dpart + (size_t)(bb & 3) * NDW * L + gi;
      double v = dp[0];
#pragma unroll
      for (int k = 1; k < NDW; ++k) v += dp[k * L];
      const double va = __shfl_sync(0xffffffffu, v, (2 * lane) & 31), vb = __shfl_sync(0xffffffffu, v, (2 * lane + 1) & 31);
      if (lane < L / 2) {
        const uint32_t off_s = (uint32_t)((bb & (NPS - 1)) * 16 * L * 8), boff = (uint32_t)((bb & (NPS - 1)) * 8);
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (q < CS) st_async_f64x2(rdst[q] + off_s, rbar[q] + boff, va, vb);
      }
      if (lane == 0) chain_trace(a.prof, cr, bb, 7);
    }
  } else if (warp < NDW) {
    // ---------------- dot warps: a~_bb = R_bb w_{bb-2}, lanes = rows ----------------
    constexpr int NCOL = 32 / Cf::DSPLIT;
    static_assert(NDW * HALVES * NCOL == SW, "dot warps cover the slice");
    const int l = lane % L;
    const int c0 = (warp * HALVES + lane / L) * NCOL;
    int off[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) off[jj] = jj ^ (l & 15);
    for (int bb = 0; bb < nblk; ++bb) {
      const int s = bb & (NB - 1);
      const int wi = bb >= 2 ? bb - 2 : 0;  // w_{wi}
      if (warp == 0 && lane == 0) chain_trace2(a.prof, cr, bb, 0);  // loop top (before the waits)
      const bool fok = mbar_test(&full[s], (uint32_t)((bb / NB) & 1));
      if (wi >= 1) mbar_spin(&wready[wi & (NW - 1)], (uint32_t)(((wi - 1) / NW) & 1));  // slot's k-th phase (slot 0: w_NW first)
      if (!fok) mbar_spin(&full[s], (uint32_t)((bb / NB) & 1));
      if (warp == 0 && lane == 0) chain_trace(a.prof, cr, bb, 0);
      const double* x = rows + (size_t)s * L * SW + (size_t)l * SW + c0;
      const double* wb = wsm + (size_t)(wi & (NW - 1)) * SW + c0;
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
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&empty[s]);  // this warp's reads of rows[s] are done
      if constexpr (HALVES == 2) v += __shfl_xor_sync(0xffffffffu, v, 16);
      if (lane < L) dpart[(size_t)(bb & 3) * NDW * L + warp * L + l] = v;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_local(&dotdone[bb & 3]);
        if (warp == 0) chain_trace(a.prof, cr, bb, 1);
        if (warp == NDW - 1) chain_trace2(a.prof, cr, bb, 1);  // last dot warp done
      }
    }
  } else {
    // ---------------- update warps: column slice0 + t, rows [hh L/2, (hh + 1) L/2) ----------------
    // warps 2g and 2g + 1 share the 32 columns of group g; the second hands its partial sums to
    // the first (named barrier 1 + g), which finishes w_{b+1} and the running sum
    constexpr int LH = L / 2;
    const int uw = warp - WU0, g = uw >> 1, hh = uw & 1;
    const int t = 32 * g + lane;
    const int64_t col = slice0 + t;
    const bool act = col < a.ld;
    double w = act ? a.state[col] : 0.0;
    double S = act ? a.state[a.ld + col] : 0.0;
    const double muc = act ? a.mu[col] : 0.0;
    int off[16];  // column t of row l sits at l * SW + off[l & 15]
#pragma unroll
    for (int k = 0; k < 16; ++k) off[k] = pk_swz(t, k);
    for (int b = 0; b < nblk; ++b) {
      const int s = b & (NB - 1);
      const int Lb = (int)min((int64_t)L, a.steps - (int64_t)b * L);
      const double* rb = rows + (size_t)s * L * SW + (size_t)hh * LH * SW;
      const double* dd = dl + (b & 3) * L + hh * LH;
      const double* ee = d2 + (b & 3) * L + hh * LH;
      const int ws = (b + 1) & (NW - 1);
      // the block's column goes to registers before delta_b is known (slot released at once)
      double xr[LH];
      if (!mbar_test(&full[s], (uint32_t)((b / NB) & 1))) mbar_spin(&full[s], (uint32_t)((b / NB) & 1));
      const bool dok = mbar_test(&dready[b & 3], (uint32_t)((b >> 2) & 1));  // answer arrives under the loads
#pragma unroll
      for (int l = 0; l < LH; ++l) xr[l] = rb[l * SW + off[(hh * LH + l) & 15]];
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&empty[s]);
      if (uw == 0 && lane == 0) chain_trace(a.prof, cr, b, 6);
      if (!dok) mbar_spin(&dready[b & 3], (uint32_t)((b >> 2) & 1));
      if (uw == 0 && lane == 0) chain_trace(a.prof, cr, b, 4);
      // rows past Lb (the tail block of an epoch) are zero rows with delta = 0
      double u0 = 0.0, u1 = 0.0, v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int l = 0; l < LH; l += 4) {
        const double4 dq = *reinterpret_cast<const double4*>(dd + l);
        const double4 eq = *reinterpret_cast<const double4*>(ee + l);
        u0 = fma(dq.x, xr[l], u0); u1 = fma(dq.y, xr[l + 1], u1);
        u0 = fma(dq.z, xr[l + 2], u0); u1 = fma(dq.w, xr[l + 3], u1);
        v0 = fma(eq.x, xr[l], v0); v1 = fma(eq.y, xr[l + 1], v1);
        v0 = fma(eq.z, xr[l + 2], v0); v1 = fma(eq.w, xr[l + 3], v1);
      }
      double u = u0 + u1, vv = v0 + v1;
      if (hh == 1) {
        *reinterpret_cast<double2*>(ubuf + 2 * t) = make_double2(u, vv);
        named_bar(1 + g, 64);  // partials visible to the first warp ...
        named_bar(1 + g, 64);  // ... and read before the next block overwrites them
      } else {
        named_bar(1 + g, 64);
        const double2 o = *reinterpret_cast<const double2*>(ubuf + 2 * t);
        named_bar(1 + g, 64);
        u += o.x;
        vv += o.y;
        const double wn = w - a.eta * u - a.eta * (double)Lb * muc;
        wsm[ws * SW + t] = wn;  // w_{b+1}
        __syncwarp();
        if (uw == 0 && lane == 0) chain_trace(a.prof, cr, b, 5);
        if (uw == 2 * NUW - 2 && lane == 0) chain_trace2(a.prof, cr, b, 2);  // last column group's w out
        if (lane == 0) mbar_arrive_local(&wready[ws]);
        S += (double)Lb * w - a.eta * vv - a.eta * muc * (0.5 * (double)Lb * (double)(Lb + 1));
        w = wn;
      }
    }
    if (act && hh == 0) {
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
