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
// reduction through DSMEM started) while block b-1 is still being resolved; the
// exchange latency leaves the dependent chain.  PREP folds eta L e_b into
// p'_b = p_b + eta L e_b for every block but the first of a launch, whose a_0 is
// computed directly.
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

// ---------------------------------------------------------------------------
// PREP: one CTA (256 threads, 8 warps) per block of L = 32 steps.  One FP64
// tensor-core (DMMA m8n8k4) product of the block's rows against the staged rows
// [R_b; R_{b-1}; mu; wbar] gives G = R_b R_b^T, X = R_b R_{b-1}^T (look-ahead),
// e = R_b mu and b = R_b wbar in one pass over the rows (column chunks of 32,
// register-prefetched one chunk ahead).  Then M = (I + eta C G_strict)^{-1} C by
// forward substitution.  Outputs: Mout[b] (L x L, stored TRANSPOSED:
// Mout[b][j*L + i] = M[i][j]), pout[b] (L), Xout[b] (transposed, blocks > 0 of
// the launch).  Padded steps (beyond `steps`) get c_l = 0, so delta_l = 0 there.
template <class T, int L>
__global__ void __launch_bounds__(256)
sstep_prep_kernel(SstepRows R, const int64_t* __restrict__ idx, int64_t steps, const double* __restrict__ inv_nq,
                  double data_coef, double reg_coef, const double* __restrict__ mu,
                  const double* __restrict__ wbar, double eta, double* __restrict__ Mout,
                  double* __restrict__ pout, double* __restrict__ Xout) {
  static_assert(L == 32, "warp tiling assumes L = 32");
  constexpr int KC = 32, SP = KC + 4;         // staged columns per chunk, padded row stride (conflict-free frags)
  constexpr int NR = 2 * L + 8;               // staged rows: block b, block b-1, mu, wbar, zero pad
  constexpr int NTN = NR / 8;                 // n-tiles (9)
  constexpr int PER = NR * KC / 256;          // staged elements per thread per chunk (9)
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
    const int mt = warp & 3, nb = warp >> 2;  // m-tile; n-tiles nb, nb+2, ...
    double acc[5][2] = {};
    double v[PER];
    fetch(0, v);
    for (int64_t c0 = 0; c0 < R.d; c0 += KC) {
      __syncthreads();
  #pragma unroll
      for (int q = 0; q < PER; ++q) {
        const int e = tid + q * 256;
        st[(e / KC) * SP + e % KC] = v[q];
      }
      __syncthreads();
      if (c0 + KC < R.d) fetch(c0 + KC, v);  // next chunk in flight during the products
  #pragma unroll
      for (int k4 = 0; k4 < KC; k4 += 4) {
        const double a = st[(8 * mt + (lane >> 2)) * SP + k4 + (lane & 3)];
  #pragma unroll
        for (int j = 0; j < 5; ++j) {
          const int nt = nb + 2 * j;
          if (nt < NTN) dmma_884(acc[j][0], acc[j][1], a, st[(8 * nt + (lane >> 2)) * SP + k4 + (lane & 3)]);
        }
      }
    }
    __syncthreads();
    double* res = st;  // res[i*RS + n]: n < L: G, L..2L-1: X, 2L: e, 2L+1: b
  #pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int nt = nb + 2 * j;
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
// CHAIN: one cluster of CS CTAs; each CTA = 4 consumer warps + 2 producer warps
// + 1 signaller warp.
// CTA r owns columns [r*SW, r*SW + SW), SW = 128*CPT; consumer thread t owns
// columns r*SW + t*CPT + [0, CPT) of w and of the running sum (registers).
//  * row producer warp: per block, loads the L indices and issues one bulk copy
//    (cp.async.bulk, 1-D TMA) per row slice into an NB-deep ring (full/empty
//    mbarriers), running up to NB blocks ahead;
//  * M/X producer warp: bulk-copies M_b^T, X_b^T and p_b (from PREP) into an
//    MXB-deep shared ring, so no consumer register or LSU slot holds them;
//  * consumers, iteration b: (1) partial dots a~_{b+1} = R_{b+1} w_b over the
//    slice -> transposed warp reductions -> pushed by remote DSMEM stores into
//    apub[(b+1)%4][rank] of every CTA; (2) wait (acquire) on ready[b%4] —
//    completed one iteration earlier, normally — sum the CS partials from local
//    shared memory, z = a~_b - eta X_b delta_{b-1} - p'_b (threads L..2L-1 form
//    the X term), delta_b = M_b z (M, X staged in shared memory by a producer
//    warp); (3) the two rank-L updates with the rows of block b;
//  * signaller warp: after each block's partials are pushed (local mbarrier),
//    arrives (release, cluster scope) on every CTA's ready mbarrier, keeping
//    the fence latency off the consumers.
//    No cluster-wide barrier inside the loop.
// w and the running sum persist in global state[0..ld) / [ld..2 ld) between
// launches (one launch per chunk of blocks).
struct ChainArgs {
  SstepRows R;
  const int64_t* idx;   // chunk indices
  int64_t steps;        // steps in this chunk
  const double* M;      // nblk x L x L (transposed)
  const double* p;      // nblk x L  (p'_b: look-ahead correction folded in for b >= 1)
  const double* X;      // nblk x L x L (transposed): R_b R_{b-1}^T, b >= 1
  const double* mu;     // ld
  double eta;
  double* state;        // [0, ld) w ; [ld, 2 ld) sum
  unsigned long long* prof;  // optional: per-phase cycle totals of CTA 0 / thread 0 (debug)
};

constexpr int kChainIdxAhead = 4;  // blocks of step indices the row producer keeps in flight

// row-ring depth: 4 for 1 KB row slices (blocks b, b+1 in use, two in flight), 3 when
// the slices are 2 KB (shared memory)
constexpr int chain_nb(int slice_doubles) { return slice_doubles <= 128 ? 4 : 3; }

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive (release, cluster scope) on the mbarrier at the same offset in CTA `rank`
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
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

// consumers + 2 delta warps + row producer + M/X producer + signaller + second
// row producer [+ two wideners for fp32 rows].  (A st.async exchange with
// mbarrier complete_tx in place of the signaller was ~9 % faster per block but
// not run-to-run deterministic at c3 (16 ranks): removed.)
template <class T, int CPT, int NT>
constexpr int chain_threads() {
  return NT + 192 + ((CPT == 1 && NT == 128 && sizeof(T) == 4) ? 64 : 0);
}

template <class T, int CPT, int L, int MXB, int NT>
__global__ void __launch_bounds__(chain_threads<T, CPT, NT>(), 1) sstep_chain_kernel(ChainArgs a) {
  // warps: NCW consumers | 2 delta warps | row producer | M/X producer | signaller
  constexpr int NCW = NT / 32;
  constexpr int DW = NCW, WROW = NCW + 2, WMX = NCW + 3, WSIG = NCW + 4;
  static_assert(2 * L <= 64, "the two delta warps hold the M and X rows");
  constexpr int SW = NT * CPT, NB = chain_nb(NT * CPT);
  constexpr int MXW = 2 * L * L + L;  // doubles per M/X slot: M_b^T, X_b^T, then p_b
  constexpr size_t ROWB = (size_t)SW * 8;  // bytes per row slot (fits an fp64 slice)
  constexpr int IA = kChainIdxAhead;       // index ring depth (blocks of indices in flight)
  static_assert(L == 32, "one row per producer lane");
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* rows = sm;                                                  // [NB][L][ROWB]
  double* mx = reinterpret_cast<double*>(sm + (size_t)NB * L * ROWB);       // [MXB][MXW] M_b^T, X_b^T, p_b
  // PUSH (CPT = 1): every rank pushes its partials into apub[slot][rank] of all
  // ranks and gathers locally; pull (CPT = 2, where shared memory is tight): each
  // rank keeps its own apub[slot] and the gather reads the ranks remotely.
  constexpr bool PUSH = CPT == 1 && NT == 128;
  constexpr int NP = 2;             // row producer warps (each gathers 16 rows of a block)
  constexpr int RPP = L / NP;       // rows per producer warp
  constexpr int WPR2 = NCW + 5;  // second row producer
  constexpr int WWID = NCW + 6;  // first widener warp
  constexpr int NWID = 2;        // widener warps
  // fp32 data rows are widened to fp64 in their ring slot by two widener warps as
  // soon as they land, so the consumers' dots and update read fp64 only.  With
  // 256-column slices (d > 2048) the wideners cannot keep up (c4: 3.2 K -> 3.8 K
  // cycles per block) and the consumers widen in the dots instead.
  constexpr bool PWIDEN = sizeof(T) == 4 && PUSH;
  double* apub = mx + MXB * MXW;                                             // [4][PUSH ? 16 : 1][L]
  double* zbuf = apub + 4 * (PUSH ? 16 : 1) * L;                             // [L] (also the X term)
  double* xterm = zbuf;                                                      // thread i reads xterm[i] then writes zbuf[i]
  double* dl = zbuf + L;                                                     // [2][L] delta_b (by parity)
  double* delta2 = dl + 2 * L;                                               // [2][L]
  uint64_t* full = reinterpret_cast<uint64_t*>(delta2 + 2 * L);              // [NB]
  uint64_t* empty = full + NB;                                               // [NB]
  uint64_t* ready = empty + NB;                                              // [4]
  uint64_t* mx_full = ready + 4;                                             // [MXB]
  uint64_t* mx_empty = mx_full + MXB;                                        // [MXB]
  uint64_t* pub = mx_empty + MXB;                                            // [2] local: partials pushed
  uint64_t* dready = pub + 2;                                                // [2] local: delta_b published
  uint64_t* dmask = dready + 2;                                              // [NB] bit l: row l is a data row
  double* wsm = reinterpret_cast<double*>(dmask + NB);                       // [2][SW] w slice by block parity
  int64_t* iring = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(wsm + 2 * SW) + 15) & ~uintptr_t(15));  // [IA][L]
  uint64_t* ifull = reinterpret_cast<uint64_t*>(iring + IA * L);             // [2][IA] (per producer)
  uint64_t* wide = ifull + 2 * IA;                                           // [NB][NWID] fp32 rows widened

  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SstepRows& R = a.R;
  const int64_t slice0 = (int64_t)cr * SW;
  const int64_t nblk = (a.steps + L - 1) / L;
  if (tid == 0) {
    for (int q = 0; q < NB; ++q) {
      mbar_init(&full[q], NP);  // one (expect_tx) arrival per row producer warp
      mbar_init(&empty[q], 1);
    }
    for (int q = 0; q < 4; ++q) {
      // push: one local arrival (the arming expect_tx) + CS * L * 8 bytes of st.async
      // partials; pull: one release arrive per rank from its signaller
      mbar_init(&ready[q], CS);  // one release arrive per rank (its signaller)
    }
    for (int q = 0; q < MXB; ++q) {
      mbar_init(&mx_full[q], 1);
      mbar_init(&mx_empty[q], 1);
    }
    mbar_init(&pub[0], NCW);
    mbar_init(&pub[1], NCW);
    mbar_init(&dready[0], 1);
    mbar_init(&dready[1], 1);
    for (int q = 0; q < 2 * IA; ++q) mbar_init(&ifull[q], 1);
    for (int q = 0; q < NB * NWID; ++q) mbar_init(&wide[q], 1);  // [slot][widener warp]
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();  // every CTA's barriers exist before any remote arrive

  if (warp == WSIG) {
    // ---------------- signaller: once this CTA's partials of block j are pushed
    // (pub), arrive (release, cluster scope) on every rank's ready[j % 4].  The
    // release fence latency stays off the consumers' path.  pub is 2-deep: the
    // consumers cannot complete phase j+2 before their ready[j] wait, which needs
    // this warp's arrive for j.
    for (int64_t j = 0; j < nblk; ++j) {
      mbar_wait(&pub[j & 1], (uint32_t)((j >> 1) & 1));
      if (lane < CS) mbar_arrive_remote(&ready[j & 3], (uint32_t)lane);
    }
  } else if (warp == WMX) {
    // ---------------- M/X producer: M_b^T, X_b^T, p_b by bulk copy ----------------
    if (lane == 0) {
      for (int64_t b = 0; b < nblk; ++b) {
        const int slot = (int)(b % MXB);
        if (b >= MXB) mbar_wait(&mx_empty[slot], (uint32_t)(((b / MXB) - 1) & 1));
        double* dst = mx + slot * MXW;
        mbar_expect_tx(&mx_full[slot], (uint32_t)(MXW * 8));
        bulk_g2s(dst, a.M + b * L * L, (uint32_t)(L * L * 8), &mx_full[slot]);
        bulk_g2s(dst + L * L, a.X + b * L * L, (uint32_t)(L * L * 8), &mx_full[slot]);  // b = 0: unused
        bulk_g2s(dst + 2 * L * L, a.p + b * L, (uint32_t)(L * 8), &mx_full[slot]);
      }
    }
  } else if (warp == WROW || warp == WPR2) {
    // ---------------- row producer warps ----------------
    // NP warps gather the sampled rows, each RPP of them.  A bulk copy costs ~70 cycles of issue
    // (an elect/broadcast loop per lane), so one warp issuing all 32 rows took
    // ~2.2 K cycles per block — about the whole block.
    const int h = warp == WROW ? 0 : 1;   // this producer's half
    const int64_t slice_elems = std::min<int64_t>(SW, R.ld - slice0);  // may be <= 0 past ld
    // The step indices of full blocks travel IA blocks ahead through a shared ring
    // (one bulk copy per block): a register load one block ahead left the producer
    // waiting a dependent global-load latency (~2 K cycles) per block.
    const int64_t nfull = a.steps / L;  // blocks whose L indices all exist
    int64_t* my_ring = iring + h * IA * RPP;
    uint64_t* my_full = ifull + h * IA;
    auto issue_idx = [&](int64_t b) {
      if (b < nfull) {
        const int q = (int)(b % IA);
        mbar_expect_tx(&my_full[q], (uint32_t)(RPP * 8));
        bulk_g2s(my_ring + q * RPP, a.idx + b * L + h * RPP, (uint32_t)(RPP * 8), &my_full[q]);
      }
    };
    if (lane == 0)
      for (int64_t b = 0; b < IA; ++b) issue_idx(b);
    const bool pprof = a.prof && cr == 0 && lane == 0 && h == 0;
    unsigned long long pw = 0, pi = 0;
    const bool mine = lane < RPP;  // lane owns row h * RPP + lane
    for (int64_t b = 0; b < nblk; ++b) {
      const int slot = (int)(b % NB);
      unsigned long long q0 = pprof ? clock64() : 0;
      int64_t i = -1;
      if (b < nfull) {
        const int q = (int)(b % IA);
        mbar_wait(&my_full[q], (uint32_t)((b / IA) & 1));
        if (mine) i = my_ring[q * RPP + lane];
        __syncwarp();  // every lane has read slot q before it is refilled
        if (lane == 0) issue_idx(b + IA);
      } else if (mine) {  // the partial last block of the launch: direct loads
        const int64_t t = b * L + h * RPP + lane;
        i = t < a.steps ? a.idx[t] : -1;
      }
      if (b >= NB) mbar_wait(&empty[slot], (uint32_t)(((b / NB) - 1) & 1));
      unsigned long long q1 = pprof ? clock64() : 0;
      // data-row mask (this half), then one bulk copy (1-D TMA) per row slice
      uint32_t bytes = (i >= 0 && slice_elems > 0) ? (uint32_t)(slice_elems * (i < R.n ? (int64_t)sizeof(T) : 8)) : 0u;
      const unsigned bal = __ballot_sync(0xffffffffu, i >= 0 && i < R.n);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, off);
      if (lane == 0) {
        reinterpret_cast<uint16_t*>(&dmask[slot])[h] = (uint16_t)(bal & 0xFFFFu);  // rows 16h..16h+15
        if (bytes) mbar_expect_tx(&full[slot], bytes);
        else mbar_arrive_local(&full[slot]);
      }
      __syncwarp();
      if (i >= 0 && slice_elems > 0) {
        unsigned char* dst = rows + ((size_t)slot * L + h * RPP + lane) * ROWB;
        if (i < R.n)
          bulk_g2s(dst, static_cast<const T*>(R.Xt) + i * R.ld + slice0, (uint32_t)(slice_elems * sizeof(T)),
                   &full[slot]);
        else
          bulk_g2s(dst, R.B + (i - R.n) * R.ld + slice0, (uint32_t)(slice_elems * 8), &full[slot]);
      }
      if (pprof) {
        const unsigned long long q2 = clock64();
        pw += q1 - q0;
        pi += q2 - q1;
      }
    }
    if (pprof) {
      atomicAdd(a.prof + 7, pw);
      atomicAdd(a.prof + 8, pi);
    }
  } else if (PWIDEN && warp >= WWID && warp < WWID + NWID) {
    // ---------------- two widener warps (rows 0..15 / 16..31): the fp32 data rows
    // of each landed block -> fp64 in place (the slot is sized for fp64).  Lane l
    // reads 8-byte float pairs l, l+32, ... and writes them as 16-byte double pairs
    // at the same indices: conflict-free both ways.  Every lane reads a batch of
    // rows before any lane writes it; no per-row branches ----------------
    constexpr int NV = SW / 64;                  // float pairs per lane per row
    constexpr int BR = SW <= 128 ? L / 2 : 4;    // rows per batch (register budget)
    const int64_t slice_elems = std::min<int64_t>(SW, R.ld - slice0);
    bool act[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) act[k] = 2 * (lane + 32 * k) < slice_elems;
    const int rbeg = (warp - WWID) * (L / NWID);
    for (int64_t b = 0; b < nblk; ++b) {
      const int slot = (int)(b % NB);
      mbar_wait(&full[slot], (uint32_t)((b / NB) & 1));
      const uint32_t dm = (uint32_t)dmask[slot];  // L = 32
      unsigned char* base = rows + (size_t)slot * L * ROWB;
#pragma unroll
      for (int r0 = rbeg; r0 < rbeg + L / NWID; r0 += BR) {
        float2 f[BR][NV];
#pragma unroll
        for (int r = 0; r < BR; ++r) {
          const float2* src = reinterpret_cast<const float2*>(base + (size_t)(r0 + r) * ROWB);
#pragma unroll
          for (int k = 0; k < NV; ++k) f[r][k] = act[k] ? src[lane + 32 * k] : make_float2(0.f, 0.f);
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < BR; ++r) {
          const bool dr = (dm >> (r0 + r)) & 1u;  // data row (regulariser rows are fp64 already)
          double2* o = reinterpret_cast<double2*>(base + (size_t)(r0 + r) * ROWB);
#pragma unroll
          for (int k = 0; k < NV; ++k)
            if (dr && act[k]) o[lane + 32 * k] = make_double2((double)f[r][k].x, (double)f[r][k].y);
        }
        __syncwarp();
      }
      // order these generic-proxy stores before the bulk copy that refills the slot
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&wide[slot * NWID + (warp - WWID)]);
    }
  } else if (warp == DW || warp == DW + 1) {
    // ---------------- delta warps (64 threads): resolve block b while the consumers
    // compute the look-ahead dots of block b+1 ----------------
    const int j = tid - NT;  // 0..63
    for (int64_t b = 0; b < nblk; ++b) {
      const int Lb = (int)min((int64_t)L, a.steps - b * L);
      const int mslot = (int)(b % MXB);
      const double* Ms = mx + mslot * MXW;
      const double* Xs = Ms + L * L;
      const double* ps = Ms + 2 * L * L;
      mbar_wait(&mx_full[mslot], (uint32_t)((b / MXB) & 1));
      // X term (threads L..2L-1): xterm_i = (X_b delta_{b-1})_i
      if (j >= L && j < 2 * L && b > 0) {
        const double* dp = dl + ((b - 1) & 1) * L;
        const int i = j - L;
        double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
#pragma unroll
        for (int k = 0; k < L; k += 4) {
          x0 = fma(Xs[k * L + i], dp[k], x0);
          x1 = fma(Xs[(k + 1) * L + i], dp[k + 1], x1);
          x2 = fma(Xs[(k + 2) * L + i], dp[k + 2], x2);
          x3 = fma(Xs[(k + 3) * L + i], dp[k + 3], x3);
        }
        xterm[i] = (x0 + x1) + (x2 + x3);
      }
      named_bar(2, 64);  // xterm visible
      // a_b: the CS partials of block b (DSMEM), z = a - eta X delta_prev - p'
      mbar_wait_cluster(&ready[b & 3], (uint32_t)((b >> 2) & 1));
      if (j < L) {
        double part[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          part[q] = q >= CS ? 0.0
                    : PUSH  ? apub[((b & 3) * 16 + q) * L + j]
                            : cluster.map_shared_rank(apub, q)[(b & 3) * L + j];
        double sum = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) sum += part[q];
        if (b > 0) sum -= a.eta * xterm[j];
        zbuf[j] = sum - ps[j];
      }
      named_bar(2, 64);
      // delta_b = M_b z (thread j < L: row j, four partial sums)
      double* dcur = dl + (b & 1) * L;
      double* d2 = delta2 + (b & 1) * L;
      if (j < L) {
        double d0 = 0.0, d1 = 0.0, d2v = 0.0, d3 = 0.0;
#pragma unroll
        for (int k = 0; k < L; k += 4) {
          d0 = fma(Ms[k * L + j], zbuf[k], d0);
          d1 = fma(Ms[(k + 1) * L + j], zbuf[k + 1], d1);
          d2v = fma(Ms[(k + 2) * L + j], zbuf[k + 2], d2v);
          d3 = fma(Ms[(k + 3) * L + j], zbuf[k + 3], d3);
        }
        const double dv = (d0 + d1) + (d2v + d3);
        dcur[j] = dv;
        d2[j] = (double)(Lb - j) * dv;  // (Lb - l + 1) weight, 1-based l
      }
      named_bar(2, 64);  // delta_b complete, zbuf / M / X reads done
      if (j == 0) {
        // push: slot b % 4 is read; arm it for block b + 4 (no rank can send those
        // partials before every rank has consumed block b: they need delta_{b+3})
        mbar_arrive_local(&mx_empty[mslot]);  // M/X slot consumed
        mbar_arrive_local(&dready[b & 1]);   // delta_b visible to the consumers (release.cta)
      }
    }
  } else {
    // ---------------- consumer warps (128 threads) ----------------
    const int64_t col0 = slice0 + (int64_t)tid * CPT;
    bool act[CPT];
    double w[CPT], S[CPT], mu[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      act[c] = col0 + c < R.d;
      w[c] = act[c] ? a.state[col0 + c] : 0.0;
      S[c] = act[c] ? a.state[R.ld + col0 + c] : 0.0;
      mu[c] = act[c] ? a.mu[col0 + c] : 0.0;
      wsm[tid * CPT + c] = w[c];  // w at the start of block 0 in both buffers
      wsm[SW + tid * CPT + c] = w[c];
    }
    named_bar(1, NT);
    unsigned long long tp[9] = {};
    const bool prof = a.prof && cr == 0 && tid == 0;
    // partial dots of block bb's rows (ring slot) with the current w slice, pushed
    // (remote DSMEM stores) into apub[bb % 4][cr] of every CTA of the cluster
    auto dots = [&](int64_t bb) {
      const int slot = (int)(bb % NB);
      const int Lbb = (int)min((int64_t)L, a.steps - bb * L);
      const unsigned long long w0c = prof ? clock64() : 0;
      if (PWIDEN) {
#pragma unroll
        for (int q = 0; q < NWID; ++q) mbar_wait(&wide[slot * NWID + q], (uint32_t)((bb / NB) & 1));
      } else {
        mbar_wait(&full[slot], (uint32_t)((bb / NB) & 1));
      }
      if (prof) tp[8] += clock64() - w0c;
      const unsigned char* rb = rows + (size_t)slot * L * ROWB;
      const uint64_t dm = dmask[slot];
      constexpr int RPW = L / NCW;      // rows per warp: warp q owns rows [q*RPW, (q+1)*RPW)
      constexpr int CPL = SW / 32;      // columns per lane, interleaved (conflict-free)
      double wl[CPL];
      const int64_t valid = R.ld - slice0;  // columns past the copied slice hold stale smem
      bool lok[CPL];
      // w at the start of block bb - 1 (the look-ahead dots), in buffer (bb - 1) & 1; the
      // update of block bb - 1 writes the other buffer, so a warp that is already
      // updating cannot overwrite values another warp is still loading here
      const double* wb = wsm + ((bb + 1) & 1) * SW;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        lok[c] = (int64_t)(lane + 32 * c) < valid;
        wl[c] = wb[lane + 32 * c];
      }
      double v[RPW];
#pragma unroll
      for (int q = 0; q < RPW; ++q) {
        const int l = warp * RPW + q;
        const unsigned char* rowp = rb + (size_t)l * ROWB;
        double s = 0.0;
        if (sizeof(T) == 8 || PWIDEN || ((dm >> l) & 1ull) == 0) {
          const double* x = reinterpret_cast<const double*>(rowp) + lane;
#pragma unroll
          for (int c = 0; c < CPL; ++c) s = fma(lok[c] ? x[32 * c] : 0.0, wl[c], s);
        } else {
          // fp32 data row: widen once and write the fp64 values back in place (the
          // slot is sized for fp64), so the update of this block reads fp64 rows only
          const T* x = reinterpret_cast<const T*>(rowp) + lane;
          double xv[CPL];
#pragma unroll
          for (int c = 0; c < CPL; ++c) xv[c] = lok[c] ? (double)x[32 * c] : 0.0;
          __syncwarp();  // every lane has read its fp32 values before any fp64 store lands
          double* xd = reinterpret_cast<double*>(const_cast<unsigned char*>(rowp)) + lane;
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            xd[32 * c] = xv[c];
            s = fma(xv[c], wl[c], s);
          }
        }
        v[q] = l < Lbb ? s : 0.0;
      }
      warp_transpose_reduce<RPW>(v, lane);
      // lane (32/RPW) r holds row r: broadcast the warp's RPW sums, then lane q < CS
      // writes them to rank q with 16-byte stores
      double vals[RPW];
#pragma unroll
      for (int r = 0; r < RPW; ++r) vals[r] = __shfl_sync(0xffffffffu, v[0], (32 / RPW) * r);
      if (PUSH) {
        if (lane < CS) {
          double* dst = cluster.map_shared_rank(apub, lane) + ((bb & 3) * 16 + cr) * L + warp * RPW;
#pragma unroll
          for (int r = 0; r < RPW; r += 2) *reinterpret_cast<double2*>(dst + r) = make_double2(vals[r], vals[r + 1]);
        }
      } else if (lane == 0) {
#pragma unroll
        for (int r = 0; r < RPW; ++r) apub[(bb & 3) * L + warp * RPW + r] = vals[r];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&pub[bb & 1]);  // this warp's partials of block bb are published
    };
    // prologue: a_0 = R_0 w_0 directly
    if (nblk > 0) {
      dots(0);
      named_bar(1, NT);  // dots(0) read buffer 1, which the update of block 0 rewrites
    }
    for (int64_t b = 0; b < nblk; ++b) {
      const int slot = (int)(b % NB);
      const int Lb = (int)min((int64_t)L, a.steps - b * L);
      unsigned long long c0 = prof ? clock64() : 0;
      // 1. look-ahead partial dots of block b+1 with w_b, published to the cluster
      if (b + 1 < nblk) dots(b + 1);
      unsigned long long c1 = prof ? clock64() : 0;
      // delta_b from the delta warps (computed while this iteration's dots ran)
      unsigned long long c2 = prof ? clock64() : 0;
      mbar_wait(&dready[b & 1], (uint32_t)((b >> 1) & 1));
      unsigned long long c3 = c2, c4 = c2;
      const double* dcur = dl + (b & 1) * L;
      const double* dd2 = delta2 + (b & 1) * L;
      unsigned long long c5 = prof ? clock64() : 0;
      // 3. w <- w0 - eta R^T delta - eta Lb mu ; S += Lb w0 - eta R^T((Lb-l+1) delta) - eta mu Lb(Lb+1)/2
      const unsigned char* rb = rows + (size_t)slot * L * ROWB;
      // every row of the slot is fp64 by now (fp32 rows were widened in place by dots())
      auto elem = [&](int l, int c) -> double {
        return reinterpret_cast<const double*>(rb + (size_t)l * ROWB)[tid * CPT + c];
      };
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if (!act[c]) continue;
        double u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0, v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        int l = 0;
        for (; l + 3 < Lb; l += 4) {
          const double x0 = elem(l, c), x1 = elem(l + 1, c), x2 = elem(l + 2, c), x3 = elem(l + 3, c);
          const double4 dd = *reinterpret_cast<const double4*>(dcur + l);
          const double4 ee = *reinterpret_cast<const double4*>(dd2 + l);
          u0 = fma(dd.x, x0, u0); u1 = fma(dd.y, x1, u1); u2 = fma(dd.z, x2, u2); u3 = fma(dd.w, x3, u3);
          v0 = fma(ee.x, x0, v0); v1 = fma(ee.y, x1, v1); v2 = fma(ee.z, x2, v2); v3 = fma(ee.w, x3, v3);
        }
        for (; l < Lb; ++l) {
          const double x = elem(l, c);
          u0 = fma(dcur[l], x, u0);
          v0 = fma(dd2[l], x, v0);
        }
        const double u = (u0 + u1) + (u2 + u3), v = (v0 + v1) + (v2 + v3);
        const double w0 = w[c];
        S[c] += (double)Lb * w0 - a.eta * v - a.eta * mu[c] * (0.5 * (double)Lb * (double)(Lb + 1));
        w[c] = w0 - a.eta * u - a.eta * (double)Lb * mu[c];
        wsm[((b + 1) & 1) * SW + tid * CPT + c] = w[c];  // w at the start of block b + 1
      }
      named_bar(1, NT);  // every consumer is done with rows[slot]; new w visible
      if (tid == 0) mbar_arrive_local(&empty[slot]);
      if (prof) {
        const unsigned long long c6 = clock64();
        tp[0] += c2 - c1; tp[7] += c6 - c0; tp[1] += c1 - c0; tp[2] += c3 - c2; tp[3] += c4 - c3; tp[4] += c5 - c4; tp[5] += c6 - c5;
        tp[6] += 1;
      }
    }
    if (prof)
      for (int q = 0; q < 7; ++q) atomicAdd(a.prof + q, tp[q]);
    if (prof) {
      atomicAdd(a.prof + 9, tp[7]);
      atomicAdd(a.prof + 10, tp[8]);
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!act[c]) continue;
      a.state[col0 + c] = w[c];
      a.state[R.ld + col0 + c] = S[c];
    }
  }
  cluster.sync();  // no CTA exits while others may still read its smem / arrive on its barriers
}

template <int CPT, int L, int MXB, int NT>
constexpr size_t sstep_chain_smem() {
  return (size_t)chain_nb(NT * CPT) * L * NT * CPT * 8 + sizeof(double) * MXB * (2 * L * L + L) +
         sizeof(double) * (4 * (CPT == 1 && NT == 128 ? 16 : 1) * L + 5 * L) +
         sizeof(uint64_t) * (3 * chain_nb(NT * CPT) + 4 + 2 * MXB + 4) + sizeof(double) * 2 * NT * CPT +
         sizeof(int64_t) * kChainIdxAhead * L + sizeof(uint64_t) * (2 * kChainIdxAhead + 2 * chain_nb(NT * CPT)) + 128;
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
