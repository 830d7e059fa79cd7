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
// dependent part per block: a = R w0 (cluster-reduced through DSMEM, one
// cluster barrier per block), delta = M (a - p), and the two rank-L updates.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "svrg.cuh"
#include "fullgrad.cuh"

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
// PREP: one CTA (256 threads) per block of L steps.
//   Mout[b] (L x L, stored TRANSPOSED: Mout[b][j*L + i] = M[i][j]), pout[b] (L).  Padded steps (beyond `steps`)
//   get c_l = 0, so delta_l = 0 there.
template <class T, int L>
__global__ void __launch_bounds__(256)
sstep_prep_kernel(SstepRows R, const int64_t* __restrict__ idx, int64_t steps, const double* __restrict__ inv_nq,
                  double data_coef, double reg_coef, const double* __restrict__ mu,
                  const double* __restrict__ wbar, double eta, double* __restrict__ Mout,
                  double* __restrict__ pout) {
  constexpr int CW = 32;                    // column chunk staged in smem
  constexpr int TPR = L / 4;                // 4x4 register tiles: TPR x TPR threads
  __shared__ double chunk[CW][L + 2];       // chunk[k][l] = r_l[col0 + k]
  __shared__ double muc[CW], wbc[CW];
  extern __shared__ double dyn[];
  double (*Gs)[L + 1] = reinterpret_cast<double (*)[L + 1]>(dyn);          // L x (L+1)
  double (*Xs)[L + 1] = reinterpret_cast<double (*)[L + 1]>(dyn + L * (L + 1));  // column j of T^{-1}
  __shared__ double cvec[L], evec[L], bvec[L];
  __shared__ int64_t ridx[L];
  const int tid = threadIdx.x;
  const int64_t t0 = (int64_t)blockIdx.x * L;
  if (tid < L) {
    const int64_t t = t0 + tid;
    const int64_t i = t < steps ? idx[t] : -1;
    ridx[tid] = i;
    cvec[tid] = i < 0 ? 0.0 : (i < R.n ? data_coef : reg_coef) * inv_nq[i];
  }
  __syncthreads();
  const int tr = tid / TPR, tc = tid % TPR;  // tile (tr, tc) when tid < TPR*TPR
  const bool tiler = tid < TPR * TPR;
  double g[4][4] = {};
  double e_acc = 0.0, b_acc = 0.0;  // thread tid < L accumulates row tid
  for (int64_t c0 = 0; c0 < R.d; c0 += CW) {
    __syncthreads();
    for (int e = tid; e < CW * L; e += blockDim.x) {
      const int l = e / CW, k = e % CW;
      const int64_t i = ridx[l], col = c0 + k;
      chunk[k][l] = (i >= 0 && col < R.d) ? row_elem<T>(R, i, col) : 0.0;
    }
    if (tid < CW) {
      const int64_t col = c0 + tid;
      muc[tid] = col < R.d ? mu[col] : 0.0;
      wbc[tid] = col < R.d ? wbar[col] : 0.0;
    }
    __syncthreads();
    if (tiler) {
#pragma unroll 4
      for (int k = 0; k < CW; ++k) {
        const double2 a01 = *reinterpret_cast<const double2*>(&chunk[k][4 * tr]);
        const double2 a23 = *reinterpret_cast<const double2*>(&chunk[k][4 * tr + 2]);
        const double2 b01 = *reinterpret_cast<const double2*>(&chunk[k][4 * tc]);
        const double2 b23 = *reinterpret_cast<const double2*>(&chunk[k][4 * tc + 2]);
        const double a[4] = {a01.x, a01.y, a23.x, a23.y}, b[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) g[x][y] = fma(a[x], b[y], g[x][y]);
      }
    }
    if (tid < L) {
      for (int k = 0; k < CW; ++k) {
        e_acc = fma(chunk[k][tid], muc[k], e_acc);
        b_acc = fma(chunk[k][tid], wbc[k], b_acc);
      }
    }
  }
  if (tiler) {
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) Gs[4 * tr + x][4 * tc + y] = g[x][y];
  }
  if (tid < L) {
    evec[tid] = e_acc;
    bvec[tid] = b_acc;
  }
  __syncthreads();
  // T = I + eta C G_strict (unit lower).  Column j of T^{-1} by forward
  // substitution (thread j), then M = T^{-1} C  (M[i][j] = Tinv[i][j] c_j).
  double* Mb = Mout + (int64_t)blockIdx.x * L * L;
  if (tid < L) {
    const int j = tid;
    for (int i = 0; i < L; ++i) Xs[i][j] = i == j ? 1.0 : 0.0;
    for (int i = j + 1; i < L; ++i) {
      double s = 0.0;
      for (int k2 = j; k2 < i; ++k2) s = fma(Gs[i][k2], Xs[k2][j], s);
      Xs[i][j] = -eta * cvec[i] * s;
    }
    pout[(int64_t)blockIdx.x * L + j] = eta * (double)j * evec[j] + bvec[j];
  }
  __syncthreads();
  for (int e = tid; e < L * L; e += blockDim.x) {  // stored transposed: Mt[j][i] = M[i][j]
    const int j = e / L, i = e % L;
    Mb[e] = Xs[i][j] * cvec[j];
  }
}

template <int L>
constexpr size_t sstep_prep_smem() {
  return sizeof(double) * 2 * L * (L + 1);
}

// ---------------------------------------------------------------------------
// CHAIN: one cluster of CS CTAs; each CTA = 4 consumer warps + 1 producer warp.
// CTA r owns columns [r*SW, r*SW + SW), SW = 128*CPT; consumer thread t owns
// columns r*SW + t*CPT + [0, CPT) of w and of the running sum (registers).
//  * producer warp: per block, loads the L indices and issues one bulk copy
//    (cp.async.bulk, 1-D TMA) per row slice into an NB-deep ring (full/empty
//    mbarriers), running up to NB blocks ahead;
//  * consumers: partial a = R w0 over the slice -> transposed warp reductions
//    -> CTA partial published in shared memory; thread 0 then arrives
//    (release, cluster scope) on every CTA's `ready` mbarrier; after waiting on
//    its own `ready` (acquire) each CTA reads the CS partials through DSMEM,
//    forms z = a - p, delta = M z (M prefetched into registers), and applies
//    the two rank-L updates.  No cluster-wide barrier inside the loop.
// w and the running sum persist in global state[0..ld) / [ld..2 ld) between
// launches (one launch per chunk of blocks).
struct ChainArgs {
  SstepRows R;
  const int64_t* idx;   // chunk indices
  int64_t steps;        // steps in this chunk
  const double* M;      // nblk x L x L (transposed)
  const double* p;      // nblk x L
  const double* mu;     // ld
  double eta;
  double* state;        // [0, ld) w ; [ld, 2 ld) sum
  unsigned long long* prof;  // optional: per-phase cycle totals of CTA 0 / thread 0 (debug)
};

constexpr int kChainNB = 3;  // row-ring depth

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

template <class T, int CPT, int L>
__global__ void __launch_bounds__(160, 1) sstep_chain_kernel(ChainArgs a) {
  constexpr int NT = 128, SW = NT * CPT, NB = kChainNB;
  constexpr size_t ROWB = (size_t)SW * 8;  // bytes per row slot (fits an fp64 slice)
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* rows = sm;                                                  // [NB][L][ROWB]
  double* apub = reinterpret_cast<double*>(sm + (size_t)NB * L * ROWB);     // [2][L]
  double* zbuf = apub + 2 * L;                                               // [L]
  double* delta = zbuf + L;                                                  // [L]
  double* delta2 = delta + L;                                                // [L]
  double* wpart = delta2 + L;                                                // [4][L] (unused)
  int64_t* ridx = reinterpret_cast<int64_t*>(wpart + 4 * L);                 // [NB][L]
  uint64_t* full = reinterpret_cast<uint64_t*>(ridx + NB * L);               // [NB]
  uint64_t* empty = full + NB;                                               // [NB]
  uint64_t* ready = empty + NB;                                              // [2]
  uint64_t* dmask = ready + 2;                                               // [NB] bit l: row l is a data row
  double* wsm = reinterpret_cast<double*>(dmask + NB);                       // [SW] current w slice

  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SstepRows& R = a.R;
  const int64_t slice0 = (int64_t)cr * SW;
  const int64_t nblk = (a.steps + L - 1) / L;
  if (tid == 0) {
    for (int q = 0; q < NB; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 1);
    }
    mbar_init(&ready[0], CS);
    mbar_init(&ready[1], CS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();  // every CTA's barriers exist before any remote arrive

  if (warp == 4) {
    // ---------------- producer warp ----------------
    const int64_t slice_elems = std::min<int64_t>(SW, R.ld - slice0);  // may be <= 0 past ld
    // indices are loaded one block ahead (their L2 latency overlaps the copies)
    int64_t nxt[L / 32];
    auto load_idx = [&](int64_t b, int64_t (&dst)[L / 32]) {
#pragma unroll
      for (int h = 0; h < L / 32; ++h) {
        const int64_t t = b * L + lane + 32 * h;
        dst[h] = (b < nblk && t < a.steps) ? a.idx[t] : -1;
      }
    };
    load_idx(0, nxt);
    const bool pprof = a.prof && cr == 0 && lane == 0;
    unsigned long long pw = 0, pi = 0;
    for (int64_t b = 0; b < nblk; ++b) {
      const int slot = (int)(b % NB);
      unsigned long long q0 = pprof ? clock64() : 0;
      int64_t cur[L / 32];
#pragma unroll
      for (int h = 0; h < L / 32; ++h) cur[h] = nxt[h];
      load_idx(b + 1, nxt);
      if (b >= NB) mbar_wait(&empty[slot], (uint32_t)(((b / NB) - 1) & 1));
      unsigned long long q1 = pprof ? clock64() : 0;
      // row indices -> smem, data-row mask, then one bulk copy (1-D TMA) per row slice
      uint32_t bytes = 0;
      uint64_t mask = 0;
#pragma unroll
      for (int h = 0; h < L / 32; ++h) {
        const int64_t i = cur[h];
        ridx[slot * L + lane + 32 * h] = i;
        if (i >= 0 && slice_elems > 0) bytes += (uint32_t)(slice_elems * (i < R.n ? (int64_t)sizeof(T) : 8));
        const unsigned bal = __ballot_sync(0xffffffffu, i >= 0 && i < R.n);
        mask |= (uint64_t)bal << (32 * h);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, off);
      if (lane == 0) {
        dmask[slot] = mask;
        if (bytes) mbar_expect_tx(&full[slot], bytes);
        else mbar_arrive_local(&full[slot]);
      }
      __syncwarp();
      if (bytes) {
#pragma unroll
        for (int h = 0; h < L / 32; ++h) {
          const int l = lane + 32 * h;
          const int64_t i = cur[h];
          if (i < 0 || slice_elems <= 0) continue;
          unsigned char* dst = rows + ((size_t)slot * L + l) * ROWB;
          if (i < R.n)
            bulk_g2s(dst, static_cast<const T*>(R.Xt) + i * R.ld + slice0, (uint32_t)(slice_elems * sizeof(T)),
                     &full[slot]);
          else
            bulk_g2s(dst, R.B + (i - R.n) * R.ld + slice0, (uint32_t)(slice_elems * 8), &full[slot]);
        }
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
      wsm[tid * CPT + c] = w[c];
    }
    named_bar(1, NT);
    unsigned long long tp[8] = {};
    const bool prof = a.prof && cr == 0 && tid == 0;
    for (int64_t b = 0; b < nblk; ++b) {
      const int slot = (int)(b % NB), par = (int)(b & 1);
      const int Lb = (int)min((int64_t)L, a.steps - b * L);
      unsigned long long c0 = prof ? clock64() : 0;
      mbar_wait(&full[slot], (uint32_t)((b / NB) & 1));
      unsigned long long c1 = prof ? clock64() : 0;
      const unsigned char* rb = rows + (size_t)slot * L * ROWB;
      const int64_t* ri = ridx + slot * L;
      // 1. a_l over this CTA's slice: warp q owns rows [q*L/4, (q+1)*L/4) entirely;
      //    lane j takes columns j, j+32, ... of the slice (w from shared memory), one
      //    transposed warp reduction per warp — no cross-warp stage.
      const uint64_t dm = dmask[slot];
      auto elem = [&](int l, int c) -> double {
        if constexpr (sizeof(T) == 8) {
          return reinterpret_cast<const double*>(rb + (size_t)l * ROWB)[tid * CPT + c];
        } else {
          return ((dm >> l) & 1ull) ? (double)reinterpret_cast<const T*>(rb + (size_t)l * ROWB)[tid * CPT + c]
                                    : reinterpret_cast<const double*>(rb + (size_t)l * ROWB)[tid * CPT + c];
        }
      };
      {
        constexpr int RPW = L / 4;        // rows per warp
        constexpr int CPL = SW / 32;      // columns per lane
        double wl[CPL];
        // columns past the copied slice (ld - slice0) hold stale shared memory: mask them
        const int64_t valid = R.ld - slice0;
        bool lok[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {  // interleaved: lane j takes columns j, j+32, ... (conflict-free)
          lok[c] = (int64_t)(lane + 32 * c) < valid;
          wl[c] = wsm[lane + 32 * c];
        }
        double v[RPW];
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
          const int l = warp * RPW + q;
          const unsigned char* rowp = rb + (size_t)l * ROWB;
          double s = 0.0;
          if (sizeof(T) == 8 || ((dm >> l) & 1ull) == 0) {
            const double* x = reinterpret_cast<const double*>(rowp) + lane;
#pragma unroll
            for (int c = 0; c < CPL; ++c) s = fma(lok[c] ? x[32 * c] : 0.0, wl[c], s);
          } else {
            const T* x = reinterpret_cast<const T*>(rowp) + lane;
#pragma unroll
            for (int c = 0; c < CPL; ++c) s = fma(lok[c] ? (double)x[32 * c] : 0.0, wl[c], s);
          }
          v[q] = l < Lb ? s : 0.0;
        }
        warp_transpose_reduce<RPW>(v, lane);
        if ((lane & ((32 / RPW) - 1)) == 0) apub[par * L + warp * RPW + row_of_lane<RPW>(lane)] = v[0];
      }
      // M column `tid` and p_tid of this block: loads in flight across the exchange
      double Mc[L];
      double pl = 0.0;
      if (tid < L) {
        const double* Mg = a.M + b * L * L;
#pragma unroll
        for (int k = 0; k < L; ++k) Mc[k] = Mg[(int64_t)k * L + tid];
        pl = a.p[b * L + tid];
      }
      named_bar(1, NT);  // this CTA's partials are complete before they are published
      unsigned long long c2 = prof ? clock64() : 0;
      // 2. publish to the cluster and gather the CS partials (DSMEM)
      if (tid < CS) mbar_arrive_remote(&ready[par], (uint32_t)tid);
      mbar_wait_cluster(&ready[par], (uint32_t)((b >> 1) & 1));
      unsigned long long c3 = prof ? clock64() : 0;
      if (tid < L) {
        double part[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) part[q] = q < CS ? cluster.map_shared_rank(apub, q)[par * L + tid] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) s += part[q];
        zbuf[tid] = s - pl;
      }
      named_bar(1, NT);
      unsigned long long c4 = prof ? clock64() : 0;
      // delta = M z (thread tid < L: row tid, four partial sums)
      if (tid < L) {
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
        for (int k = 0; k < L; k += 4) {
          d0 = fma(Mc[k], zbuf[k], d0);
          d1 = fma(Mc[k + 1], zbuf[k + 1], d1);
          d2 = fma(Mc[k + 2], zbuf[k + 2], d2);
          d3 = fma(Mc[k + 3], zbuf[k + 3], d3);
        }
        delta[tid] = (d0 + d1) + (d2 + d3);
        delta2[tid] = (double)(Lb - tid) * delta[tid];  // (Lb - l + 1) weight, 1-based l
      }
      named_bar(1, NT);
      unsigned long long c5 = prof ? clock64() : 0;
      // 3. w <- w0 - eta R^T delta - eta Lb mu ; S += Lb w0 - eta R^T((Lb-l+1) delta) - eta mu Lb(Lb+1)/2
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if (!act[c]) continue;
        double u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0, v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
        int l = 0;
        for (; l + 3 < Lb; l += 4) {
          const double x0 = elem(l, c), x1 = elem(l + 1, c), x2 = elem(l + 2, c), x3 = elem(l + 3, c);
          const double4 dd = *reinterpret_cast<const double4*>(delta + l);
          const double4 ee = *reinterpret_cast<const double4*>(delta2 + l);
          u0 = fma(dd.x, x0, u0); u1 = fma(dd.y, x1, u1); u2 = fma(dd.z, x2, u2); u3 = fma(dd.w, x3, u3);
          v0 = fma(ee.x, x0, v0); v1 = fma(ee.y, x1, v1); v2 = fma(ee.z, x2, v2); v3 = fma(ee.w, x3, v3);
        }
        for (; l < Lb; ++l) {
          const double x = elem(l, c);
          u0 = fma(delta[l], x, u0);
          v0 = fma(delta2[l], x, v0);
        }
        const double u = (u0 + u1) + (u2 + u3), v = (v0 + v1) + (v2 + v3);
        const double w0 = w[c];
        S[c] += (double)Lb * w0 - a.eta * v - a.eta * mu[c] * (0.5 * (double)Lb * (double)(Lb + 1));
        w[c] = w0 - a.eta * u - a.eta * (double)Lb * mu[c];
        wsm[tid * CPT + c] = w[c];
      }
      named_bar(1, NT);  // every consumer is done with rows[slot], zbuf, delta; new w visible
      if (tid == 0) mbar_arrive_local(&empty[slot]);
      if (prof) {
        const unsigned long long c6 = clock64();
        tp[0] += c1 - c0; tp[1] += c2 - c1; tp[2] += c3 - c2; tp[3] += c4 - c3; tp[4] += c5 - c4; tp[5] += c6 - c5;
        tp[6] += 1;
      }
    }
    if (prof)
      for (int q = 0; q < 7; ++q) atomicAdd(a.prof + q, tp[q]);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (!act[c]) continue;
      a.state[col0 + c] = w[c];
      a.state[R.ld + col0 + c] = S[c];
    }
  }
  cluster.sync();  // no CTA exits while others may still read its smem / arrive on its barriers
}

template <int CPT, int L>
constexpr size_t sstep_chain_smem() {
  return (size_t)kChainNB * L * 128 * CPT * 8 + sizeof(double) * (2 * L + L + 2 * L + 4 * L) +
         sizeof(int64_t) * kChainNB * L + sizeof(uint64_t) * (3 * kChainNB + 2) + sizeof(double) * 128 * CPT + 128;
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
