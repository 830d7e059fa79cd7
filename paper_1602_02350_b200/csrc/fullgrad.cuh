// K9 — the fused full-gradient + objective pass over the preconditioned rows.
//
// Replaces PreconditionedRidge::full_gradient / ::objective in Dense mode
// (ridge.cpp:174-236), which read X~ twice (dense_tmul_vec then dense_mul_vec)
// and call the objective as a third pass.  Here ONE streaming pass per call
// computes, for every local row i,
//     r_i = x~_i . w - y_i,   g += r_i * x~_i,   loss += r_i^2
// with each row held in registers between its dot and its axpy, so X~ is read
// exactly once (n*d*s bytes) — the HBM roofline of this kernel.
//
// Layout: a CTA owns ALL d columns (thread t holds columns [t*VEC, t*VEC+VEC),
// its w slice and its fp64 partial-gradient slice in registers) and streams
// tiles of TR consecutive rows; grid = a multiple of the SM count, tiles
// grid-strided.  Per tile: TR partial dots -> warp shuffles -> one smem
// exchange + __syncthreads -> residuals -> axpy into the register partials.
// Arithmetic is fp64 (fp32 rows are widened on load; precision
// is free at AI ~ 1 flop/B).  Per-CTA partials are summed in a fixed order
// (deterministic), allreduced across ranks, then scaled and combined with the
// regulariser lambda * P^{-1} w computed through the low-rank form
// P^{-1/2} v = c v + U (D - c) U^T v (precond.cpp:67-80), applied twice as the
// reference does (ridge.cpp:232-235).
#pragma once

#include "common.cuh"

namespace skr {

// Raw vector load of VEC elements (VEC*sizeof(T) bytes, a multiple of 16).
template <class T, int VEC>
__device__ __forceinline__ void load_raw(const T* __restrict__ p, T (&v)[VEC]) {
  static_assert((VEC * sizeof(T)) % 16 == 0, "16-byte vector loads");
  const float4* q = reinterpret_cast<const float4*>(p);
  float4* o = reinterpret_cast<float4*>(v);
#pragma unroll
  for (int c = 0; c < (int)(VEC * sizeof(T) / 16); ++c) o[c] = __ldcs(q + c);  // streaming: read once
}

// Reduce TR per-lane values across the warp with a transposed butterfly
// (TR-1 + 5-log2(TR) shuffles instead of 5*TR).  Afterwards lane L holds the
// warp total of row  row_of_lane<TR>(L)  in p[0].
template <int TR>
__device__ __forceinline__ void warp_transpose_reduce(double (&p)[TR], int lane) {
  int cnt = TR;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (cnt > 1) {
      const int half = cnt / 2;
      const bool upper = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < TR / 2; ++i) {
        if (i < half) {
          const double send = upper ? p[i] : p[i + half];
          const double keep = upper ? p[i + half] : p[i];
          p[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      cnt = half;
    } else {
      p[0] += __shfl_xor_sync(0xffffffffu, p[0], off);
    }
  }
}
template <int TR>
__device__ __forceinline__ int row_of_lane(int lane) {
  int row = 0, m = TR / 2, b = 4;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    if (m >= 1) { row += ((lane >> b) & 1) * m; m /= 2; b -= 1; }
  }
  return row;
}

template <class T, int VEC, int TR, int NT>
__global__ void __launch_bounds__(NT)
fullgrad_kernel(const T* __restrict__ X, int64_t ld, int64_t n, const double* __restrict__ y,
                const double* __restrict__ w, double* __restrict__ part_g,
                double* __restrict__ part_loss) {
  constexpr int NW = NT / 32;
  static_assert(TR >= 1 && TR <= 32 && (TR & (TR - 1)) == 0, "TR power of two");
  __shared__ double red[2][NW][TR];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)tid * VEC;
  const bool active = c0 < ld;
  double wv[VEC], acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    wv[v] = active ? w[c0 + v] : 0.0;
    acc[v] = 0.0;
  }
  double loss = 0.0;
  const int my_row = row_of_lane<TR>(lane);
  const bool writer = (lane & ((32 / TR) - 1)) == 0;
  const int64_t ntiles = (n + TR - 1) / TR;
  int par = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * TR;
    T xv[TR][VEC];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      if (active && r0 + t < n) {
        load_raw<T, VEC>(X + (r0 + t) * ld + c0, xv[t]);
      } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) xv[t][v] = T(0);
      }
    }
    // label of the row this lane will own after the reduction (issued early)
    const double yl = (lane < TR && r0 + lane < n) ? y[r0 + lane] : 0.0;
    double p[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      double s = 0.0;
#pragma unroll
      for (int v = 0; v < VEC; ++v) s = fma((double)xv[t][v], wv[v], s);
      p[t] = s;
    }
    warp_transpose_reduce<TR>(p, lane);
    if (writer) red[par][warp][my_row] = p[0];
    __syncthreads();
    // lane t < TR forms the residual of row t, then broadcasts it
    double rl = 0.0;
    if (lane < TR) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) s += red[par][q][lane];
      rl = (r0 + lane < n) ? s - yl : 0.0;
    }
    if (warp == 0) loss = fma(rl, rl, loss);
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      const double rt = __shfl_sync(0xffffffffu, rl, t);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = fma(rt, (double)xv[t][v], acc[v]);
    }
    par ^= 1;
  }
  if (active) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) part_g[(int64_t)blockIdx.x * ld + c0 + v] = acc[v];
  }
  if (warp == 0) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, off);
    if (lane == 0) part_loss[blockIdx.x] = loss;
  }
}

// ---------------------------------------------------------------------------
// K9 v3: the same pass with the rows staged through shared memory by the bulk
// copy engine (cp.async.bulk, the 1-D TMA) into an S-deep mbarrier ring.  A
// tile is TR consecutive rows = one contiguous byte range, so one bulk copy
// moves a whole tile; each CTA walks a contiguous range of tiles, refilling the
// stage it just drained S-1 tiles ahead.  Threads own interleaved 16-byte
// column chunks (chunk j of thread t at byte 16*t + 16*NT*j of the row) so the
// shared-memory reads are conflict-free; compute is identical to v2.
// (shared-memory address / mbarrier / bulk-copy helpers: common.cuh)
template <class T, int VEC, int NT>
__device__ __forceinline__ void lds_cols(const unsigned char* row, int tid, T (&v)[VEC]) {
  constexpr int PER = 16 / sizeof(T);  // elements per 16-byte chunk
#pragma unroll
  for (int j = 0; j < VEC / PER; ++j) {
    const float4 q = *reinterpret_cast<const float4*>(row + 16 * ((size_t)tid + (size_t)NT * j));
    *reinterpret_cast<float4*>(&v[j * PER]) = q;
  }
}

template <class T, int VEC, int TR, int NT>
__global__ void __launch_bounds__(NT, (NT <= 256) ? 2 : 1)
fullgrad_tma_kernel(const T* __restrict__ X, int64_t ld, int64_t n, const double* __restrict__ y,
                    const double* __restrict__ w, double* __restrict__ part_g,
                    double* __restrict__ part_loss, int stages) {
  constexpr int NW = NT / 32;
  constexpr int PER = 16 / sizeof(T);
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[16];
  __shared__ double red[2][NW][TR];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t row_bytes = (size_t)ld * sizeof(T);
  const size_t tile_bytes = row_bytes * TR;
  // column of element v of this thread: chunk j = v / PER
  double wv[VEC], acc[VEC];
  bool act[VEC / PER];
#pragma unroll
  for (int j = 0; j < VEC / PER; ++j) {
    const int64_t col0 = ((int64_t)tid + (int64_t)NT * j) * PER;
    act[j] = col0 < ld;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      wv[j * PER + e] = act[j] ? w[col0 + e] : 0.0;
      acc[j * PER + e] = 0.0;
    }
  }
  // tiles of this CTA: one contiguous range
  const int64_t ntiles = (n + TR - 1) / TR;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t_begin = (int64_t)blockIdx.x * per;
  const int64_t t_end = min(ntiles, t_begin + per);
  const int64_t count = t_end > t_begin ? t_end - t_begin : 0;
  auto tile_of = [&](int64_t i) { return t_begin + i; };

  auto issue = [&](int64_t i) {  // tile i of this CTA into stage i % stages
    const int64_t tile = tile_of(i);
    const int64_t r0 = tile * TR;
    const int64_t rows = min((int64_t)TR, n - r0);
    const uint32_t bytes = (uint32_t)(rows * row_bytes);
    uint64_t* bar = &full[i % stages];
    mbar_expect_tx(bar, bytes);
    bulk_g2s(smem + (size_t)(i % stages) * tile_bytes, reinterpret_cast<const unsigned char*>(X) + r0 * row_bytes,
             bytes, bar);
  };
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int64_t i = 0; i < min((int64_t)stages, count); ++i) issue(i);
  }
  __syncthreads();

  double loss = 0.0;
  const int my_row = row_of_lane<TR>(lane);
  const bool writer = (lane & ((32 / TR) - 1)) == 0;
  const bool full_cols = (int64_t)NT * VEC <= ld;  // every thread's column chunks lie inside the row
  int par = 0;
  for (int64_t i = 0; i < count; ++i) {
    const int stage = (int)(i % stages);
    const int64_t r0 = tile_of(i) * TR;
    mbar_wait(&full[stage], (uint32_t)((i / stages) & 1));
    const unsigned char* base = smem + (size_t)stage * tile_bytes;
    T xv[TR][VEC];
    if (full_cols && r0 + TR <= n) {
      // every column chunk and row of the tile is real: no per-element selects (they
      // were 19 % of the instructions and kept the ALU pipe 52 % busy at c5)
#pragma unroll
      for (int t = 0; t < TR; ++t) lds_cols<T, VEC, NT>(base + (size_t)t * row_bytes, tid, xv[t]);
    } else {
#pragma unroll
      for (int t = 0; t < TR; ++t) {
        if (r0 + t < n) {
          lds_cols<T, VEC, NT>(base + (size_t)t * row_bytes, tid, xv[t]);
#pragma unroll
          for (int j = 0; j < VEC / PER; ++j)
            if (!act[j])
#pragma unroll
              for (int e = 0; e < PER; ++e) xv[t][j * PER + e] = T(0);
        } else {
#pragma unroll
          for (int v = 0; v < VEC; ++v) xv[t][v] = T(0);
        }
      }
    }
    const double yl = (lane < TR && r0 + lane < n) ? y[r0 + lane] : 0.0;
    double p[TR];
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      double s = 0.0;
#pragma unroll
      for (int v = 0; v < VEC; ++v) s = fma((double)xv[t][v], wv[v], s);
      p[t] = s;
    }
    warp_transpose_reduce<TR>(p, lane);
    if (writer) red[par][warp][my_row] = p[0];
    __syncthreads();
    // every thread has read stage `stage` into registers: refill it S tiles ahead
    if (tid == 0 && i + stages < count) issue(i + stages);
    double rl = 0.0;
    if (lane < TR) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) s += red[par][q][lane];
      rl = (r0 + lane < n) ? s - yl : 0.0;
    }
    if (warp == 0) loss = fma(rl, rl, loss);
#pragma unroll
    for (int t = 0; t < TR; ++t) {
      const double rt = __shfl_sync(0xffffffffu, rl, t);
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[v] = fma(rt, (double)xv[t][v], acc[v]);
    }
    par ^= 1;
  }
#pragma unroll
  for (int j = 0; j < VEC / PER; ++j) {
    if (!act[j]) continue;
    const int64_t col0 = ((int64_t)tid + (int64_t)NT * j) * PER;
#pragma unroll
    for (int e = 0; e < PER; ++e) part_g[(int64_t)blockIdx.x * ld + col0 + e] = acc[j * PER + e];
  }
  if (warp == 0) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, off);
    if (lane == 0) part_loss[blockIdx.x] = loss;
  }
}

// ---------------------------------------------------------------------------
// K9 v4 for narrow rows (ld * sizeof(T) <= 8 KB, i.e. d <= 1024): WARP per row.
// Lane l owns the 16-byte chunks l, l+32, ... of every row (coalesced), w sits
// in shared memory, the fp64 partial gradient in registers; a row costs one
// warp reduction and no block-level synchronisation at all, so every warp
// streams independently (RPI rows in flight per warp).  Warps are combined
// once at the end through shared memory.
constexpr int kRowwarpThreads = 384;  // 12 warps, one CTA per SM at <= 168 registers

__device__ __noinline__ void head_projection(const double* __restrict__ Ut, double* __restrict__ uw, int64_t ld,
                                             int64_t d, int64_t k, const double* __restrict__ w, int64_t j,
                                             int lane) {
  const double* row = j < k ? Ut + j * ld : w;
  double s = 0.0;
  for (int64_t i = lane; i < d; i += 32) s = fma(row[i], w[i], s);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) uw[j] = s;
}

// Optional head work: warps 0..k of the grid first compute uw[j] = U_j . w
// (uw[k] = w . w) for the column reduction, saving a launch.
struct UwHead {
  const double* Ut;  // k x ld, or nullptr: no head work
  double* uw;
  int64_t d, k;
};

template <class T, int CH, int RPI>
__global__ void __launch_bounds__(kRowwarpThreads, 1)
fullgrad_rowwarp_kernel(const T* __restrict__ X, int64_t ld, int64_t n, const double* __restrict__ y,
                        const double* __restrict__ w, double* __restrict__ part_g,
                        double* __restrict__ part_loss, UwHead head) {
  constexpr int PER = 16 / sizeof(T);
  constexpr int E = CH * PER;  // elements per lane per row
  extern __shared__ double sw[];  // [0, ld): w; [ld, 2 ld): warp combine buffer
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) sw[i] = w[i];
  __syncthreads();
  const int64_t chunks_per_row = ld / PER;  // ld is a multiple of 16 elements
  bool act[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) act[c] = (int64_t)lane + 32 * c < chunks_per_row;
  double acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.0;
  double loss = 0.0;
  const int64_t gw = (int64_t)blockIdx.x * nw + warp, GW = (int64_t)gridDim.x * nw;
  if (head.Ut && gw <= head.k) head_projection(head.Ut, head.uw, ld, head.d, head.k, w, gw, lane);
  for (int64_t r0 = gw * RPI; r0 < n; r0 += GW * RPI) {
    T x[RPI][E];
    double yv[RPI];
#pragma unroll
    for (int q = 0; q < RPI; ++q) {
      const int64_t row = r0 + q;
      const float4* src = reinterpret_cast<const float4*>(X + row * ld);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < n && act[c]) v = __ldcs(src + lane + 32 * c);
        *reinterpret_cast<float4*>(&x[q][c * PER]) = v;
      }
      yv[q] = row < n ? y[row] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < RPI; ++q) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (!act[c]) continue;  // x is zero there; also keeps the w read inside [0, ld)
#pragma unroll
        for (int e = 0; e < PER; ++e) s = fma((double)x[q][c * PER + e], sw[(lane + 32 * c) * PER + e], s);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      const double r = (r0 + q < n) ? s - yv[q] : 0.0;
      loss = fma(r, r, loss);  // identical on every lane; lane 0 reports it
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = fma(r, (double)x[q][e], acc[e]);
    }
  }
  // combine the warps of this CTA in warp order (deterministic)
  double* buf = sw + ld;
  __shared__ double sloss[32];
  for (int q = 0; q < nw; ++q) {
    if (warp == q) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (!act[c]) continue;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
          const int64_t col = ((int64_t)lane + 32 * c) * PER + e;
          buf[col] = (q == 0 ? 0.0 : buf[col]) + acc[c * PER + e];
        }
      }
      if (lane == 0) sloss[q] = loss;
    }
    __syncthreads();
  }
  for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) part_g[(int64_t)blockIdx.x * ld + i] = buf[i];
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int q = 0; q < nw; ++q) l += sloss[q];
    part_loss[blockIdx.x] = l;
  }
}

// K9 v5 for narrow rows: warp per row (as v4), but each warp streams its rows
// through a private NB-deep shared-memory ring filled by the bulk-copy engine
// (cp.async.bulk, one 1-D copy per row, mbarrier complete_tx).  NB rows per warp
// stay in flight without holding registers, and no block barrier is needed
// inside the loop: the warp re-arms a slot right after consuming it.
template <class T, int CH, int NB, int NTH>
__global__ void __launch_bounds__(NTH, 1)
fullgrad_rowring_kernel(const T* __restrict__ X, int64_t ld, int64_t n, const double* __restrict__ y,
                        const double* __restrict__ w, double* __restrict__ part_g,
                        double* __restrict__ part_loss, UwHead head) {
  constexpr int PER = 16 / sizeof(T);
  constexpr int E = CH * PER;  // elements per lane per row
  extern __shared__ __align__(128) unsigned char rr_sm[];
  double* sw = reinterpret_cast<double*>(rr_sm);  // [0, ld): w; [ld, 2 ld): warp combine buffer
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t row_bytes = (uint32_t)(ld * sizeof(T));
  unsigned char* ring = rr_sm + ((2 * ld * sizeof(double) + 127) / 128) * 128;
  unsigned char* mine = ring + (size_t)warp * NB * row_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + (size_t)nw * NB * row_bytes) + warp * NB;
  for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) sw[i] = w[i];
  const int64_t gw = (int64_t)blockIdx.x * nw + warp, GW = (int64_t)gridDim.x * nw;
  if (lane == 0) {
    for (int s = 0; s < NB; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (lane == 0) {
    for (int s = 0; s < NB; ++s) {
      const int64_t row = gw + (int64_t)s * GW;
      if (row < n) {
        mbar_expect_tx(&bars[s], row_bytes);
        bulk_g2s(mine + (size_t)s * row_bytes, X + row * ld, row_bytes, &bars[s]);
      }
    }
  }
  if (head.Ut && gw <= head.k) head_projection(head.Ut, head.uw, ld, head.d, head.k, w, gw, lane);
  const int64_t chunks_per_row = ld / PER;  // ld is a multiple of 16 elements
  bool act[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) act[c] = (int64_t)lane + 32 * c < chunks_per_row;
  const bool all_act = chunks_per_row >= 32 * CH;  // uniform: the fast path below needs no selects
  double acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.0;
  double loss = 0.0;
  int64_t j = 0;
  for (int64_t row = gw; row < n; row += GW, ++j) {
    const int s = (int)(j % NB);
    const double yv = y[row];
    mbar_wait(&bars[s], (uint32_t)((j / NB) & 1));
    const unsigned char* slot = mine + (size_t)s * row_bytes;
    T x[E];
    double sdot = 0.0;
    if (all_act) {
      // every chunk of every lane is inside the row: no per-element selects
      if constexpr (sizeof(T) == 8) {
        const double2* src = reinterpret_cast<const double2*>(slot);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const double2 v = src[lane + 32 * c];
          x[2 * c] = v.x;
          x[2 * c + 1] = v.y;
        }
      } else {
        const float4* src = reinterpret_cast<const float4*>(slot);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const float4 v = src[lane + 32 * c];
          x[4 * c] = v.x;
          x[4 * c + 1] = v.y;
          x[4 * c + 2] = v.z;
          x[4 * c + 3] = v.w;
        }
      }
#pragma unroll
      for (int c = 0; c < CH; ++c)
#pragma unroll
        for (int e = 0; e < PER; ++e) sdot = fma((double)x[c * PER + e], sw[(lane + 32 * c) * PER + e], sdot);
    } else {
      if constexpr (sizeof(T) == 8) {
        const double2* src = reinterpret_cast<const double2*>(slot);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const double2 v = act[c] ? src[lane + 32 * c] : make_double2(0.0, 0.0);
          x[2 * c] = v.x;
          x[2 * c + 1] = v.y;
        }
      } else {
        const float4* src = reinterpret_cast<const float4*>(slot);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const float4 v = act[c] ? src[lane + 32 * c] : make_float4(0.f, 0.f, 0.f, 0.f);
          x[4 * c] = v.x;
          x[4 * c + 1] = v.y;
          x[4 * c + 2] = v.z;
          x[4 * c + 3] = v.w;
        }
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (!act[c]) continue;
#pragma unroll
        for (int e = 0; e < PER; ++e) sdot = fma((double)x[c * PER + e], sw[(lane + 32 * c) * PER + e], sdot);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, off);
    const double r = sdot - yv;
    loss = fma(r, r, loss);  // identical on every lane; lane 0 reports it
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = fma(r, (double)x[e], acc[e]);
    __syncwarp();  // every lane is done with slot s
    if (lane == 0) {
      const int64_t nxt = row + (int64_t)NB * GW;
      if (nxt < n) {
        mbar_expect_tx(&bars[s], row_bytes);
        bulk_g2s(mine + (size_t)s * row_bytes, X + nxt * ld, row_bytes, &bars[s]);
      }
    }
  }
  // combine the warps of this CTA in warp order (deterministic)
  double* buf = sw + ld;
  __shared__ double sloss[32];
  for (int q = 0; q < nw; ++q) {
    if (warp == q) {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (!act[c]) continue;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
          const int64_t col = ((int64_t)lane + 32 * c) * PER + e;
          buf[col] = (q == 0 ? 0.0 : buf[col]) + acc[c * PER + e];
        }
      }
      if (lane == 0) sloss[q] = loss;
    }
    __syncthreads();
  }
  for (int64_t i = threadIdx.x; i < ld; i += blockDim.x) part_g[(int64_t)blockIdx.x * ld + i] = buf[i];
  if (threadIdx.x == 0) {
    double l = 0.0;
    for (int q = 0; q < nw; ++q) l += sloss[q];
    part_loss[blockIdx.x] = l;
  }
}

template <int NB, int NTH>
inline size_t rowring_smem(int64_t ld, size_t elem) {
  return ((2 * ld * sizeof(double) + 127) / 128) * 128 + (size_t)(NTH / 32) * NB * ld * elem +
         (size_t)(NTH / 32) * NB * sizeof(uint64_t);
}

// Single-level deterministic reduction + finalisation: one warp per column
// (column ld = the loss), lanes sum the per-CTA partials in a fixed order, and
// the warp writes mu = sums/n + lambda (c^2 w + U (D^2 - c^2) U^T w) for its column
// (P^{-1} = c^2 I + U (D^2 - c^2) U^T; ridge.cpp:232-235) — or the raw sums when
// mu == nullptr (distributed path, allreduced afterwards).
__global__ void __launch_bounds__(256)
fullgrad_colreduce_kernel(const double* __restrict__ part_g, const double* __restrict__ part_loss,
                          int64_t ld, int parts, int64_t d, double n, double lambda,
                          const double* __restrict__ w, const double* __restrict__ Ut,
                          const double* __restrict__ uw, int64_t k, const double* __restrict__ D,
                          double c, double* __restrict__ mu, double* __restrict__ obj,
                          double* __restrict__ sums) {
  // one warp per column (j == ld: the loss); lanes take partials lane, lane+32, ...
  // in a fixed order, then a butterfly: deterministic, ~parts/32 loads in flight per lane
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j > ld) return;
  const double* src = j < ld ? part_g + j : part_loss;
  const int64_t stride = j < ld ? ld : 1;
  double a0 = 0.0, a1 = 0.0;
  int b = lane;
  for (; b + 32 < parts; b += 64) {
    a0 += src[(int64_t)b * stride];
    a1 += src[(int64_t)(b + 32) * stride];
  }
  if (b < parts) a0 += src[(int64_t)b * stride];
  double acc = a0 + a1;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  const double cc = c * c;
  if (sums) {
    if (lane == 0) sums[j] = acc;
  } else if (j < ld) {
    // lambda P^{-1} w_j = lambda (c^2 w_j + sum_l U_lj (D_l^2 - c^2) (U^T w)_l), lanes split l
    double r = 0.0;
    if (j < d)
      for (int64_t l = lane; l < k; l += 32) r = fma(Ut[l * ld + j], (D[l] * D[l] - cc) * uw[l], r);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
    if (lane == 0) mu[j] = j < d ? acc * (1.0 / n) + lambda * (cc * w[j] + r) : 0.0;
  } else if (obj) {
    double reg = 0.0;
    for (int64_t l = lane; l < k; l += 32) reg += (D[l] * D[l] - cc) * uw[l] * uw[l];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) reg += __shfl_xor_sync(0xffffffffu, reg, off);
    if (lane == 0) *obj = acc / (2.0 * n) + 0.5 * lambda * (cc * uw[k] + reg);
  }
}

// uw[j] = U_j . w (j < k) and uw[k] = w . w: one warp per projection, 8 per CTA.
__global__ void __launch_bounds__(256)
proj_kernel(const double* __restrict__ Ut, int64_t ld, int64_t d, int64_t k, const double* __restrict__ w,
            double* __restrict__ uw) {
  const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j > k) return;
  const double* row = j < k ? Ut + j * ld : w;
  double a0 = 0.0, a1 = 0.0;
  int64_t i = lane;
  for (; i + 32 < d; i += 64) {
    a0 = fma(row[i], w[i], a0);
    a1 = fma(row[i + 32], w[i + 32], a1);
  }
  if (i < d) a0 = fma(row[i], w[i], a0);
  double s = a0 + a1;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) uw[j] = s;
}

// proj[j] = U_j . v for j < k (one warp per basis vector; Ut is k x ld rows);
// the extra warp j == k computes v . v into proj[k].
__global__ void lowrank_proj_kernel(const double* __restrict__ Ut, int64_t ld, int64_t d,
                                    int64_t k, const double* __restrict__ v,
                                    double* __restrict__ proj) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp > k) return;
  const double* row = warp < k ? Ut + (int64_t)warp * ld : v;
  double s = 0.0;
  for (int64_t i = lane; i < d; i += 32) s = fma(row[i], v[i], s);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) proj[warp] = s;
}

// out_i = c v_i + sum_j U_ij (D_j - c) proj_j   (precond.cpp:67-80); zero pad to ld.
__global__ void lowrank_apply_kernel(const double* __restrict__ Ut, int64_t ld, int64_t d,
                                     int64_t k, const double* __restrict__ D, double c,
                                     const double* __restrict__ v, const double* __restrict__ proj,
                                     double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ld) return;
  if (i >= d) {
    out[i] = 0.0;
    return;
  }
  double s = 0.0;
  for (int64_t j = 0; j < k; ++j) s = fma(Ut[j * ld + i], (D[j] - c) * proj[j], s);
  out[i] = c * v[i] + s;
}

// Distributed path: mu from the allreduced sums (same algebra as the fused kernel).
__global__ void fullgrad_finalize_kernel(const double* __restrict__ sums, int64_t ld, int64_t d,
                                         double n, double lambda, const double* __restrict__ w,
                                         const double* __restrict__ Ut, const double* __restrict__ uw,
                                         int64_t k, const double* __restrict__ D, double c,
                                         double* __restrict__ mu, double* __restrict__ obj) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < ld) {
    if (j < d) {
      double r = c * c * w[j];
      for (int64_t l = 0; l < k; ++l) r = fma(Ut[l * ld + j], (D[l] * D[l] - c * c) * uw[l], r);
      mu[j] = sums[j] * (1.0 / n) + lambda * r;
    } else {
      mu[j] = 0.0;
    }
  }
  if (j == 0 && obj) {
    double reg = c * c * uw[k];
    for (int64_t l = 0; l < k; ++l) reg += (D[l] * D[l] - c * c) * uw[l] * uw[l];
    *obj = sums[ld] / (2.0 * n) + 0.5 * lambda * reg;
  }
}

}  // namespace skr
