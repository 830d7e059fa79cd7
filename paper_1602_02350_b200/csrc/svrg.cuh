// K8 — sampling tables and the index stream; K10 — the sequential SVRG inner loop.
//
// Reference: svrg_solve + DenseEpochState (svrg.cpp:18-54, :90-211) over the
// (n+d)-component preconditioned ridge (ridge.cpp:238-278).  Device layout is
// the stacked-row form R = [X~ ; B]: component i < n is
// data row x~_i with coefficient (n+d)/n and label y_i; component n+j is row j
// of B = P^{-1/2} (materialised, symmetric) with coefficient lambda(n+d) and
// label 0.  Every step is then "one row, two dots, one axpy".
#pragma once

#include "common.cuh"

namespace skr {

// make_cumulative_weights (svrg.cpp:90-106) bit-exactly: the sequential fp64
// sum and running prefix in index order (one thread; a parallel scan would
// reassociate and could flip indices at table boundaries).  Also writes
// total to *total_out.
// One CTA.  Warp 0 lane 0 runs the two dependent fp64 chains (total, then the
// running prefix) out of shared memory; warps 1.. stream beta in (and compute the
// quotients beta_i / total, which are independent) one tile ahead and write the
// finished prefix tile back, so the chain never waits on global memory.
constexpr int CUM_T = 2048;
__global__ void __launch_bounds__(512) cumulative_kernel(const double* __restrict__ beta, int64_t N,
                                                         double* __restrict__ cum, double* __restrict__ total_out) {
  __shared__ __align__(16) double buf[2][CUM_T];
  __shared__ double s_total;
  const int t = threadIdx.x, nl = blockDim.x - 32;  // loader threads: t >= 32
  const int64_t ntile = (N + CUM_T - 1) / CUM_T;
  auto load = [&](int64_t tile, bool div, double tot) {
    double* b = buf[tile & 1];
    for (int j = t - 32; j < CUM_T; j += nl) {
      const int64_t i = tile * CUM_T + j;
      const double v = i < N ? beta[i] : 0.0;
      b[j] = div ? __ddiv_rn(v, tot) : v;
    }
  };
  auto store = [&](int64_t tile) {
    const double* b = buf[tile & 1];
    for (int j = t - 32; j < CUM_T; j += nl) {
      const int64_t i = tile * CUM_T + j;
      if (i < N) cum[i] = b[j];
    }
  };
  // total = sum_i beta_i in index order (svrg.cpp:92-94)
  double total = 0.0;
  if (t >= 32) load(0, false, 0.0);
  __syncthreads();
  for (int64_t k = 0; k < ntile; ++k) {
    if (t >= 32 && k + 1 < ntile) load(k + 1, false, 0.0);
    if (t == 0) {
      const int cnt = (int)min((int64_t)CUM_T, N - k * CUM_T);
      const double* b = buf[k & 1];
      int j = 0;
      // 16 operands staged in registers per group (8-byte aligned 16-byte loads), so the
      // only serial dependence left is the add itself
      for (; j + 16 <= cnt; j += 16) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; q += 2) *reinterpret_cast<double2*>(&v[q]) = *reinterpret_cast<const double2*>(&b[j + q]);
#pragma unroll
        for (int q = 0; q < 16; ++q) total = __dadd_rn(total, v[q]);
      }
      for (; j < cnt; ++j) total = __dadd_rn(total, b[j]);
    }
    __syncthreads();
  }
  if (t == 0) s_total = total;
  __syncthreads();
  const double tot = s_total;
  // run += beta_i / total; cum_i = run  (svrg.cpp:95-104)
  double run = 0.0;
  if (t >= 32) load(0, true, tot);
  __syncthreads();
  for (int64_t k = 0; k < ntile; ++k) {
    if (t >= 32) {
      if (k >= 1) store(k - 1);
      if (k + 1 < ntile) load(k + 1, true, tot);
    }
    if (t == 0) {
      const int cnt = (int)min((int64_t)CUM_T, N - k * CUM_T);
      double* b = buf[k & 1];
      int j = 0;
      for (; j + 16 <= cnt; j += 16) {
        double v[16];
#pragma unroll
        for (int q = 0; q < 16; q += 2) *reinterpret_cast<double2*>(&v[q]) = *reinterpret_cast<const double2*>(&b[j + q]);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          run = __dadd_rn(run, v[q]);
          v[q] = run;
        }
#pragma unroll
        for (int q = 0; q < 16; q += 2) *reinterpret_cast<double2*>(&b[j + q]) = *reinterpret_cast<const double2*>(&v[q]);
      }
      for (; j < cnt; ++j) {
        run = __dadd_rn(run, b[j]);
        b[j] = run;
      }
    }
    __syncthreads();
  }
  if (t >= 32 && ntile > 0) store(ntile - 1);
  __syncthreads();
  if (t == 0) {
    cum[N - 1] = 1.0;
    *total_out = tot;
  }
}

// The same two sequential sums, bit for bit, at block-scan speed.  While a running
// sum S stays inside one binade [2^e, 2^(e+1)) it is an integer multiple K of
// u = 2^(e-52), and for an operand x >= 0 whose scaled value x/u is not a tie
// (fraction exactly 1/2) RN(S + x) = (K + RN(x/u)) u whatever K is.  A tile of
// operands without a tie whose sum stays inside the binade therefore reduces to an
// integer prefix sum (one block scan); every other tile (S = 0 at the start, a tie, a
// binade change - about 50 per table -, a negative or non-finite operand) is summed by
// thread 0 in index order, as cumulative_kernel does.  c5 (N = 16.8 M): 158 -> ~6 ms.
constexpr int CE_T = 512, CE_V = 8, CE_TILE = CE_T * CE_V;
template <bool DIV>
__device__ double cum_exact_chain(const double* __restrict__ beta, int64_t N, double tot, double* __restrict__ cum,
                                  double* xbuf, long long* wsum, double* s_S) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t ntile = (N + CE_TILE - 1) / CE_TILE;
  double S = 0.0;
  double nx[CE_V];
  auto fetch = [&](int64_t tile) {
    const int64_t i0 = tile * CE_TILE + (int64_t)t * CE_V;
#pragma unroll
    for (int v = 0; v < CE_V; ++v) nx[v] = i0 + v < N ? beta[i0 + v] : 0.0;
  };
  if (ntile > 0) fetch(0);
  for (int64_t k = 0; k < ntile; ++k) {
    double x[CE_V];
#pragma unroll
    for (int v = 0; v < CE_V; ++v) x[v] = DIV ? __ddiv_rn(nx[v], tot) : nx[v];
    if (k + 1 < ntile) fetch(k + 1);  // in flight under this tile's scan
    const int64_t i0 = k * CE_TILE + (int64_t)t * CE_V;
    const int cnt = (int)min((int64_t)CE_TILE, N - k * CE_TILE);
    // S in [2^e, 2^(e+1)): scale = 2^(52-e), u = 2^(e-52)
    const long long sb = __double_as_longlong(S);
    const int e = (int)((sb >> 52) & 0x7ff) - 1023;
    bool bad = !(S > 0.0) || e < -900 || e > 900;
    const double scale = __longlong_as_double((long long)(1023 + 52 - (bad ? 0 : e)) << 52);
    const double u = __longlong_as_double((long long)(1023 - 52 + (bad ? 0 : e)) << 52);
    const long long K = bad ? 0 : (long long)(S * scale);
    long long pre[CE_V], run = 0;
#pragma unroll
    for (int v = 0; v < CE_V; ++v) {
      const double xs = x[v] * scale;  // exact: a power of two, no overflow below
      if (!(xs >= 0.0) || !(xs < 9007199254740992.0)) bad = true;
      const double fl = floor(xs), fr = xs - fl;
      if (fr == 0.5) bad = true;
      run += bad ? 0 : (long long)fl + (fr > 0.5 ? 1 : 0);
      pre[v] = run;
    }
    // block scan of the per-thread sums
    long long inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    const int anybad = __syncthreads_or(bad ? 1 : 0);
    long long base = 0, all = 0;
#pragma unroll 1
    for (int w = 0; w < CE_T / 32; ++w) {
      const long long y = wsum[w];
      if (w < warp) base += y;
      all += y;
    }
    const bool exact = !anybad && all >= 0 && K + all < 9007199254740992LL && all < 9007199254740992LL;
    if (exact) {
      const long long off = K + base + (inc - run);
      if (DIV) {
#pragma unroll
        for (int v = 0; v < CE_V; ++v)
          if (i0 + v < N) cum[i0 + v] = (double)(off + pre[v]) * u;
      }
      S = (double)(K + all) * u;
      __syncthreads();  // wsum is rewritten by the next tile
    } else {
#pragma unroll
      for (int v = 0; v < CE_V; ++v) xbuf[t * CE_V + v] = x[v];
      __syncthreads();
      if (t == 0) {
        double r = S;
        for (int j = 0; j < cnt; ++j) {
          r = __dadd_rn(r, xbuf[j]);
          xbuf[j] = r;
        }
        *s_S = r;
      }
      __syncthreads();
      S = *s_S;
      if (DIV) {
#pragma unroll
        for (int v = 0; v < CE_V; ++v)
          if (i0 + v < N) cum[i0 + v] = xbuf[t * CE_V + v];
      }
      __syncthreads();
    }
  }
  return S;
}

// dynamic shared memory: CE_TILE doubles (the in-order fallback's tile) [+ padding that reserves the SM]
__global__ void __launch_bounds__(CE_T) cumulative_exact_kernel(const double* __restrict__ beta, int64_t N,
                                                                 double* __restrict__ cum,
                                                                 double* __restrict__ total_out) {
  extern __shared__ __align__(16) unsigned char ce_smem[];
  double* xbuf = reinterpret_cast<double*>(ce_smem);
  __shared__ long long wsum[CE_T / 32];
  __shared__ double s_S;
  const double tot = cum_exact_chain<false>(beta, N, 0.0, nullptr, xbuf, wsum, &s_S);  // svrg.cpp:92-94
  cum_exact_chain<true>(beta, N, tot, cum, xbuf, wsum, &s_S);                          // svrg.cpp:95-104
  __syncthreads();
  if (threadIdx.x == 0 && N > 0) {
    cum[N - 1] = 1.0;
    *total_out = tot;
  }
}

// inv_nq_i = total / (N * beta_i)  (svrg.cpp:167-172)
__global__ void inv_nq_kernel(const double* __restrict__ beta, int64_t N,
                              const double* __restrict__ total, double* __restrict__ inv_nq) {
  const double t = *total;
  const double Nd = (double)N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x)
    inv_nq[i] = __ddiv_rn(t, __dmul_rn(Nd, beta[i]));
}

// lookup_index (svrg.cpp:122-126): std::lower_bound, clamped to N-1.
__global__ void lower_bound_kernel(const double* __restrict__ cum, int64_t N,
                                   const double* __restrict__ u, int64_t count,
                                   int64_t* __restrict__ idx) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const double x = u[t];
    int64_t lo = 0, len = N;
    while (len > 0) {
      const int64_t half = len >> 1;
      if (cum[lo + half] < x) {
        lo += half + 1;
        len -= half + 1;
      } else {
        len = half;
      }
    }
    idx[t] = lo == N ? N - 1 : lo;
  }
}

// ---------------------------------------------------------------------------
// K10: one epoch of the inner loop in ONE persistent CTA.
//
// Thread t owns columns [t*VEC, t*VEC+VEC) of w, the snapshot, mu and the
// running sum, all in registers.  The epoch's indices are known in advance,
// so rows are prefetched DEPTH steps ahead with cp.async into a per-thread
// shared-memory ring (each thread copies and later reads only its own
// columns, so the ring needs no barrier); per-step scalars (index, inv_nq,
// label) are gathered in chunks.  Per step: two dots (w, snapshot) -> one
// block reduction (shuffles + one __syncthreads) -> the update
//   dir = (g(w) - g(snap)) * inv_nq + mu,  w -= eta * dir,  sum += w
// (svrg.cpp:37-43, :142-150).
constexpr int K10_DEPTH = 8;
constexpr int K10_CHUNK = 512;

__device__ __forceinline__ void cp_async_bytes16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_bytes8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_bytes4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BYTES>
__device__ __forceinline__ void cp_async_span(void* smem, const void* gmem) {
  if constexpr (BYTES % 16 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 16; ++c)
      cp_async_bytes16(static_cast<char*>(smem) + 16 * c, static_cast<const char*>(gmem) + 16 * c);
  } else if constexpr (BYTES % 8 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 8; ++c)
      cp_async_bytes8(static_cast<char*>(smem) + 8 * c, static_cast<const char*>(gmem) + 8 * c);
  } else {
#pragma unroll
    for (int c = 0; c < BYTES / 4; ++c)
      cp_async_bytes4(static_cast<char*>(smem) + 4 * c, static_cast<const char*>(gmem) + 4 * c);
  }
}

struct EpochArgs {
  const void* Xt;            // n_total x ld rows of dtype T (data components)
  const double* B;           // d x ld rows (regulariser components)
  int64_t ld, n, N;
  const double* y;           // n labels
  const double* inv_nq;      // N
  double data_coef, reg_coef;
  const int64_t* idx;        // m indices
  int64_t m;
  double eta;
  const double* snapshot;    // ld
  const double* mu;          // ld
  double* w_avg;             // ld
};

template <class T, int VEC, int NT>
__global__ void __launch_bounds__(NT, 1) svrg_epoch_kernel(EpochArgs a) {
  constexpr int NW = NT / 32;
  constexpr int SLOT = NT * VEC;  // doubles per ring slot (fits an fp64 B row)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);                      // DEPTH * SLOT
  int64_t* s_idx = reinterpret_cast<int64_t*>(ring + K10_DEPTH * SLOT);     // CHUNK + DEPTH
  double* s_q = reinterpret_cast<double*>(s_idx + K10_CHUNK + K10_DEPTH);  // CHUNK
  double* s_y = s_q + K10_CHUNK;                                            // CHUNK
  __shared__ double2 red[2][NW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = (int64_t)tid * VEC;
  const bool active = c0 < a.ld;
  const T* Xt = static_cast<const T*>(a.Xt);

  double w[VEC], ws[VEC], mu[VEC], sum[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    ws[v] = active ? a.snapshot[c0 + v] : 0.0;
    w[v] = ws[v];
    mu[v] = active ? a.mu[c0 + v] : 0.0;
    sum[v] = 0.0;
  }

  auto issue = [&](int64_t step, int64_t i) {  // prefetch row of component i into slot
    double* slot = ring + (step % K10_DEPTH) * SLOT + (int64_t)tid * VEC;
    if (active) {
      if (i < a.n) cp_async_span<VEC * (int)sizeof(T)>(slot, Xt + i * a.ld + c0);
      else cp_async_span<VEC * 8>(slot, a.B + (i - a.n) * a.ld + c0);
    }
    cp_async_commit();
  };
  auto load_chunk = [&](int64_t t0) {  // indices [t0, t0+CHUNK+DEPTH), scalars [t0, t0+CHUNK)
    __syncthreads();
    for (int e = tid; e < K10_CHUNK + K10_DEPTH; e += NT) {
      const int64_t t = t0 + e;
      s_idx[e] = t < a.m ? a.idx[t] : 0;
    }
    __syncthreads();
    for (int e = tid; e < K10_CHUNK; e += NT) {
      const int64_t i = s_idx[e];
      s_q[e] = a.inv_nq[i];
      s_y[e] = i < a.n ? a.y[i] : 0.0;
    }
    __syncthreads();
  };

  load_chunk(0);
  for (int s = 0; s < K10_DEPTH; ++s) {
    if (s < a.m) issue(s, s_idx[s]);
    else cp_async_commit();
  }
  int par = 0;
  for (int64_t t = 0; t < a.m; ++t) {
    const int e = (int)(t % K10_CHUNK);
    if (e == 0 && t > 0) load_chunk(t);
    const int64_t i = s_idx[e];
    cp_async_wait<K10_DEPTH - 1>();  // this thread's copy for step t has landed
    const double* slot = ring + (t % K10_DEPTH) * SLOT + (int64_t)tid * VEC;
    double x[VEC];
    if (i < a.n) {
      const T* xs = reinterpret_cast<const T*>(slot);
#pragma unroll
      for (int v = 0; v < VEC; ++v) x[v] = active ? (double)xs[v] : 0.0;
    } else {
#pragma unroll
      for (int v = 0; v < VEC; ++v) x[v] = active ? slot[v] : 0.0;
    }
    double p1 = 0.0, p2 = 0.0;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      p1 = fma(x[v], w[v], p1);
      p2 = fma(x[v], ws[v], p2);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      p1 += __shfl_xor_sync(0xffffffffu, p1, off);
      p2 += __shfl_xor_sync(0xffffffffu, p2, off);
    }
    if (lane == 0) red[par][warp] = make_double2(p1, p2);
    // refill the ring slot consumed DEPTH steps from now (slot of step t is
    // reused for step t+DEPTH; this thread has already read its part into x[])
    {
      const int64_t tn = t + K10_DEPTH;
      if (tn < a.m) issue(tn, s_idx[e + K10_DEPTH]);
      else cp_async_commit();
    }
    __syncthreads();
    double d1 = 0.0, d2 = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      const double2 r = red[par][q];
      d1 += r.x;
      d2 += r.y;
    }
    par ^= 1;
    const double coef = i < a.n ? a.data_coef : a.reg_coef;
    const double yi = s_y[e];
    const double q = s_q[e];
    const double g1 = coef * (d1 - yi), g2 = coef * (d2 - yi);
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const double dir = (g1 * x[v] - g2 * x[v]) * q + mu[v];
      w[v] = fma(-a.eta, dir, w[v]);
      sum[v] += w[v];
    }
  }
  cp_async_wait<0>();
  if (active) {
    const double inv_m = 1.0 / (double)a.m;
#pragma unroll
    for (int v = 0; v < VEC; ++v) a.w_avg[c0 + v] = sum[v] * inv_m;
  }
}

template <class T, int VEC, int NT>
size_t svrg_epoch_smem() {
  return (size_t)K10_DEPTH * NT * VEC * 8 + (K10_CHUNK + K10_DEPTH) * 8 + 2 * K10_CHUNK * 8;
}

}  // namespace skr
