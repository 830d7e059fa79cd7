// Micro-benchmark of the K10 chain's per-block warp work in isolation (one CTA,
// no cluster): the dot-warp loop (lanes = rows, 32 swizzled columns per lane,
// 8 FMA chains) and the update-warp loop (thread = column, 32 rows, two rank-L
// FMA chains), alone and concurrently, plus DSMEM fan-out variants in a
// 16-CTA cluster (st.async 8 B x 32 lanes per rank, 16 B x 16 lanes per rank,
// one 16-B store per rank from 16 lanes (reduce-scatter shape), and a
// 256-B bulk copy shared::cta -> shared::cluster per rank).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o profiles/ubench_chain profiles/ubench_chain.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int SW = 64, L = 32, ITERS = 2000;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode bit 0: dot warps run; bit 1: update warps run
__global__ void k_work(double* out, long long* cyc, int mode) {
  __shared__ __align__(16) double rows[L * SW];
  __shared__ __align__(16) double w[SW];
  __shared__ __align__(16) double dd[L], ee[L];
  for (int i = threadIdx.x; i < L * SW; i += blockDim.x) rows[i] = 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < SW; i += blockDim.x) w[i] = 1.0 + i;
  for (int i = threadIdx.x; i < L; i += blockDim.x) dd[i] = ee[i] = 0.5 / (1 + i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double res = 0;
  long long t0 = clock64();
  if (warp < 2) {
    if (mode & 1) {
      const int l = lane, lsw = l & 15, c0 = warp * 32;
      for (int it = 0; it < ITERS; ++it) {
        const double* x = rows + l * SW + c0;
        double xv[32], wv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) xv[j] = x[(j & ~15) + ((j & 15) ^ lsw)];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const double2 q = *reinterpret_cast<const double2*>(w + c0 + j);
          wv[j] = q.x;
          wv[j + 1] = q.y;
        }
        double acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = xv[j] * wv[j];
#pragma unroll
        for (int j = 8; j < 32; ++j) acc[j & 7] = fma(xv[j], wv[j], acc[j & 7]);
        res += ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        __syncwarp();
      }
    }
  } else if (warp < 4) {
    if (mode & 2) {
      const int t = threadIdx.x - 64;
      double wr = 0, S = 0;
      for (int it = 0; it < ITERS; ++it) {
        double xr[L];
#pragma unroll
        for (int l = 0; l < L; ++l) xr[l] = rows[l * SW + (t ^ (l & 15))];
        double u0 = 0, u1 = 0, u2 = 0, u3 = 0, v0 = 0, v1 = 0, v2 = 0, v3 = 0;
#pragma unroll
        for (int l = 0; l < L; l += 4) {
          const double4 dq = *reinterpret_cast<const double4*>(dd + l);
          const double4 eq = *reinterpret_cast<const double4*>(ee + l);
          u0 = fma(dq.x, xr[l], u0); u1 = fma(dq.y, xr[l + 1], u1); u2 = fma(dq.z, xr[l + 2], u2); u3 = fma(dq.w, xr[l + 3], u3);
          v0 = fma(eq.x, xr[l], v0); v1 = fma(eq.y, xr[l + 1], v1); v2 = fma(eq.z, xr[l + 2], v2); v3 = fma(eq.w, xr[l + 3], v3);
        }
        const double u = (u0 + u1) + (u2 + u3), vv = (v0 + v1) + (v2 + v3);
        S += wr - 1e-3 * vv;
        wr = wr - 1e-3 * u;
        __syncwarp();
      }
      res = wr + S;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = res;
  if (lane == 0) cyc[warp] = t1 - t0;
}

// DSMEM fan-out in a 16-CTA cluster: every CTA sends 32 doubles to every rank
// (variant 0: 16 x st.async.b64 from 32 lanes; 1: 16 x st.async.v2.b64 from 16
// lanes; 2: reduce-scatter shape — ONE st.async.v2 instruction, lane q -> rank q;
// 3: bulk copy 256 B per rank from one lane), and waits for its own 16 x 256 B
// (variant 2: 16 x 16 B).  Measures cycles per round (CTA 0).
__global__ void k_fan(long long* cyc, int variant, int iters) {
  __shared__ __align__(16) double inbox[2][16 * 32];
  __shared__ __align__(16) double src[32];
  __shared__ __align__(8) uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int lane = threadIdx.x & 31;
  const int CS = (int)cl.num_blocks();
  const uint32_t bytes = variant == 2 ? CS * 16 : CS * 256;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < 2; ++s)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(bytes)
                   : "memory");
  }
  if (threadIdx.x < 32) src[threadIdx.x] = r + 0.01 * threadIdx.x;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cl.sync();
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    for (int it = 0; it < iters; ++it) {
      const int s = it & 1;
      const double v = src[lane] + it;
      const uint32_t mybar = smem_u32(&bar[s]);
      if (variant == 0) {
#pragma unroll
        for (int q = 0; q < CS; ++q) {
          uint32_t rd, rb;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(smem_u32(&inbox[s][r * 32 + lane])), "r"(q));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(mybar), "r"(q));
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rd),
                       "l"(__double_as_longlong(v)), "r"(rb) : "memory");
        }
      } else if (variant == 1) {
        const double vn = __shfl_down_sync(0xffffffffu, v, 1);
        if ((lane & 1) == 0) {
#pragma unroll
          for (int q = 0; q < CS; ++q) {
            uint32_t rd, rb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(smem_u32(&inbox[s][r * 32 + lane])), "r"(q));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(mybar), "r"(q));
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(rd),
                         "l"(__double_as_longlong(v)), "l"(__double_as_longlong(vn)), "r"(rb) : "memory");
          }
        }
      } else if (variant == 2) {
        const double vn = __shfl_down_sync(0xffffffffu, v, 1);
        if (lane < CS) {
          uint32_t rd, rb;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(smem_u32(&inbox[s][r * 2])), "r"(lane));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(mybar), "r"(lane));
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(rd),
                       "l"(__double_as_longlong(v)), "l"(__double_as_longlong(vn)), "r"(rb) : "memory");
        }
      } else if (variant == 4) {
        // transposed: instruction k, lane q -> rank q, pair k (16 B)
        if (lane < CS) {
          uint32_t rb;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(mybar), "r"(lane));
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            uint32_t rd;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(smem_u32(&inbox[s][r * 32 + 2 * k])), "r"(lane));
            const double2 pv = *reinterpret_cast<const double2*>(src + 2 * k);
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(rd),
                         "l"(__double_as_longlong(pv.x + it)), "l"(__double_as_longlong(pv.y)), "r"(rb) : "memory");
          }
        }
      } else if (variant == 5) {
        // transposed 8 B: lane = (rank q = lane % CS, part h = lane / CS), 32 / (32 / CS) values each
        const int q = lane % CS, h = lane / CS, per = 32 / (32 / CS);
        uint32_t rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(mybar), "r"(q));
        for (int k = 0; k < per; ++k) {
          const int e = h * per + k;
          uint32_t rd;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(smem_u32(&inbox[s][r * 32 + e])), "r"(q));
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rd),
                       "l"(__double_as_longlong(src[e] + it)), "r"(rb) : "memory");
        }
      } else {
        if (lane == 0) {
          for (int q = 0; q < CS; ++q) {
            uint32_t rd, rb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(smem_u32(&inbox[s][r * 32])), "r"(q));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(mybar), "r"(q));
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];" ::"r"(rd),
                "r"(smem_u32(src)), "r"(rb)
                : "memory");
          }
        }
      }
      // wait for this round's inbound bytes, then re-arm the slot for round it + 2
      asm volatile(
          "{\n.reg .pred P1;\nWF:\n"
          "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
          "@!P1 bra WF;\n}\n" ::"r"(mybar), "r"((uint32_t)((it >> 1) & 1)) : "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mybar), "r"(bytes) : "memory");
      // keep ranks within one round of each other (a slot is re-armed before peers reuse it)
      __syncwarp();
      asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
    }
  }
  long long t1 = clock64();
  if (r == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
  cl.sync();
}

// Reference: the cluster barrier alone per round
__global__ void k_clbar(long long* cyc, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
  long long t1 = clock64();
  if (cl.block_rank() == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* names[] = {"", "dots only", "update only", "dots + update"};
  for (int mode = 1; mode <= 3; ++mode) {
    for (int k = 0; k < 8; ++k) cyc[k] = 0;
    k_work<<<1, 192>>>(out, cyc, mode);
    cudaDeviceSynchronize();
    printf("%-14s: dot warp %.1f cyc/iter, update warp %.1f cyc/iter\n", names[mode], cyc[0] / (double)ITERS,
           cyc[2] / (double)ITERS);
  }
  const int iters = 2000;
  cudaFuncSetAttribute(k_clbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_fan, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* vn[] = {"st.async b64 x32 lanes per rank", "st.async v2.b64 x16 lanes per rank",
                      "st.async v2.b64, lane q -> rank q (one instr)", "bulk copy 256 B per rank (one lane)",
                      "transposed v2: lane q -> rank q, 16 instrs", "transposed b64: lane -> rank lane % CS"};
  for (int CS : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(32);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cyc[0] = 0;
    cudaLaunchKernelEx(&cfg, k_clbar, cyc, iters);
    cudaError_t e = cudaDeviceSynchronize();
    const double clbar = cyc[0] / (double)iters;
    printf("CS=%2d cluster barrier alone: %.1f cyc/round %s\n", CS, clbar, cudaGetErrorString(e));
    for (int v = 0; v < 6; ++v) {
      cyc[0] = 0;
      cudaLaunchKernelEx(&cfg, k_fan, cyc, v, iters);
      e = cudaDeviceSynchronize();
      printf("CS=%2d fan-out %-46s: %.1f cyc/round (%.1f beyond the barrier)  %s\n", CS, vn[v], cyc[0] / (double)iters,
             cyc[0] / (double)iters - clbar, cudaGetErrorString(e));
    }
  }
  return 0;
}
