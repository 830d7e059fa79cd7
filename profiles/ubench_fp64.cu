// Micro-benchmarks behind the K10 chain design (one warp unless stated):
//  1. DFMA dependent-chain latency, 2. DFMA issue rate (8 independent chains),
//  3. LDS.64 dependent latency, 4. one warp-wide shuffle-add (fp64) latency,
//  5. cluster ping-pong: st.async + mbarrier complete_tx round trip between two
//     CTAs of a cluster (half of it = one-way exchange latency).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp64 profiles/ubench_fp64.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__global__ void k_dfma(double* out, long long* cyc, double a, double b) {
  double x = threadIdx.x * 1e-3, y[8];
  for (int k = 0; k < 8; ++k) y[k] = x + k;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 1000; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) x = fma(x, a, b);  // dependent
  }
  long long t1 = clock64();
#pragma unroll 1
  for (int it = 0; it < 1000; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) y[r] = fma(y[r], a, b);  // 8 independent chains
  }
  long long t2 = clock64();
  double s = x;
  for (int k = 0; k < 8; ++k) s += y[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
}

__global__ void k_lds(double* out, long long* cyc) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)((i * 7 + 1) % 1024);
  __syncthreads();
  double v = sm[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 1000; ++it) v = sm[((int)v + threadIdx.x) & 1023];
  long long t1 = clock64();
  double a = threadIdx.x;
#pragma unroll 1
  for (int it = 0; it < 1000; ++it) a += __shfl_xor_sync(0xffffffffu, a, 1);
  long long t2 = clock64();
  out[threadIdx.x] = v + a;
  if (threadIdx.x == 0) {
    cyc[2] = t1 - t0;
    cyc[3] = t2 - t1;
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// two-CTA cluster ping-pong through st.async + complete_tx
__global__ void __cluster_dims__(2, 1, 1) k_ping(long long* cyc, int iters) {
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) double slot;
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  if (threadIdx.x == 0) {
    uint32_t rd, rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rd) : "r"(smem_u32(&slot)), "r"(1 - r));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(smem_u32(&bar)), "r"(1 - r));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8;" ::"r"(smem_u32(&bar)) : "memory");
      if (r == 0 || it > 0) {
        // rank 0 starts; rank 1 answers after receiving
      }
      if (r == 0) {
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rd),
                     "l"((long long)it), "r"(rb) : "memory");
      }
      asm volatile(
          "{\n.reg .pred P1;\nW1:\n"
          "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
          "@!P1 bra W1;\n}\n" ::"r"(smem_u32(&bar)), "r"((uint32_t)(it & 1)) : "memory");
      if (r == 1) {
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rd),
                     "l"((long long)it), "r"(rb) : "memory");
      }
    }
    long long t1 = clock64();
    if (r == 0) cyc[4] = t1 - t0;
  }
  cl.sync();
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  for (int nt : {32, 64, 128, 256, 512}) {
    k_dfma<<<1, nt>>>(out, cyc, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
    printf("threads %d: DFMA dependent %.2f cyc, 8-chain issue %.2f cyc per warp-DFMA (SM: %.1f lanes/clk)\n", nt,
           cyc[0] / 8000.0, cyc[1] / 8000.0, nt / (cyc[1] / 8000.0));
  }
  k_lds<<<1, 32>>>(out, cyc);
  k_ping<<<2, 32>>>(cyc, 1000);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\n", cudaGetErrorString(e));
  printf("DFMA dependent latency: %.2f cyc\n", cyc[0] / 8000.0);
  printf("DFMA issue, 8 independent chains (one warp): %.2f cyc per DFMA\n", cyc[1] / 8000.0);
  printf("LDS.64 dependent latency (incl. int convert): %.2f cyc\n", cyc[2] / 1000.0);
  printf("SHFL.64 + DADD dependent: %.2f cyc\n", cyc[3] / 1000.0);
  printf("st.async ping-pong round trip: %.1f cyc (one-way %.1f)\n", cyc[4] / 1000.0, cyc[4] / 2000.0);
  return 0;
}
