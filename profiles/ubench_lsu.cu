// Shared-memory / shuffle / FP64 issue costs on B200 (cycles per warp-instruction),
// for 1..16 concurrent warps of one CTA: the cost model behind the K10 chain layout.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o profiles/ubench_lsu profiles/ubench_lsu.cu
#include <cstdint>
#include <cstdio>

constexpr int N = 64;  // independent ops per iteration
constexpr int IT = 200;

template <int KIND>
__global__ void k(double* out, long long* cyc, int active_warps) {
  __shared__ __align__(16) double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1e-3 * (i & 255);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long bits[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // integer sinks: keep the FP64 pipe out of LDS timings
  long long t0 = clock64();
  if (warp < active_warps) {
    const int base = (warp * 256) & 2047;
    for (int it = 0; it < IT; ++it) {
      const int rot = (it & 7) * 32;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if (KIND == 0) {  // LDS.64 distinct, conflict-free
          bits[j & 7] ^= __double_as_longlong(sm[base + ((j * 32 + lane + rot) & 255)]);
        } else if (KIND == 1) {  // LDS.128 distinct, conflict-free
          const double2 v = *reinterpret_cast<const double2*>(sm + 2 * ((base / 2 + j * 32 + lane + rot) & 2047));
          bits[j & 7] ^= __double_as_longlong(v.x) ^ __double_as_longlong(v.y);
        } else if (KIND == 2) {  // LDS.128 broadcast
          const double2 v = *reinterpret_cast<const double2*>(sm + 2 * ((j + it) & 63));
          bits[j & 7] ^= __double_as_longlong(v.x) ^ __double_as_longlong(v.y);
        } else if (KIND == 3) {  // LDS.64 broadcast
          bits[j & 7] ^= __double_as_longlong(sm[(j + it) & 255]);
        } else if (KIND == 4) {  // SHFL of a double (2 x SHFL.32)
          acc[j & 7] = __shfl_xor_sync(0xffffffffu, acc[j & 7] + 1.0, j & 31);
        } else {  // DFMA independent (8 chains)
          acc[j & 7] = fma(acc[j & 7], 1.0000001, 1e-9);
        }
      }
      __syncwarp();
    }
  }
  for (int j = 0; j < 8; ++j) acc[j] += (double)(bits[j] & 1023);
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < 8; ++j) s += acc[j];
  out[threadIdx.x] = s;
  if (lane == 0) cyc[warp] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 32 * sizeof(long long));
  const char* names[] = {"LDS.64 distinct", "LDS.128 distinct", "LDS.128 broadcast", "LDS.64 broadcast",
                         "SHFL f64 (+DADD)", "DFMA independent"};
  void (*ks[])(double*, long long*, int) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>};
  for (int kind = 0; kind < 6; ++kind) {
    printf("%-20s", names[kind]);
    for (int aw : {1, 2, 4, 8, 16}) {
      ks[kind]<<<1, 512>>>(out, cyc, aw);
      cudaDeviceSynchronize();
      printf("  %2dw: %6.2f", aw, cyc[0] / (double)(IT * N));
    }
    printf("   cyc per warp-instr (warp 0)\n");
  }
  return 0;
}
