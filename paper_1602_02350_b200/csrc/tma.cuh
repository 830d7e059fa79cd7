// TMA tensor maps (host) and tile loads (device) shared by the GEMM kernels.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace skr {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    SKR_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) raise(SKR_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D tensor map over a row-major matrix (rows x cols, row stride ld elements of
// `esize` bytes), box = box_rows x box_cols, out-of-range elements read as zero.
inline CUtensorMap make_tmap_2d(const void* ptr, int esize, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                                int box_cols, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * (cuuint64_t)esize};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = encode_tiled()(&m, esize == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                    2, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(SKR_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// 2-D fp32 tensor map (tcgen05 GEMM): box = box_rows x box_cols (32 columns by default), 128-byte swizzle.
inline CUtensorMap make_tmap_f32(const float* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                                 CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B, int box_cols = 32) {
  return make_tmap_2d(ptr, 4, rows, cols, ld, box_rows, box_cols, swz);
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Byte offset of (row r, byte column cb) inside a TMA box with 128-byte rows and
// CU_TENSOR_MAP_SWIZZLE_128B: the 16-byte chunk index is XORed with r mod 8.
__device__ __forceinline__ uint32_t swz128(uint32_t r, uint32_t cb) {
  return r * 128u + ((((cb >> 4) ^ (r & 7u)) << 4) | (cb & 15u));
}

}  // namespace skr
