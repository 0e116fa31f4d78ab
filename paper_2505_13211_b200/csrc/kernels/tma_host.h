// Host-side TMA tensor-map construction. The driver entry point is resolved
// through the runtime so the library does not link libcuda directly.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace magi {

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult status;
    cudaError_t err =
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &status);
    if (err != cudaSuccess || status != cudaDriverEntryPointSuccess || ptr == nullptr) {
      throw std::runtime_error("cannot resolve cuTensorMapEncodeTiled");
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }();
  return fn;
}

// bf16 tensor of `rank` dims (dim 0 innermost, contiguous), 128B swizzle.
// strides_bytes[i] is the stride of dim i+1. box[0] * 2 must be <= 128.
inline CUtensorMap make_tmap_bf16(const void* base, int rank, const uint64_t* dims,
                                  const uint64_t* strides_bytes, const uint32_t* box,
                                  CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap map;
  uint32_t elem_strides[5] = {1, 1, 1, 1, 1};
  CUresult r = tensor_map_encoder()(
      &map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, static_cast<cuuint32_t>(rank),
      const_cast<void*>(base), reinterpret_cast<const cuuint64_t*>(dims),
      reinterpret_cast<const cuuint64_t*>(strides_bytes),
      reinterpret_cast<const cuuint32_t*>(box), elem_strides, CU_TENSOR_MAP_INTERLEAVE_NONE,
      swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw std::runtime_error("cuTensorMapEncodeTiled failed with code " + std::to_string(r));
  }
  return map;
}

// [rows, cols] f32 matrix (row stride cols * 4 bytes, must be a multiple of
// 16), box = box_cols x 1, no swizzle. Used for per-row lse / delta vectors.
inline CUtensorMap make_tmap_f32_rows(const void* base, uint64_t rows, uint64_t cols,
                                      uint32_t box_cols) {
  CUtensorMap map;
  const uint64_t dims[2] = {cols, rows};
  const uint64_t strides[1] = {cols * 4};
  const uint32_t box[2] = {box_cols, 1};
  const uint32_t elem_strides[2] = {1, 1};
  CUresult r = tensor_map_encoder()(
      &map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base),
      reinterpret_cast<const cuuint64_t*>(dims), reinterpret_cast<const cuuint64_t*>(strides),
      reinterpret_cast<const cuuint32_t*>(box), elem_strides, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    throw std::runtime_error("cuTensorMapEncodeTiled (f32 rows) failed with code " + std::to_string(r));
  }
  return map;
}

// [tokens, heads, dim] token-major bf16 tensor viewed as 3-D (dim, heads, tokens);
// one box = box_rows tokens x 64 dims of one head.
inline CUtensorMap make_tmap_thd(const void* base, int64_t tokens, int64_t heads, int64_t dim,
                                 uint32_t box_rows) {
  const uint64_t dims[3] = {static_cast<uint64_t>(dim), static_cast<uint64_t>(heads),
                            static_cast<uint64_t>(tokens)};
  const uint64_t strides[2] = {static_cast<uint64_t>(dim) * 2,
                               static_cast<uint64_t>(heads * dim) * 2};
  const uint32_t box[3] = {64, 1, box_rows};
  return make_tmap_bf16(base, 3, dims, strides, box);
}

}  // namespace magi
