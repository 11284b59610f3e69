// tma.h — host-side TMA tensor-map construction (driver entry point resolved
// at runtime, so the library does not hard-link a specific libcuda symbol set).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.h"

namespace mrsp {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    MRSP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    MRSP_REQUIRE(p != nullptr, MRSP_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 2-D bf16 tensor [rows][cols] with row pitch `ld` elements; box = box_rows x
// box_cols (box_cols * 2 bytes must equal the swizzle span for SWIZZLE_128B).
inline CUtensorMap make_tmap_bf16_2d(const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                                     uint32_t box_rows, uint32_t box_cols,
                                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  MRSP_REQUIRE((ld * 2) % 16 == 0, MRSP_INVALID_ARGUMENT,
               "TMA: row pitch must be a multiple of 16 bytes");
  MRSP_REQUIRE(reinterpret_cast<uintptr_t>(base) % 16 == 0, MRSP_INVALID_ARGUMENT,
               "TMA: base must be 16-byte aligned");
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t elem[2] = {1, 1};
  CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                 dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MRSP_REQUIRE(r == CUDA_SUCCESS, MRSP_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
  return m;
}

// 3-D bf16 view of [rows][ld] as [rows][heads][hs] (head stride hs elements,
// row pitch ld): box = box_rows x 1 head x box_cols, so a box starting at
// column x of a head reads min(box_cols, hs - x) real columns and zero-fills
// the rest (heads narrower than the tile, e.g. hd 72 in 128-wide tiles).
inline CUtensorMap make_tmap_bf16_3d_heads(const void* base, uint64_t rows, uint64_t heads,
                                           uint64_t hs, uint64_t ld, uint32_t box_rows,
                                           uint32_t box_cols,
                                           CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  MRSP_REQUIRE((ld * 2) % 16 == 0 && (hs * 2) % 16 == 0, MRSP_INVALID_ARGUMENT,
               "TMA: row pitch and head stride must be multiples of 16 bytes");
  MRSP_REQUIRE(reinterpret_cast<uintptr_t>(base) % 16 == 0, MRSP_INVALID_ARGUMENT,
               "TMA: base must be 16-byte aligned");
  CUtensorMap m;
  cuuint64_t dims[3] = {hs, heads, rows};
  cuuint64_t strides[2] = {hs * 2, ld * 2};
  cuuint32_t box[3] = {box_cols, 1, box_rows};
  cuuint32_t elem[3] = {1, 1, 1};
  CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base),
                                 dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MRSP_REQUIRE(r == CUDA_SUCCESS, MRSP_CUDA_ERROR, "cuTensorMapEncodeTiled (3-D) failed");
  return m;
}

// 2-D fp32 tensor [rows][cols], row pitch `ld` elements (epilogue stores /
// reduce-adds of fp32 outputs and the residual stream).
inline CUtensorMap make_tmap_f32_2d(const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                                    uint32_t box_rows, uint32_t box_cols,
                                    CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  MRSP_REQUIRE((ld * 4) % 16 == 0, MRSP_INVALID_ARGUMENT,
               "TMA: row pitch must be a multiple of 16 bytes");
  MRSP_REQUIRE(reinterpret_cast<uintptr_t>(base) % 16 == 0, MRSP_INVALID_ARGUMENT,
               "TMA: base must be 16-byte aligned");
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t elem[2] = {1, 1};
  CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base),
                                 dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MRSP_REQUIRE(r == CUDA_SUCCESS, MRSP_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
  return m;
}

}  // namespace mrsp
