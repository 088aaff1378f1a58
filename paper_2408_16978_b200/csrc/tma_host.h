// Host-side TMA tensor-map construction (driver entry point fetched at runtime, no -lcuda needed).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fpdt {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Tensor map over a bf16 tensor [rows][heads][head_dim] (row-major, head_dim contiguous).
// Box = {box_cols, 1, box_rows}: one head, `box_rows` tokens, `box_cols` dims starting at a column offset.
// swizzle: CU_TENSOR_MAP_SWIZZLE_128B for 64-column boxes, _32B for 16-column boxes.
inline bool make_tmap_rows_heads_dim(CUtensorMap* m, const void* base, uint64_t rows, uint32_t heads,
                                     uint32_t head_dim, uint32_t box_cols, uint32_t box_rows,
                                     CUtensorMapSwizzle swizzle) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {head_dim, heads, rows};
  cuuint64_t strides[2] = {(cuuint64_t)head_dim * 2, (cuuint64_t)heads * head_dim * 2};
  cuuint32_t box[3] = {box_cols, 1, box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Tensor map of the attention operand tiles (attn_tile.cuh): box = one swizzle atom of 128 rows.
template <int D>
inline bool make_tile_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint32_t heads) {
  if (D == 80) return make_tmap_rows_heads_dim(m, base, rows, heads, D, 16, 128, CU_TENSOR_MAP_SWIZZLE_32B);
  return make_tmap_rows_heads_dim(m, base, rows, heads, D, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Tensor map over an fp32 tensor [rows][heads][head_dim] (used for TMA reduce-add into the dq accumulator);
// swizzled boxes let threads that own one row each stage a tile without shared-memory bank conflicts.  Box = {box_cols, 1, box_rows}.
inline bool make_tmap_f32_rows_heads_dim(CUtensorMap* m, const void* base, uint64_t rows, uint32_t heads,
                                         uint32_t head_dim, uint32_t box_cols, uint32_t box_rows,
                                         CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_NONE) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {head_dim, heads, rows};
  cuuint64_t strides[2] = {(cuuint64_t)head_dim * 4, (cuuint64_t)heads * head_dim * 4};
  cuuint32_t box[3] = {box_cols, 1, box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Tensor map over a head-major fp32 tensor [heads][head_stride/head_dim rows][head_dim] (the dq accumulator):
// coordinates (col, row, head); box = {box_cols, box_rows, 1}.
inline bool make_tmap_f32_head_major(CUtensorMap* m, const void* base, uint64_t rows, uint32_t heads,
                                     uint32_t head_dim, uint64_t head_stride, uint32_t box_cols, uint32_t box_rows,
                                     CUtensorMapSwizzle swizzle) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {head_dim, rows, heads};
  cuuint64_t strides[2] = {(cuuint64_t)head_dim * 4, (cuuint64_t)head_stride * 4};
  cuuint32_t box[3] = {box_cols, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace fpdt
