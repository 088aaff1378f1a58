// Thread-written shared-memory operand in the MN-major, 128B-swizzled canonical UMMA layout.
//
// Used for a [128 (M) x 128 (K)] bf16 A operand that threads produce row-by-row along K
// (e.g. dS^T held by KV-row threads, consumed as dS with M = query rows):
//   M is split into 2 atoms of 64 elements (128 B per K-row), LBO = 16 KB between M atoms;
//   K is split into 16 groups of 8 rows, SBO = 1 KB between groups;
//   inside a 1 KB atom, 16-byte chunk c of K-row r is stored at chunk (c XOR r).
#pragma once
#include "sm100_ptx.cuh"

namespace fpdt {

// Byte offset of the 8-element (16 B) chunk holding A[m .. m+7][k], m % 8 == 0.
__device__ __forceinline__ uint32_t mn_sw128_offset(int m, int k) {
  return (uint32_t)((m >> 6) * 16384 + (k >> 3) * 1024 + (k & 7) * 128 + ((((m & 63) >> 3) ^ (k & 7)) << 4));
}
__device__ __forceinline__ uint64_t desc_a_mn_sw128(uint32_t base, int kk) {
  return ptx::smem_desc(base + kk * 2048, 16384, 1024, ptx::kSw128);
}
// The same bytes read as a K-major A operand [128 (M) x 128 (K)] with M = the former K index (rows of 128 B,
// 8-row groups 1 KB apart, the two 64-element K atoms 16 KB apart): contraction step kk = 16 elements.
__device__ __forceinline__ uint64_t desc_a_kmajor_sw128(uint32_t base, int kk) {
  return ptx::smem_desc(base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, ptx::kSw128);
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, const uint32_t (&w)[4]) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
               : "memory");
}

}  // namespace fpdt
