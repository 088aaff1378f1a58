// Shared-memory tile format of a [128 rows x D] bf16 operand tile (Q, K, V or dO) and its
// tcgen05 smem descriptors.
//
// A tile is loaded by TMA as D/64 boxes of [128 rows x 64 cols] with 128B swizzle (16 KB each,
// 1024B-aligned), plus, when D % 64 == 16 (D = 80), one box of [128 rows x 16 cols] with 32B
// swizzle (4 KB).  The same bytes serve as
//   * a K-major operand (rows = M or N, contraction over D)       -> desc_kmajor(kk)
//   * an MN-major operand (rows = contraction K, N = D columns)   -> desc_mnmajor_main/tail(kk)
// kk indexes 16-element contraction steps (UMMA_K = 16 for bf16).
#pragma once
#include "sm100_ptx.cuh"

namespace fpdt {

template <int D>
struct Tile {
  static_assert(D == 64 || D == 80 || D == 128, "head_dim must be 64, 80 or 128");
  static constexpr int kMain = D / 64;        // 128B-swizzled 64-column boxes
  static constexpr int kTail = D % 64;        // 0 or 16 (32B-swizzled box)
  static constexpr int kMainBytes = 128 * 64 * 2;
  static constexpr int kTailBytes = 128 * 16 * 2;
  static constexpr int kBytes = 128 * D * 2;  // whole tile
  static constexpr int kKSteps = D / 16;      // contraction steps when D is the K dimension
  static constexpr int kMainN = kMain * 64;   // N covered by the main region when D is the N dimension

  // K-major descriptor for contraction step kk over D (operand rows = 128).
  static __device__ __forceinline__ uint64_t desc_kmajor(uint32_t tile, int kk) {
    const int col = kk * 16;
    if (col < kMainN)
      return ptx::smem_desc(tile + (col >> 6) * kMainBytes + (col & 63) * 2, 16, 1024, ptx::kSw128);
    return ptx::smem_desc(tile + kMain * kMainBytes, 16, 256, ptx::kSw32);
  }
  // MN-major descriptors for contraction step kk over the 128 rows (N = D columns).
  static __device__ __forceinline__ uint64_t desc_mn_main(uint32_t tile, int kk) {
    return ptx::smem_desc(tile + kk * 2048, kMainBytes, 1024, ptx::kSw128);
  }
  static __device__ __forceinline__ uint64_t desc_mn_tail(uint32_t tile, int kk) {
    return ptx::smem_desc(tile + kMain * kMainBytes + kk * 512, 512, 256, ptx::kSw32);
  }
  // Issue the TMA loads of rows [row0, row0+128) of head `head` into `tile` (bytes = kBytes).
  static __device__ __forceinline__ void load(uint32_t tile, const CUtensorMap* m_main, const CUtensorMap* m_tail,
                                              uint32_t bar, int head, int row0, uint64_t policy) {
#pragma unroll
    for (int a = 0; a < kMain; ++a) ptx::tma_load_3d(tile + a * kMainBytes, m_main, bar, a * 64, head, row0, policy);
    if constexpr (kTail) ptx::tma_load_3d(tile + kMain * kMainBytes, m_tail, bar, kMainN, head, row0, policy);
  }
};

}  // namespace fpdt
