// Shared-memory tile format of a [128 rows x D] bf16 operand tile (Q, K, V or dO) and its
// tcgen05 smem descriptors.
//
// D = 64, 128: D/64 boxes of [128 rows x 64 cols] with 128B swizzle (16 KB atoms, 1024B-aligned).
// D = 80:      5 boxes of [128 rows x 16 cols] with 32B swizzle (4 KB atoms): 16 columns per atom, so the
//              same 20 KB serve a K-major operand (one atom per 16-wide contraction step) and an MN-major
//              operand with N = 80 in ONE instruction (5 atoms, LBO = 4 KB).  (Measured on B200: a
//              tcgen05.mma costs >= ~45 cycles whatever N <= 80, so an N = 64 + N = 16 split costs twice
//              an N = 80 instruction; microbenchmark in selftest_perf.cu.)
// The tile serves as
//   * a K-major operand (rows = M or N, contraction over D)       -> desc_kmajor(kk)
//   * an MN-major operand (rows = contraction K, N = D columns)   -> desc_mn(kk), N = D in one MMA
// kk indexes 16-element contraction steps (UMMA_K = 16 for bf16).
#pragma once
#include "sm100_ptx.cuh"

namespace fpdt {

template <int D>
struct Tile {
  static_assert(D == 64 || D == 80 || D == 128, "head_dim must be 64, 80 or 128");
  static constexpr bool kSw32 = (D == 80);
  static constexpr int kAtomCols = kSw32 ? 16 : 64;          // columns per swizzle atom
  static constexpr int kAtoms = D / kAtomCols;
  static constexpr int kAtomBytes = 128 * kAtomCols * 2;     // 4 KB (SW32) or 16 KB (SW128)
  static constexpr int kBytes = 128 * D * 2;                 // whole tile
  static constexpr int kKSteps = D / 16;                     // contraction steps when D is the K dimension
  static constexpr uint32_t kSwizzle = kSw32 ? ptx::kSw32 : ptx::kSw128;
  static constexpr uint32_t kRowBytes = kAtomCols * 2;       // 32 or 128
  static constexpr uint32_t kSBO = 8 * kRowBytes;            // 8-row group stride: 256 or 1024

  // K-major descriptor for contraction step kk over D (operand rows = 128).
  static __device__ __forceinline__ uint64_t desc_kmajor(uint32_t tile, int kk) {
    const int col = kk * 16;
    return ptx::smem_desc(tile + (col / kAtomCols) * kAtomBytes + (col % kAtomCols) * 2, 16, kSBO, kSwizzle);
  }
  // MN-major descriptor for contraction step kk over the 128 rows (N = D columns, atoms LBO apart).
  static __device__ __forceinline__ uint64_t desc_mn(uint32_t tile, int kk) {
    return ptx::smem_desc(tile + kk * 16 * kRowBytes, kAtomBytes, kSBO, kSwizzle);
  }
  // Issue the TMA loads of rows [row0, row0+128) of head `head` into `tile` (bytes = kBytes).
  static __device__ __forceinline__ void load(uint32_t tile, const CUtensorMap* m, uint32_t bar, int head, int row0,
                                              uint64_t policy) {
#pragma unroll
    for (int a = 0; a < kAtoms; ++a)
      ptx::tma_load_3d(tile + a * kAtomBytes, m, bar, a * kAtomCols, head, row0, policy);
  }
  // TMA box of one atom
  static constexpr uint32_t kBoxCols = kAtomCols;
};

// 2^x for a pair on the FMA pipe (FA4-style MUFU offload): x = j + f, j = rint(x), f in [-1/2, 1/2];
// degree-3 minimax for 2^f (max rel. error 7.5e-5 << bf16's 2^-9); the exponent is added as an integer.
// x is clamped to >= -126 (callers use it only where x is finite; at -127 the exponent addition would wrap into
// the sign bit and give a NaN, so keys far below the running max must still give ~0).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 kRnd = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 j = __fadd2_rn(x, kRnd);
  const float2 f = __fadd2_rn(x, __fadd2_rn(kRnd, make_float2(-j.x, -j.y)));
  float2 p = __ffma2_rn(f, make_float2(0.055169348f, 0.055169348f), make_float2(0.24260798f, 0.24260798f));
  p = __ffma2_rn(p, f, make_float2(0.69326115f, 0.69326115f));
  p = __ffma2_rn(p, f, make_float2(0.9999283f, 0.9999283f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}

}  // namespace fpdt
