// Self-test kernels for the tcgen05 / TMA operand formats used by the attention kernels.
//
// Each probe runs ONE 128-row tile product on one CTA, exactly in the operand formats the
// attention kernels use, and writes the fp32 accumulator to global memory so a test can
// compare it with a host matmul:
//   variant 0 (QK^T):  C[128x128] = A[128xD] * B[128xD]^T   A,B: K-major TMA tiles (SS)
//   variant 1 (P V):   C[128xD]   = P[128x128] * V[128xD]   P: bf16 in TMEM (TS), V: MN-major TMA tile
//   variant 2 (dS K):  C[128xD]   = A[128x128] * V[128xD]   A: MN-major, written to smem by threads
//                                                           in the 128B-swizzled canonical layout (SS)
#include "attn_tile.cuh"
#include "tma_host.h"
#include "smem_layout.cuh"
#include "fpdt.h"
#include "fpdt_diag.h"

namespace fpdt {
namespace {

using namespace ptx;

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

template <int D>
__global__ void __launch_bounds__(128, 1)
probe_kernel(int variant, const __grid_constant__ CUtensorMap a_map, const __grid_constant__ CUtensorMap b_map,
             const __nv_bfloat16* __restrict__ a_plain, int ha, int hb, float* __restrict__ out) {
  using T = Tile<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const uint32_t sA = smem_u32(smem);
  const uint32_t sB = sA + 32768;
  __shared__ uint64_t bars[2];
  __shared__ uint32_t tmem_slot;
  const uint32_t warp = warp_id(), lane = lane_id(), tid = threadIdx.x;
  const uint32_t bar_load = smem_u32(&bars[0]), bar_mma = smem_u32(&bars[1]);
  if (warp == 0) tmem_alloc<256>(smem_u32(&tmem_slot));
  if (tid == 0) {
    mbar_init(bar_load, 1);
    mbar_init(bar_mma, 1);
    fence_mbar_init();
  }
  const uint32_t lane_base = (32 * (warp & 3)) << 16;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (variant == 1) {
    // P row `tid` (128 bf16 = 64 packed columns) -> TMEM columns [128, 192)
    uint32_t r[16];
    for (int j = 0; j < 4; ++j) {
      for (int i = 0; i < 16; ++i) {
        __nv_bfloat162 v;
        v.x = a_plain[tid * 128 + j * 32 + 2 * i];
        v.y = a_plain[tid * 128 + j * 32 + 2 * i + 1];
        r[i] = *reinterpret_cast<uint32_t*>(&v);
      }
      tmem_st16(tmem + lane_base + 128 + 16 * j, r);
    }
    tmem_wait_st();
  } else if (variant == 2) {
    // A[m][k] (m = output row, k = contraction) given row-major [128][128]; thread tid owns k = tid
    // and writes A[:, k] into the MN-major swizzled layout.
    for (int m8 = 0; m8 < 16; ++m8) {
      uint32_t w[4];
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 v;
        v.x = a_plain[(m8 * 8 + 2 * i) * 128 + tid];
        v.y = a_plain[(m8 * 8 + 2 * i + 1) * 128 + tid];
        w[i] = *reinterpret_cast<uint32_t*>(&v);
      }
      st_shared_v4(sA + mn_sw128_offset(m8 * 8, tid), w);
    }
    fence_async_shared();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint64_t pol = policy_evict_first();
    if (variant == 0) {
      mbar_expect_tx(bar_load, 2 * T::kBytes);
      T::load(sA, &a_map, bar_load, ha, 0, pol);
      T::load(sB, &b_map, bar_load, hb, 0, pol);
    } else {
      mbar_expect_tx(bar_load, T::kBytes);
      T::load(sB, &b_map, bar_load, hb, 0, pol);
    }
    mbar_wait(bar_load, 0);
    tc_fence_after();
    if (variant == 0) {
      const uint32_t id = idesc_bf16(128, 128, 0, 0);
      for (int kk = 0; kk < T::kKSteps; ++kk) mma_ss(tmem, T::desc_kmajor(sA, kk), T::desc_kmajor(sB, kk), id, kk > 0);
    } else if (variant == 1) {
      const uint32_t idm = idesc_bf16(128, D, 0, 1);
      for (int kk = 0; kk < 8; ++kk) mma_ts(tmem, tmem + 128 + kk * 8, T::desc_mn(sB, kk), idm, kk > 0);
    } else {
      const uint32_t idm = idesc_bf16(128, D, 1, 1);
      for (int kk = 0; kk < 8; ++kk) mma_ss(tmem, desc_a_mn_sw128(sA, kk), T::desc_mn(sB, kk), idm, kk > 0);
    }
    mma_commit(bar_mma);
  }
  __syncwarp();
  mbar_wait(bar_mma, 0);
  tc_fence_after();
  const int ncols = (variant == 0) ? 128 : D;
  const int row = 32 * (warp & 3) + lane;
  for (int c = 0; c < ncols; c += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + lane_base + c, r);
    tmem_wait_ld();
    for (int i = 0; i < 16; ++i) out[row * ncols + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

template <int D>
int run_probe(int variant, const void* a, const void* b, int H, int rows, void* out, cudaStream_t stream) {
  CUtensorMap am{}, bm{};
  if (variant == 0 && !make_tile_tmap<D>(&am, a, rows, H)) return 1;
  if (!make_tile_tmap<D>(&bm, b, rows, H)) return 1;
  if (variant != 0) am = bm;
  const int smem = 32768 * 2 + 1024;
  cudaFuncSetAttribute(probe_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<D><<<1, 128, smem, stream>>>(variant, am, bm, (const __nv_bfloat16*)a, H - 1, H - 1,
                                            (float*)out);
  return (int)cudaGetLastError();
}

}  // namespace
}  // namespace fpdt

extern "C" int fpdt_selftest_umma(int variant, int head_dim, const void* a, const void* b, int n_heads, int rows,
                                  void* out, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  switch (head_dim) {
    case 64: return fpdt::run_probe<64>(variant, a, b, n_heads, rows, out, stream);
    case 80: return fpdt::run_probe<80>(variant, a, b, n_heads, rows, out, stream);
    case 128: return fpdt::run_probe<128>(variant, a, b, n_heads, rows, out, stream);
  }
  return 3;
}
