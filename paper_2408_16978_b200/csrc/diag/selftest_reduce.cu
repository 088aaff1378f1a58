// Diagnostic micro-benchmark of the dQ reduce-add path (fp32 shared -> global reduce-add through L2), not on the
// hot path: one CTA per SM repeatedly reduces a 40 KB staging tile ([128 rows][80] fp32, the d = 80 dQ partial of
// one 128 x 128 (key, query) tile) into global memory, and reports SM cycles per tile.
#include "fpdt.h"
#include "fpdt_diag.h"
#include "sm100_ptx.cuh"
#include "tma_host.h"

namespace fpdt {
namespace {

using namespace ptx;

__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* m, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_reduce_f32(float* g, uint32_t s, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<uint64_t>(g)),
               "r"(s), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_store(float* g, uint32_t s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(g)),
               "r"(s), "r"(bytes)
               : "memory");
}

struct Maps {
  CUtensorMap m32, m16, m80;
};

// mode 0: three swizzled boxes (32, 32, 16 columns x 128 rows) per tile (the kernel's form)
// mode 1: one 1-D bulk reduce of the 40 KB tile (contiguous target)
// mode 2: ten 1-D bulk reduces of 4 KB
// mode 3: one unswizzled [128 x 80] tensor box
// mode 4: plain 1-D bulk STORE of 40 KB (no reduction), for comparison
// mode 5: mode 0 plus a 40 KB bulk LOAD per tile (global -> shared, mbarrier completion): the backward's Q + dO
// mode 6: the 40 KB bulk load alone
// inflight: bulk groups allowed in flight (cp.async.bulk.wait_group.read inflight-1 before reusing the staging)
// shared_target: all CTAs reduce into the same 40 KB (else one region per CTA)
__global__ void __launch_bounds__(128, 1) reduce_kernel(const __grid_constant__ Maps mp, float* gbase, int mode, int iters,
                                                          int inflight, int shared_target, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t s0 = smem_u32(smem);
  float* sf = reinterpret_cast<float*>(smem);
  for (int i = threadIdx.x; i < 2 * 10240; i += blockDim.x) sf[i] = 1e-6f;
  fence_async_shared();
  __syncthreads();
  const int cta = shared_target ? 0 : blockIdx.x;
  float* g = gbase + (size_t)cta * 10240;
  __shared__ uint64_t lbar;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&lbar), 1);
    fence_mbar_init();
  }
  __syncthreads();
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    const float* src = gbase + (size_t)148 * 10240 + (size_t)blockIdx.x * 10240;  // a separate 40 KB per CTA
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t st = s0 + (uint32_t)((it % 2) * 40960);
      if (mode == 5 || mode == 6) {
        mbar_expect_tx(smem_u32(&lbar), 40960);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         s0 + 81920u),
                     "l"(reinterpret_cast<uint64_t>(src)), "r"(40960), "r"(smem_u32(&lbar))
                     : "memory");
      }
      if (mode == 0 || mode == 5) {
        tma_reduce_add_3d(&mp.m32, st, 0, cta * 128, 0);
        tma_reduce_add_3d(&mp.m32, st + 16384, 32, cta * 128, 0);
        tma_reduce_add_3d(&mp.m16, st + 32768, 64, cta * 128, 0);
      } else if (mode == 1) {
        bulk_reduce_f32(g, st, 40960);
      } else if (mode == 2) {
        for (int k = 0; k < 10; ++k) bulk_reduce_f32(g + k * 1024, st + k * 4096, 4096);
      } else if (mode == 3) {
        tma_reduce_add_3d(&mp.m80, st, 0, cta * 128, 0);
      } else if (mode == 4) {
        bulk_store(g, st, 40960);
      }
      if (mode == 5 || mode == 6) mbar_wait(smem_u32(&lbar), it & 1);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (inflight <= 1)
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      else
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    t1 = clock64();
    if (blockIdx.x == 0) out[0] = (float)(t1 - t0) / iters;
  }
}

}  // namespace
}  // namespace fpdt

// Diagnostic: the dQ reduce-add path.  gbuf: device fp32 of >= 2 * 148 * 10240 floats (zeroed by the caller).  See
// reduce_kernel for the modes.  out[0] = SM cycles per 40 KB tile (CTA 0).  Returns 0 or a CUDA error code (-1: maps).
extern "C" int fpdt_selftest_reduce(int mode, int iters, int inflight, int shared_target, float* gbuf, float* out,
                                    void* stream) {
  fpdt::Maps mp;
  // the target viewed as [148 * 128 rows][1 head][80] fp32 (one 128-row tile per CTA)
  bool ok = fpdt::make_tmap_f32_head_major(&mp.m32, gbuf, 148 * 128, 1, 80, (uint64_t)148 * 128 * 80, 32, 128,
                                           CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= fpdt::make_tmap_f32_head_major(&mp.m16, gbuf, 148 * 128, 1, 80, (uint64_t)148 * 128 * 80, 16, 128,
                                       CU_TENSOR_MAP_SWIZZLE_64B);
  ok &= fpdt::make_tmap_f32_head_major(&mp.m80, gbuf, 148 * 128, 1, 80, (uint64_t)148 * 128 * 80, 80, 128,
                                       CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!ok) return -1;
  const int smem = 3 * 40960 + 1024;
  cudaFuncSetAttribute(fpdt::reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  fpdt::reduce_kernel<<<148, 128, smem, static_cast<cudaStream_t>(stream)>>>(mp, gbuf, mode, iters, inflight,
                                                                            shared_target, out);
  return (int)cudaGetLastError();
}
