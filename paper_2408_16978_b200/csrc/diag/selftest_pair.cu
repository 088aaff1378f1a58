// Micro-benchmark of the CTA-pair tensor-core MMA (tcgen05.mma.cta_group::2, M = 256 over two SMs of a cluster)
// against the single-CTA M = 128 MMA, both cluster-launched with one CTA per SM (148 CTAs, 74 pairs).
// Diagnostic groundwork for the CTA-pair backward of DESIGN.md §6 (not on the hot path): each CTA of a pair supplies
// its own 128 rows of A and half of the N rows of B from the same shared-memory offsets; the leader CTA (cluster
// rank 0) issues every MMA; the commit arrives on the mbarrier of both CTAs (multicast).
#include "attn_tile.cuh"
#include "fpdt.h"
#include "fpdt_diag.h"

namespace fpdt {
namespace {

using namespace ptx;

__device__ __forceinline__ void mma_ss_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// mode 0: cta_group::1 SS MMA M = 128, N = n, K = 16 on every CTA (mode 2: on the leader CTA only, the partner SM
// idle).  mode 1: cta_group::2 SS MMA M = 256, N = n,
// K = 16, issued by the leader of each pair.  out[0] = SM cycles per MMA (pair 0's leader).
template <int mode>
__global__ void __launch_bounds__(128, 1) pair_perf_kernel(int n, int iters, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t rank = cluster_ctarank();
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) {
    if constexpr (mode == 1) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      tmem_alloc<512>(smem_u32(&slot));
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t s0 = smem_u32(smem);
  const bool issuer = threadIdx.x == 0 && (mode != 2 || rank == 0) && (mode != 1 || rank == 0);  // mode 2: mode 0 on the leader only
  long long t0 = 0;
  if (issuer) {
    const uint32_t id = idesc_bf16(mode == 1 ? 256 : 128, n, 0, 0);
    const uint64_t da = smem_desc(s0, 16, 1024, kSw128), db = smem_desc(s0 + 32768, 16, 1024, kSw128);
    const uint32_t acc1 = tmem + (n <= 128 ? 128 : 256);
    t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if constexpr (mode == 1)
          mma_ss_pair((u & 1) ? acc1 : tmem, da + 2 * u, db + 2 * u, id, 1);
        else
          mma_ss((u & 1) ? acc1 : tmem, da + 2 * u, db + 2 * u, id, 1);
      }
    }
    if constexpr (mode == 1)
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"((uint16_t)3)
          : "memory");
    else
      mma_commit(smem_u32(&bar));
  }
  if (threadIdx.x == 0 && (mode != 2 || rank == 0)) {
    mbar_wait(smem_u32(&bar), 0);
    if (issuer && blockIdx.x == 0) out[0] = (float)(clock64() - t0) / (float)iters;
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 0) {
    if constexpr (mode == 1)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      tmem_dealloc<512>(tmem);
  }
}

}  // namespace
}  // namespace fpdt

extern "C" int fpdt_selftest_pair(int mode, int n, int iters, float* out, void* stream) {
  if (mode < 0 || mode > 2 || n < 16 || n > 256 || n % 16 || iters < 8 || !out) return FPDT_ERR_ARG;
  const int smem = 64 * 1024 + 1024;
  auto kern = mode == 0 ? fpdt::pair_perf_kernel<0> : mode == 1 ? fpdt::pair_perf_kernel<1> : fpdt::pair_perf_kernel<2>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, n, iters, out);
  return e == cudaSuccess ? (int)cudaGetLastError() : (int)e;
}
