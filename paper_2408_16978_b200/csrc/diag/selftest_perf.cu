// Micro-benchmarks of the sm_100a units the attention kernels lean on (diagnostic, not on the hot path):
// tcgen05.mma issue cost per instruction shape, MUFU ex2 throughput, TMEM load throughput.
// Each runs one CTA per SM (148 CTAs) and reports the median SM-cycles per operation of CTA 0.
#include <cuda_fp16.h>

#include "attn_tile.cuh"
#include "fpdt.h"
#include "fpdt_diag.h"

namespace fpdt {
namespace {

using namespace ptx;

// what: 0 = SS MMA M=128 N=n K=16, 1 = TS MMA (A in TMEM) M=128 N=n K=16, 2 = MUFU.EX2 per thread (128 thr),
//       3 = tcgen05.ld 32x32b.x32 per warp (4 warps), 4 = FFMA-poly exp2 per thread
__global__ void __launch_bounds__(1024, 1) perf_kernel(int what, int n, int iters, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t warp = warp_id();
  if (warp == 0) tmem_alloc<512>(smem_u32(&slot));
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t s0 = smem_u32(smem);
  long long t0 = 0, t1 = 0;
  float sink = 0.f;
  if (what <= 1) {
    if (threadIdx.x == 0) {
      const uint32_t id = idesc_bf16(128, n, 0, 0);
      const uint64_t da = smem_desc(s0, 16, 1024, kSw128), db = smem_desc(s0 + 32768, 16, 1024, kSw128);
      const int chains = (iters & 7) ? (iters & 7) : 1;
      const uint32_t stride = n <= 128 ? 128 : 256;
      const uint32_t acc0 = tmem, acc1 = tmem + (chains > 1 ? stride : 0);
      t0 = clock64();
      if (what == 0) {
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) mma_ss((u & 1) ? acc1 : acc0, da + 2 * u, db + 2 * u, id, 1);
        }
      } else {
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) mma_ts((u & 1) ? acc1 : acc0, tmem + 256 + 8 * u, db + 2 * u, id, 1);
        }
      }
      mma_commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), 0);
      t1 = clock64();
    }
  } else if (what == 2 || what == 4) {
    float x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = -0.001f * threadIdx.x - 0.1f * c;
    t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float y;
        if (what == 2) {
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[c]));
        } else {
          const float xc = fmaxf(x[c], -127.f);
          const float fl = floorf(xc);
          const float f = xc - fl;
          float p = fmaf(f, 0.0790393f, 0.2261766f);
          p = fmaf(p, f, 0.6951474f);
          p = fmaf(p, f, 1.0f);
          y = __int_as_float(__float_as_int(p) + ((int)fl << 23));
        }
        x[c] = x[c] + y * 1e-9f;
      }
    }
    t1 = clock64();
#pragma unroll
    for (int c = 0; c < 8; ++c) sink += x[c];
  } else if (what == 5 || what == 6 || what == 7 || what == 8) {
    // 5: MUFU ex2 throughput, 32 independent chains per thread; 6: MUFU ex2 latency, one chain;
    // 7: FMA-pipe exp2 (packed f32x2 polynomial) throughput, 16 independent pairs; 8: ex2.approx.f16x2, 16 chains
    float x[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) x[c] = -0.001f * threadIdx.x - 0.01f * c;
    t0 = clock64();
    if (what == 5) {
      for (int i = 0; i < iters; i += 32) {
#pragma unroll
        for (int c = 0; c < 32; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
      }
    } else if (what == 6) {
      for (int i = 0; i < iters; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[0]));
    } else if (what == 7) {
      for (int i = 0; i < iters; i += 32) {
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          float2 v = make_float2(fmaxf(x[c], -127.f), fmaxf(x[c + 1], -127.f));
          const float2 kR = make_float2(12582912.f, 12582912.f);
          const float2 j = __fadd2_rn(v, kR);
          const float2 f = __fadd2_rn(v, __fadd2_rn(kR, make_float2(-j.x, -j.y)));
          float2 p = __ffma2_rn(f, make_float2(0.055f, 0.055f), make_float2(0.2426f, 0.2426f));
          p = __ffma2_rn(p, f, make_float2(0.6933f, 0.6933f));
          p = __ffma2_rn(p, f, make_float2(0.99993f, 0.99993f));
          x[c] = -__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23));
          x[c + 1] = -__int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23));
        }
      }
    } else {
      uint32_t h[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        __half2 t = __floats2half2_rn(x[2 * c], x[2 * c + 1]);
        h[c] = *reinterpret_cast<uint32_t*>(&t);
      }
      for (int i = 0; i < iters; i += 32) {
#pragma unroll
        for (int c = 0; c < 16; ++c) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[c]));
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) x[c] = __uint_as_float(h[c]);
    }
    t1 = clock64();
#pragma unroll
    for (int c = 0; c < 32; ++c) sink += x[c];
  } else if (what == 3) {
    const uint32_t lane_off = ((warp & 3) * 32) << 16;
    uint32_t r[32];
    t0 = clock64();
    uint32_t r2[32], r3[32], r4[32];
    for (int i = 0; i < iters; i += 4) {
      tmem_ld32(tmem + lane_off + 0, r);
      tmem_ld32(tmem + lane_off + 32, r2);
      tmem_ld32(tmem + lane_off + 64, r3);
      tmem_ld32(tmem + lane_off + 96, r4);
      tmem_wait_ld();
      sink += __uint_as_float(r[3]) + __uint_as_float(r2[7]) + __uint_as_float(r3[11]) + __uint_as_float(r4[31]);
    }
    t1 = clock64();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0) / iters;
  if (sink == 12345.f) out[1] = sink;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

// The forward softmax's exponential stage on one row of kElems columns per thread, registers only: FFMA2 scale,
// MUFU ex2 or (every `every`-th pair, 0 = none) the FMA-pipe polynomial, bf16 packing.  Cycles per row of CTA 0.
template <int kElems, int every>
__global__ void __launch_bounds__(kElems == 128 ? 256 : 512, 1) softmax_bench_kernel(int iters, float* out) {
  float x[kElems];
#pragma unroll
  for (int c = 0; c < kElems; ++c) x[c] = -0.03f * c - 0.001f * threadIdx.x;
  uint32_t acc0 = 0, acc1 = 0;
  const float2 s2 = make_float2(0.161f, 0.161f);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float mb = -1.5f - 1e-7f * it;  // per-iteration (as the running max): nothing is loop-invariant
    const float2 nm = make_float2(mb, mb);
#pragma unroll
    for (int i = 0; i < kElems; i += 2) {
      const float2 e = __ffma2_rn(make_float2(x[i], x[i + 1]), s2, nm);
      float2 pr;
      if (every && (i / 2) % (every ? every : 1) == every - 1) {
        float2 v = make_float2(fmaxf(e.x, -127.f), fmaxf(e.y, -127.f));
        const float2 kR = make_float2(12582912.f, 12582912.f);
        const float2 j = __fadd2_rn(v, kR);
        const float2 f = __fadd2_rn(v, __fadd2_rn(kR, make_float2(-j.x, -j.y)));
        float2 p = __ffma2_rn(f, make_float2(0.055f, 0.055f), make_float2(0.2426f, 0.2426f));
        p = __ffma2_rn(p, f, make_float2(0.6933f, 0.6933f));
        p = __ffma2_rn(p, f, make_float2(0.99993f, 0.99993f));
        pr = make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                         __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
      } else {
        float a0, a1;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(a0) : "f"(e.x));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(a1) : "f"(e.y));
        pr = make_float2(a0, a1);
      }
      if ((i / 2) & 1)
        acc1 ^= pack_bf16x2(pr.x, pr.y);
      else
        acc0 ^= pack_bf16x2(pr.x, pr.y);
    }
    x[0] += 1e-7f;
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0) / iters;
  if ((acc0 ^ acc1) == 12345u) out[1] = x[1];
}

}  // namespace
}  // namespace fpdt

// Diagnostic: fwd-softmax exponential stage throughput (what = 0: 128 columns per thread, 1: 64), `threads` per
// CTA, one pair in `every` on the FMA-pipe polynomial (0 = all MUFU).  out[0] = SM cycles per row per thread.
extern "C" int fpdt_selftest_softmax(int what, int threads, int every, int iters, float* out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
#define FPDT_SMB(E, V) fpdt::softmax_bench_kernel<E, V><<<148, threads, 0, s>>>(iters, out)
  if (what == 0) {
    if (every == 0) FPDT_SMB(128, 0); else if (every == 2) FPDT_SMB(128, 2); else if (every == 4) FPDT_SMB(128, 4); else FPDT_SMB(128, 8);
  } else {
    if (every == 0) FPDT_SMB(64, 0); else if (every == 2) FPDT_SMB(64, 2); else if (every == 4) FPDT_SMB(64, 4); else FPDT_SMB(64, 8);
  }
#undef FPDT_SMB
  return (int)cudaGetLastError();
}

extern "C" int fpdt_selftest_perf(int what, int n, int iters, float* out, void* stream) {
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(fpdt::perf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int threads = ((what == 2 || what >= 4) && n > 0) ? n : 128;  // n = threads per CTA for the ALU tests
  fpdt::perf_kernel<<<148, threads, smem, static_cast<cudaStream_t>(stream)>>>(what, n, iters, out);
  return (int)cudaGetLastError();
}
