// Device twin of fpdt_inputs/__init__.py (the seeded input generator).
//
// Test/bench infrastructure, NOT part of the product path and NOT part of the
// oracle: it holds no arithmetic of the method.  It writes rank r's shard
// [s_local, n_heads, head_dim] of tensor q/k/v/do in the rank-ordinal token
// order, bitwise identical to the numpy generator, so the
// oracle can regenerate any row on the host.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

__device__ __forceinline__ float base_value(uint32_t a, uint64_t idx) {
  uint32_t h1 = mix32(mix32(a ^ (uint32_t)(idx >> 32)) ^ (uint32_t)(idx & 0xffffffffu));
  uint32_t h2 = mix32(h1 + 0x9E3779B9u);
  int32_t n = (int32_t)(h1 & 0xffffu) + (int32_t)(h1 >> 16) + (int32_t)(h2 & 0xffffu) +
              (int32_t)(h2 >> 16) - 131070;
  return __fmul_rn((float)n, 3.0517578125e-05f);  // 2^-15, exact
}

// dist ids follow fpdt_inputs.DISTRIBUTIONS
enum { D_NORMAL = 0, D_PEAKY, D_DRIFT, D_SINK, D_SAME, D_CLASS, D_EXTREME, D_DRIFT32 };

template <typename OutT>
__global__ void gen_kernel(OutT* __restrict__ out, int tensor, int dist, uint32_t a, int64_t s_local,
                           int n_heads, int head_dim, int64_t seq_len, int rank, int world_size,
                           int64_t chunk_local, float drift_step, float drift_step32) {
  int64_t total = s_local * n_heads * head_dim;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = e / ((int64_t)n_heads * head_dim);
    int64_t rem = e - t * n_heads * head_dim;
    int h = (int)(rem / head_dim);
    int dim = (int)(rem - (int64_t)h * head_dim);
    int64_t g = ((t / chunk_local) * world_size + rank) * chunk_local + (t % chunk_local);
    float x;
    if (tensor == 1 && (dist == D_SAME || dist == D_CLASS)) {
      int64_t cls = 0;
      if (dist == D_CLASS) {
        uint32_t hh = mix32((uint32_t)(g & 0xffffffffu) ^ 0xC1A55u);
        cls = hh % (g >= seq_len / 2 ? 4u : 3u);
      }
      x = base_value(a, ((uint64_t)cls * n_heads + h) * head_dim + dim);
      if (cls == 3) x = __fmul_rn(x, 4.0f);
    } else {
      x = base_value(a, ((uint64_t)g * n_heads + h) * head_dim + dim);
      if (dist == D_PEAKY && tensor == 0) x = __fmul_rn(x, 4.0f);
      if (dist == D_EXTREME && tensor == 0) x = __fmul_rn(x, 30.0f);
      if (dist == D_DRIFT || dist == D_DRIFT32) {
        if (tensor == 0 && dim == 0) x = __fadd_rn(x, 2.0f);
        if (tensor == 1 && dim == 0) x = __fadd_rn(x, __fmul_rn((float)g, dist == D_DRIFT ? drift_step : drift_step32));
      }
      if (dist == D_SINK) {
        if (tensor == 0) x = __fadd_rn(x, 0.5f);
        if (tensor == 1 && g == 0) x = 2.0f;
      }
    }
    __nv_bfloat16 b = __float2bfloat16_rn(x);
    if constexpr (sizeof(OutT) == 2) out[e] = b;
    else out[e] = __bfloat162float(b);
  }
}

uint32_t host_mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

}  // namespace

extern "C" {

// Fill rank `rank`'s shard of tensor (0=q,1=k,2=v,3=do) with distribution `dist`.
// out: device pointer, [s_local, n_heads, head_dim] contiguous, bf16 (out_dtype 0) or fp32 (1).
// Returns 0 on success, else the cudaError_t of the launch.
int fpdt_gen_fill(void* out, int out_dtype, int tensor, int dist, uint32_t seed, int64_t s_local,
                  int n_heads, int head_dim, int64_t seq_len, int rank, int world_size,
                  int64_t chunk_size, cudaStream_t stream) {
  uint32_t a = host_mix32(seed * 0x9E3779B9u + (uint32_t)tensor * 0x85EBCA6Bu + 0x632BE5ABu);
  int64_t chunk_local = chunk_size / world_size;
  float drift_step = (float)(8.0 / (double)seq_len), drift_step32 = (float)(32.0 / (double)seq_len);
  int threads = 256, blocks = 148 * 16;
  if (out_dtype == 0)
    gen_kernel<__nv_bfloat16><<<blocks, threads, 0, stream>>>((__nv_bfloat16*)out, tensor, dist, a,
        s_local, n_heads, head_dim, seq_len, rank, world_size, chunk_local, drift_step, drift_step32);
  else
    gen_kernel<float><<<blocks, threads, 0, stream>>>((float*)out, tensor, dist, a, s_local, n_heads,
        head_dim, seq_len, rank, world_size, chunk_local, drift_step, drift_step32);
  return (int)cudaGetLastError();
}

}  // extern "C"
