// HBM-bound support kernels of the FPDT path: D preprocess (B1), output conversion, all-to-all
// pack/unpack (F3/F10/B2/B7), lse layout change.  Coalesced, 16-byte vectorised.
#include "kernels.h"

namespace fpdt {
namespace {

constexpr int kBlock = 256;
inline int grid_for(int64_t n) {
  int64_t b = (n + kBlock - 1) / kBlock;
  const int64_t cap = 148 * 32;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

// B1: D[h*ld + t] = <dO[t,h,:], O[t,h,:]> in fp32 (backward needs o_f, o_g; reading R9).
// Block = 8 warps on 8 consecutive rows: warp w streams row t0 + w's heads*head_dim elements as consecutive 16-byte
// vectors (one contiguous run per row, coalesced), writes each vector's partial dot product to shared memory, then
// threads (head, row) add the head_dim / vector-width partials of one head and write D with consecutive threads on
// consecutive rows (32-byte runs).  Dynamic shared memory: 8 * heads * vectors-per-head floats.
constexpr int kDRows = 8;
template <typename T>
__global__ void __launch_bounds__(256) preprocess_D_kernel(const T* __restrict__ o, const T* __restrict__ dout,
                                                           int64_t rows, int heads, int head_dim, int64_t row_ld,
                                                           const __nv_bfloat16* __restrict__ resid, int64_t resid_ld,
                                                           float* __restrict__ D, int64_t ld) {
  extern __shared__ float part[];  // [kDRows][heads * vph]
  constexpr int epv = 16 / sizeof(T);  // elements per 16-byte vector
  const int vph = head_dim / epv, nv = heads * vph;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t t0 = (int64_t)blockIdx.x * kDRows; t0 < rows; t0 += (int64_t)gridDim.x * kDRows) {
    const int64_t t = t0 + warp;
    if (t < rows) {
      const T* po = o + t * row_ld;
      const T* pd = dout + t * row_ld;
      for (int v = lane; v < nv; v += 32) {
        float acc = 0.f;
        if constexpr (sizeof(T) == 2) {
          const uint4 a = *reinterpret_cast<const uint4*>(po + (int64_t)v * epv);
          const uint4 b = *reinterpret_cast<const uint4*>(pd + (int64_t)v * epv);
          uint4 rr = make_uint4(0, 0, 0, 0);
          if (resid) rr = *reinterpret_cast<const uint4*>(resid + t * resid_ld + (int64_t)v * epv);
          const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
          const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
          const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rr);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 fa = __bfloat1622float2(a2[i]), fb = __bfloat1622float2(b2[i]);
            const float2 fr = __bfloat1622float2(r2[i]);
            acc = fmaf(fa.x + fr.x, fb.x, acc);
            acc = fmaf(fa.y + fr.y, fb.y, acc);
          }
        } else {
          const float4 a = *reinterpret_cast<const float4*>(po + (int64_t)v * epv);
          const float4 b = *reinterpret_cast<const float4*>(pd + (int64_t)v * epv);
          acc = fmaf(a.x, b.x, acc);
          acc = fmaf(a.y, b.y, acc);
          acc = fmaf(a.z, b.z, acc);
          acc = fmaf(a.w, b.w, acc);
        }
        part[warp * nv + v] = acc;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < heads * kDRows; i += blockDim.x) {
      const int h = i / kDRows, rr = i - h * kDRows;
      if (t0 + rr < rows) {
        const float* pp = part + rr * nv + h * vph;
        float acc = 0.f;
        for (int k = 0; k < vph; ++k) acc += pp[k];
        D[(int64_t)h * ld + t0 + rr] = acc;
      }
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void convert_out_kernel(const float* __restrict__ src, int64_t rows, int heads, int head_dim,
                                   int64_t src_head_stride, float scale, T* __restrict__ dst, int64_t dst_ld,
                                   int dst_head0) {
  const int64_t per_row = (int64_t)heads * head_dim / 4;
  const int64_t n = rows * per_row;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx / per_row;
    const int64_t w = (idx - t * per_row) * 4;  // element offset within the destination row
    const int64_t h = w / head_dim, e = w - h * head_dim;
    const float4 v = *reinterpret_cast<const float4*>(src + h * src_head_stride + t * head_dim + e);
    T* out = dst + t * dst_ld + (int64_t)dst_head0 * head_dim + w;
    if constexpr (sizeof(T) == 2) {
      __nv_bfloat162 a = __floats2bfloat162_rn(v.x * scale, v.y * scale);
      __nv_bfloat162 b = __floats2bfloat162_rn(v.z * scale, v.w * scale);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&a);
      u.y = *reinterpret_cast<uint32_t*>(&b);
      *reinterpret_cast<uint2*>(out) = u;
    } else {
      *reinterpret_cast<float4*>(out) = make_float4(v.x * scale, v.y * scale, v.z * scale, v.w * scale);
    }
  }
}

// Generic 16-byte-vector row/head re-layout shared by pack and unpack.
// Element (peer, t, hh, e) of the head-sharded side <-> (t, peer*hp + hh, e) of the sequence side.
template <bool kPack>
__global__ void relayout_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t c, int H, int p,
                                int vec_per_head, int64_t hs_peer_stride_v, int64_t hs_row_ld_v, int hs_head0,
                                int64_t seq_row_ld_v) {
  const int hp = H / p;
  const int64_t n = c * H * (int64_t)vec_per_head;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx / ((int64_t)H * vec_per_head);
    const int64_t rem = idx - t * H * vec_per_head;
    const int hg = (int)(rem / vec_per_head);
    const int e = (int)(rem - (int64_t)hg * vec_per_head);
    const int peer = hg / hp, hh = hg - peer * hp;
    const int64_t seq_off = t * seq_row_ld_v + rem;  // sequence side [c][H][d], rows seq_row_ld apart
    const int64_t hs_off = peer * hs_peer_stride_v + t * hs_row_ld_v + (int64_t)(hs_head0 + hh) * vec_per_head + e;
    if (kPack)
      dst[hs_off] = src[seq_off];
    else
      dst[seq_off] = src[hs_off];
  }
}

// lse layout change [h][t] (log2) -> [t][h] (natural log) through a shared-memory tile of 32 rows x heads: reads run
// along t, writes along h (both coalesced)
__global__ void __launch_bounds__(256) lse_to_user_kernel(const float* __restrict__ src, int64_t ld, int64_t rows,
                                                          int heads, float* __restrict__ dst, int64_t dst_ld,
                                                          int dst_head0) {
  extern __shared__ float tile[];  // [heads][33]
  for (int64_t t0 = (int64_t)blockIdx.x * 32; t0 < rows; t0 += (int64_t)gridDim.x * 32) {
    for (int i = threadIdx.x; i < heads * 32; i += blockDim.x) {
      const int h = i >> 5, tt = i & 31;
      if (t0 + tt < rows) tile[h * 33 + tt] = src[(int64_t)h * ld + t0 + tt] * 0.69314718055994531f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < heads * 32; i += blockDim.x) {
      const int tt = i / heads, h = i - tt * heads;
      if (t0 + tt < rows) dst[(t0 + tt) * dst_ld + dst_head0 + h] = tile[h * 33 + tt];
    }
    __syncthreads();
  }
}

// Scheduler stress (debug): one thread sleeps ~ns nanoseconds on its stream, perturbing the relative timing of the
// library's streams so that a missing cross-stream event edge shows up as a parity failure (SURVEY §4 tier 5).
__global__ void stress_sleep_kernel(uint32_t ns) {
  for (uint32_t waited = 0; waited < ns; waited += 1000) __nanosleep(1000);
}

}  // namespace

int launch_stress_sleep(uint32_t ns, cudaStream_t s) {
  stress_sleep_kernel<<<1, 1, 0, s>>>(ns);
  return (int)cudaGetLastError();
}

int launch_bwd_preprocess_D(const void* o, const void* dout, int dtype, int64_t rows, int heads, int head_dim,
                            int64_t row_ld, const void* resid, int64_t resid_ld, float* D, int64_t ld,
                            cudaStream_t s) {
  const int epv = dtype == 0 ? 8 : 4;
  const size_t smem = (size_t)kDRows * heads * (head_dim / epv) * sizeof(float);
  const int64_t blocks = (rows + kDRows - 1) / kDRows;
  const int grid = (int)(blocks < 148 * 8 ? (blocks > 0 ? blocks : 1) : 148 * 8);
  if (smem > 48 * 1024) {
    if (smem > 227 * 1024) return (int)cudaErrorInvalidValue;
    if (int e = set_max_dynamic_smem(dtype == 0 ? (const void*)preprocess_D_kernel<__nv_bfloat16>
                                                : (const void*)preprocess_D_kernel<float>,
                                     227 * 1024))
      return e;
  }
  if (dtype == 0)
    preprocess_D_kernel<__nv_bfloat16><<<grid, 256, smem, s>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout,
                                                               rows, heads, head_dim, row_ld,
                                                               (const __nv_bfloat16*)resid, resid_ld, D, ld);
  else
    preprocess_D_kernel<float><<<grid, 256, smem, s>>>((const float*)o, (const float*)dout, rows, heads, head_dim,
                                                       row_ld, nullptr, 0, D, ld);
  return (int)cudaGetLastError();
}

int launch_convert_out(const float* src, int64_t rows, int heads, int head_dim, int64_t src_head_stride, float scale,
                       void* dst, int dtype, int64_t dst_ld, int dst_head0, cudaStream_t s) {
  const int64_t n = rows * heads * head_dim / 4;
  if (dtype == 0)
    convert_out_kernel<__nv_bfloat16><<<grid_for(n), kBlock, 0, s>>>(src, rows, heads, head_dim, src_head_stride,
                                                                     scale, (__nv_bfloat16*)dst, dst_ld, dst_head0);
  else
    convert_out_kernel<float><<<grid_for(n), kBlock, 0, s>>>(src, rows, heads, head_dim, src_head_stride, scale,
                                                             (float*)dst, dst_ld, dst_head0);
  return (int)cudaGetLastError();
}

int launch_pack_seq2head(const void* src, int64_t c, int H, int head_dim, int p, int elem_bytes, void* dst,
                         int64_t dst_peer_stride_elems, int64_t dst_row_ld, int dst_head0, cudaStream_t s,
                         int64_t src_row_ld) {
  const int vph = head_dim * elem_bytes / 16;
  const int epv = 16 / elem_bytes;
  const int64_t n = c * H * (int64_t)vph;
  const int64_t seq_ld = src_row_ld > 0 ? src_row_ld : (int64_t)H * head_dim;
  relayout_kernel<true><<<grid_for(n), kBlock, 0, s>>>((const uint4*)src, (uint4*)dst, c, H, p, vph,
                                                       dst_peer_stride_elems / epv, dst_row_ld / epv, dst_head0,
                                                       seq_ld / epv);
  return (int)cudaGetLastError();
}

int launch_unpack_head2seq(const void* src, int64_t src_peer_stride_elems, int64_t src_row_ld, int src_head0,
                           int64_t c, int H, int head_dim, int p, int elem_bytes, void* dst, cudaStream_t s,
                           int64_t dst_row_ld) {
  const int vph = head_dim * elem_bytes / 16;
  const int epv = 16 / elem_bytes;
  const int64_t n = c * H * (int64_t)vph;
  const int64_t seq_ld = dst_row_ld > 0 ? dst_row_ld : (int64_t)H * head_dim;
  relayout_kernel<false><<<grid_for(n), kBlock, 0, s>>>((const uint4*)src, (uint4*)dst, c, H, p, vph,
                                                        src_peer_stride_elems / epv, src_row_ld / epv, src_head0,
                                                        seq_ld / epv);
  return (int)cudaGetLastError();
}

int launch_lse_to_user(const float* src, int64_t ld, int64_t rows, int heads, float* dst, int64_t dst_ld,
                       int dst_head0, cudaStream_t s) {
  const int64_t blocks = (rows + 31) / 32;
  const int grid = (int)(blocks < 148 * 8 ? (blocks > 0 ? blocks : 1) : 148 * 8);
  lse_to_user_kernel<<<grid, 256, (size_t)heads * 33 * sizeof(float), s>>>(src, ld, rows, heads, dst, dst_ld,
                                                                           dst_head0);
  return (int)cudaGetLastError();
}

}  // namespace fpdt
