// fp32 validation-mode chunk-pair attention (SIMT, true FP32 FMA; no tensor cores).
//
// Same chunk-pair semantics as the bf16 tcgen05 kernels (PAPER.md L218-230 forward with the online
// attention policy; L365 nested backward), used for the fp32 I/O mode whose parity bar is 1e-4
// (TF32 tensor cores would not meet it).  One warp per row; lanes split head_dim.
// Performance is irrelevant here (config 1 is launch-bound); these are kept simple and exact.
#include <math.h>

#include "kernels.h"

namespace fpdt {
namespace {

constexpr int kWarpsPerBlock = 8;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int D>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
fwd_f32_kernel(FwdArgs a) {
  constexpr int E = D / 32 + (D % 32 ? 1 : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + warp;  // row within the query range
  const int h = blockIdx.y;
  if (row >= a.n_q_rows) return;
  const int g = h / a.G;
  const float* Q = reinterpret_cast<const float*>(a.q.base);
  const float* K = reinterpret_cast<const float*>(a.k.base);
  const float* V = reinterpret_cast<const float*>(a.v.base);
  float q[E], o[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int d = lane + 32 * e;
    q[e] = d < D ? Q[((a.q_row0 + row) * a.q.heads + a.q.head0 + h) * D + d] : 0.f;
    o[e] = 0.f;
  }
  const int64_t qpos = a.q_pos0 + row;
  int64_t n_keys = a.n_kv_rows;
  if (a.causal) {
    const int64_t vis = qpos - a.kv_pos0 + 1;
    n_keys = vis < n_keys ? (vis > 0 ? vis : 0) : n_keys;
  }
  float m = -INFINITY, l = 0.f;
  for (int64_t j = 0; j < n_keys; ++j) {
    const float* kr = K + ((a.kv_row0 + j) * a.k.heads + a.k.head0 + g) * D;
    const float* vr = V + ((a.kv_row0 + j) * a.v.heads + a.v.head0 + g) * D;
    float part = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int d = lane + 32 * e;
      if (d < D) part = fmaf(q[e], kr[d], part);
    }
    const float s = warp_sum(part) * a.scale_log2;
    if (s > m) {
      const float alpha = exp2f(m - s);
      l *= alpha;
#pragma unroll
      for (int e = 0; e < E; ++e) o[e] *= alpha;
      m = s;
    }
    const float p = exp2f(s - m);
    l += p;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int d = lane + 32 * e;
      if (d < D) o[e] = fmaf(p, vr[d], o[e]);
    }
  }
  float lse = m + log2f(l);
  float wb = 1.f / l, wa = 0.f;
  float* acc = a.o_acc ? a.o_acc + (row * a.hq + h) * D : nullptr;
  if (a.has_prev) {
    const float la = a.lse_acc[(int64_t)h * a.n_q_rows + row];
    const float mx = fmaxf(la, lse);
    const float tot = mx + log2f(exp2f(la - mx) + exp2f(lse - mx));
    wa = exp2f(la - tot);
    wb *= exp2f(lse - tot);
    lse = tot;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int d = lane + 32 * e;
    if (d >= D) continue;
    float v = o[e] * wb;
    if (a.has_prev) v = fmaf(wa, acc[d], v);
    if (a.is_final)
      reinterpret_cast<float*>(a.o_out)[row * a.o_ld + (int64_t)(a.o_head0 + h) * D + d] = v;
    else
      acc[d] = v;
  }
  if (lane == 0) {
    if (a.is_final) {
      a.lse_save[(int64_t)h * a.lse_save_ld + row] = lse;
      if (a.lse_user) a.lse_user[row * a.lse_user_ld + a.lse_user_head0 + h] = lse * 0.69314718055994531f;
    } else {
      a.lse_acc[(int64_t)h * a.n_q_rows + row] = lse;
    }
  }
}

// dK, dV of one key row per warp, summed over the G query heads of its group and the query range.
template <int D>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
bwd_dkdv_f32_kernel(BwdArgs a) {
  constexpr int E = D / 32 + (D % 32 ? 1 : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + warp;  // key row within the range
  const int g = blockIdx.y;
  if (row >= a.n_kv_rows) return;
  const float* Q = reinterpret_cast<const float*>(a.q.base);
  const float* K = reinterpret_cast<const float*>(a.k.base);
  const float* V = reinterpret_cast<const float*>(a.v.base);
  const float* dO = reinterpret_cast<const float*>(a.dout.base);
  float k[E], v[E], dk[E], dv[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int d = lane + 32 * e;
    k[e] = d < D ? K[((a.kv_row0 + row) * a.k.heads + a.k.head0 + g) * D + d] : 0.f;
    v[e] = d < D ? V[((a.kv_row0 + row) * a.v.heads + a.v.head0 + g) * D + d] : 0.f;
    dk[e] = dv[e] = 0.f;
  }
  const int64_t kpos = a.kv_pos0 + row;
  int64_t i0 = 0;
  if (a.causal && kpos > a.q_pos0) i0 = kpos - a.q_pos0;
  for (int hh = 0; hh < a.G; ++hh) {
    const int h = g * a.G + hh;
    for (int64_t i = i0; i < a.n_q_rows; ++i) {
      const float* qr = Q + ((a.q_row0 + i) * a.q.heads + a.q.head0 + h) * D;
      const float* dr = dO + ((a.q_row0 + i) * a.dout.heads + a.dout.head0 + h) * D;
      float ps = 0.f, pd = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int d = lane + 32 * e;
        if (d < D) {
          ps = fmaf(qr[d], k[e], ps);
          pd = fmaf(dr[d], v[e], pd);
        }
      }
      const float s = warp_sum(ps), dp = warp_sum(pd);
      const float P = exp2f(fmaf(s, a.scale_log2, -a.lse2[(int64_t)h * a.stat_ld + i]));
      const float dS = P * (dp - a.Dstat[(int64_t)h * a.stat_ld + i]);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int d = lane + 32 * e;
        if (d < D) {
          dv[e] = fmaf(P, dr[d], dv[e]);
          dk[e] = fmaf(dS, qr[d], dk[e]);
        }
      }
    }
  }
  const int hkv = a.hq / a.G;
  float* dka = a.dk_acc + (row * hkv + g) * D;
  float* dva = a.dv_acc + (row * hkv + g) * D;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int d = lane + 32 * e;
    if (d >= D) continue;
    float xk = dk[e] * a.scale, xv = dv[e];
    if (!a.kv_acc_init) {
      xk += dka[d];
      xv += dva[d];
    }
    if (a.kv_final) {
      reinterpret_cast<float*>(a.dk_out)[row * a.kv_out_ld + (int64_t)(a.kv_out_head0 + g) * D + d] = xk;
      reinterpret_cast<float*>(a.dv_out)[row * a.kv_out_ld + (int64_t)(a.kv_out_head0 + g) * D + d] = xv;
    } else {
      dka[d] = xk;
      dva[d] = xv;
    }
  }
}

// dQ of one query row per warp (single owner per launch: plain read-modify-write of dq_acc).
template <int D>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
bwd_dq_f32_kernel(BwdArgs a) {
  constexpr int E = D / 32 + (D % 32 ? 1 : 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
  const int h = blockIdx.y;
  if (row >= a.n_q_rows) return;
  const int g = h / a.G;
  const float* Q = reinterpret_cast<const float*>(a.q.base);
  const float* K = reinterpret_cast<const float*>(a.k.base);
  const float* V = reinterpret_cast<const float*>(a.v.base);
  const float* dO = reinterpret_cast<const float*>(a.dout.base);
  float q[E], dov[E], dq[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int d = lane + 32 * e;
    q[e] = d < D ? Q[((a.q_row0 + row) * a.q.heads + a.q.head0 + h) * D + d] : 0.f;
    dov[e] = d < D ? dO[((a.q_row0 + row) * a.dout.heads + a.dout.head0 + h) * D + d] : 0.f;
    dq[e] = 0.f;
  }
  const float lse2 = a.lse2[(int64_t)h * a.stat_ld + row];
  const float Dv = a.Dstat[(int64_t)h * a.stat_ld + row];
  const int64_t qpos = a.q_pos0 + row;
  int64_t n_keys = a.n_kv_rows;
  if (a.causal) {
    const int64_t vis = qpos - a.kv_pos0 + 1;
    n_keys = vis < n_keys ? (vis > 0 ? vis : 0) : n_keys;
  }
  for (int64_t j = 0; j < n_keys; ++j) {
    const float* kr = K + ((a.kv_row0 + j) * a.k.heads + a.k.head0 + g) * D;
    const float* vr = V + ((a.kv_row0 + j) * a.v.heads + a.v.head0 + g) * D;
    float ps = 0.f, pd = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int d = lane + 32 * e;
      if (d < D) {
        ps = fmaf(q[e], kr[d], ps);
        pd = fmaf(dov[e], vr[d], pd);
      }
    }
    const float s = warp_sum(ps), dp = warp_sum(pd);
    const float P = exp2f(fmaf(s, a.scale_log2, -lse2));
    const float dS = P * (dp - Dv);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int d = lane + 32 * e;
      if (d < D) dq[e] = fmaf(dS, kr[d], dq[e]);
    }
  }
  float* dst = a.dq_acc + (int64_t)h * a.dq_head_stride + row * D;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int d = lane + 32 * e;
    if (d < D) dst[d] += dq[e] * a.scale;
  }
}

template <int D>
int fwd_f32(const FwdArgs& a, cudaStream_t s) {
  dim3 grid((a.n_q_rows + kWarpsPerBlock - 1) / kWarpsPerBlock, a.hq);
  fwd_f32_kernel<D><<<grid, kWarpsPerBlock * 32, 0, s>>>(a);
  return (int)cudaGetLastError();
}
template <int D>
int bwd_f32(const BwdArgs& a, cudaStream_t s) {
  dim3 g1((a.n_kv_rows + kWarpsPerBlock - 1) / kWarpsPerBlock, a.hq / a.G);
  bwd_dkdv_f32_kernel<D><<<g1, kWarpsPerBlock * 32, 0, s>>>(a);
  dim3 g2((a.n_q_rows + kWarpsPerBlock - 1) / kWarpsPerBlock, a.hq);
  bwd_dq_f32_kernel<D><<<g2, kWarpsPerBlock * 32, 0, s>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_attn_fwd_f32(const FwdArgs& a, int head_dim, cudaStream_t s) {
  switch (head_dim) {
    case 64: return fwd_f32<64>(a, s);
    case 80: return fwd_f32<80>(a, s);
    case 128: return fwd_f32<128>(a, s);
  }
  return -2;
}
int launch_attn_bwd_f32(const BwdArgs& a, int head_dim, cudaStream_t s) {
  switch (head_dim) {
    case 64: return bwd_f32<64>(a, s);
    case 80: return bwd_f32<80>(a, s);
    case 128: return bwd_f32<128>(a, s);
  }
  return -2;
}

}  // namespace fpdt
