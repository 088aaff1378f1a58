// Projection GEMMs of the attention block (fpdt_block_fwd / fpdt_block_bwd): the per-chunk
// QKV projection in front of the all-to-all ("T_i is projected to query q_i, key k_i, and value v_i.
// Then, we perform the Alltoall"), the output projection, and their backward ("dq_0, dk_0, dv_0 are used to
// compute the gradient of the input hidden state").
//
// bf16 mode: one persistent tcgen05 kernel for all three operand arrangements
//   Y  = X W      (A = X K-major,   B = W MN-major)
//   dX = dY W^T   (A = dY K-major,  B = W K-major)
//   dW = X^T dY   (A = X MN-major,  B = dY MN-major; fp32 output, overwritten or accumulated over chunks)
// Tile 128 x 256 (M x N), K step 64, 4-stage TMA ring (A 16 KB + B 32 KB per stage, 128B swizzle), fp32
// accumulators double-buffered in TMEM (2 x 256 columns) so the epilogue of tile t overlaps the MMAs of tile t+1.
// Warps: 0 TMA producer, 1 TMEM allocator + single-thread MMA issuer, 2-5 epilogue (thread = accumulator row).
// The epilogue can scatter the projected chunk straight into the all-to-all send layout [p][c][hq + 2hkv][d] (the
// pack of SURVEY §8(a) F3 fused into the GEMM): column j of the projection belongs to head j / d, which goes to
// rank head / (heads per rank).
//
// fp32 mode (validation only): a plain SIMT GEMM with true FP32 FMA (tcgen05 has no fp32 kind; kind::tf32 would
// miss the 1e-4 bar).
#include <algorithm>

#include "kernels.h"
#include "sm100_ptx.cuh"
#include "tma_host.h"

namespace fpdt {
namespace {

using namespace ptx;

constexpr int kBM = 128, kBN = 256, kBK = 64, kStages = 4;
constexpr int kABytes = kBM * kBK * 2, kBBytes = kBN * kBK * 2, kStageBytes = kABytes + kBBytes;
constexpr int kGemmThreads = 192;
constexpr int kGemmSmem = kStages * kStageBytes + 1024 /* align */ + 256 /* barriers */;

struct GemmTmaps {
  CUtensorMap a, b;
};

// Output addressing of the epilogue (element offsets).
struct OutMap {
  void* out = nullptr;
  int64_t ld = 0;          // plain: row stride (elements)
  int fp32 = 0;            // 1: fp32 output (dW), else bf16
  int accumulate = 0;      // fp32 output only: out += result
  // scatter into the all-to-all send layout (scatter != 0): column j -> head j / d
  int scatter = 0, d = 0, Hq = 0, Hkv = 0, hq = 0, hkv = 0;
  int64_t peer_stride = 0;  // elements between the per-peer blocks [c][hq + 2hkv][d]
};

__device__ __forceinline__ int64_t out_offset(const OutMap& o, int64_t row, int col) {
  if (!o.scatter) return row * o.ld + col;
  const int head = col / o.d, e = col - head * o.d;
  int peer, slot;
  if (head < o.Hq) {
    peer = head / o.hq;
    slot = head - peer * o.hq;
  } else if (head < o.Hq + o.Hkv) {
    const int kh = head - o.Hq;
    peer = kh / o.hkv;
    slot = o.hq + kh - peer * o.hkv;
  } else {
    const int vh = head - o.Hq - o.Hkv;
    peer = vh / o.hkv;
    slot = o.hq + o.hkv + vh - peer * o.hkv;
  }
  return (int64_t)peer * o.peer_stride + row * (int64_t)(o.hq + 2 * o.hkv) * o.d + (int64_t)slot * o.d + e;
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

// A_MN / B_MN: operand stored MN-major in global memory (see the file comment).
template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kGemmThreads, 1)
gemm_bf16_kernel(const __grid_constant__ GemmTmaps tm, const __grid_constant__ OutMap om, int M, int N, int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  auto bar = [&](int i) { return smem_u32(&bars[i]); };
  constexpr int B_FULL = 0, B_EMPTY = kStages, B_ACCF = 2 * kStages, B_ACCE = B_ACCF + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kStages * kStageBytes + 200);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int tiles_m = (M + kBM - 1) / kBM, tiles_n = (N + kBN - 1) / kBN;
  const int n_tiles = tiles_m * tiles_n;
  const int ksteps = (K + kBK - 1) / kBK;

  if (warp == 1) tmem_alloc<512>(smem_u32(tmem_slot));
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar(B_FULL + s), 1);
      mbar_init(bar(B_EMPTY + s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(B_ACCF + b), 1);
      mbar_init(bar(B_ACCE + b), 128);
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int it = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int m0 = (t / tiles_n) * kBM, n0 = (t % tiles_n) * kBN;  // n fastest: CTAs share the A rows
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % kStages;
          if (it >= kStages) mbar_wait(bar(B_EMPTY + s), ((it / kStages) - 1) & 1);
          const uint32_t fb = bar(B_FULL + s), sa = sbase + s * kStageBytes, sb = sa + kABytes;
          mbar_expect_tx(fb, kStageBytes);
          const int k0 = ks * kBK;
          if (A_MN) {  // A^T stored [K][M]: two boxes of 64 (M) x 64 (K)
            tma_load_2d(sa, &tm.a, fb, m0, k0);
            tma_load_2d(sa + 8192, &tm.a, fb, m0 + 64, k0);
          } else {     // A stored [M][K]: one box of 64 (K) x 128 (M)
            tma_load_2d(sa, &tm.a, fb, k0, m0);
          }
          if (B_MN) {  // B^T stored [K][N]: four boxes of 64 (N) x 64 (K)
#pragma unroll
            for (int q = 0; q < 4; ++q) tma_load_2d(sb + q * 8192, &tm.b, fb, n0 + 64 * q, k0);
          } else {     // B stored [N][K]: one box of 64 (K) x 256 (N)
            tma_load_2d(sb, &tm.b, fb, k0, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16(kBM, kBN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int it = 0, tl = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
        const int ab = tl & 1;
        if (tl >= 2) mbar_wait(bar(B_ACCE + ab), ((tl >> 1) - 1) & 1);  // accumulator drained by the epilogue
        tc_fence_after();
        const uint32_t tacc = tmem + ab * kBN;
        for (int ks = 0; ks < ksteps; ++ks, ++it) {
          const int s = it % kStages;
          mbar_wait(bar(B_FULL + s), (it / kStages) & 1);
          tc_fence_after();
          const uint32_t sa = sbase + s * kStageBytes, sb = sa + kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t da = A_MN ? smem_desc(sa + kk * 2048, 8192, 1024, kSw128)
                                     : smem_desc(sa + kk * 32, 16, 1024, kSw128);
            const uint64_t db = B_MN ? smem_desc(sb + kk * 2048, 8192, 1024, kSw128)
                                     : smem_desc(sb + kk * 32, 16, 1024, kSw128);
            mma_ss(tacc, da, db, idesc, (ks > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(bar(B_EMPTY + s));  // stage s may be refilled once these MMAs have read it
        }
        mma_commit(bar(B_ACCF + ab));
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2-5)
    const int lg = (int)(warp & 3);  // TMEM lane group this warp may access
    const int r = lg * 32 + (int)lane;
    int tl = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      const int ab = tl & 1;
      const int m0 = (t / tiles_n) * kBM, n0 = (t % tiles_n) * kBN;
      mbar_wait(bar(B_ACCF + ab), (tl >> 1) & 1);
      tc_fence_after();
      const int64_t row = (int64_t)m0 + r;
      const uint32_t tacc = tmem + ab * kBN + ((uint32_t)(lg * 32) << 16);
      const int ncols = min(kBN, N - n0);
#pragma unroll 1
      for (int c = 0; c < kBN; c += 32) {
        uint32_t v[32];
        tmem_ld32(tacc + c, v);
        tmem_wait_ld();
        if (row >= M || c >= ncols) continue;
        if (om.fp32) {
          float* o = static_cast<float*>(om.out);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const int col = n0 + c + i;
            if (c + i >= ncols) break;
            float4 x = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]), __uint_as_float(v[i + 2]),
                                   __uint_as_float(v[i + 3]));
            float4* dst = reinterpret_cast<float4*>(o + out_offset(om, row, col));
            if (om.accumulate) {
              const float4 y = *dst;
              x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
            }
            *dst = x;
          }
        } else {
          __nv_bfloat16* o = static_cast<__nv_bfloat16*>(om.out);
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            const int col = n0 + c + i;
            if (c + i >= ncols) break;
            uint4 w;
            w.x = pack_bf16x2(__uint_as_float(v[i]), __uint_as_float(v[i + 1]));
            w.y = pack_bf16x2(__uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            w.z = pack_bf16x2(__uint_as_float(v[i + 4]), __uint_as_float(v[i + 5]));
            w.w = pack_bf16x2(__uint_as_float(v[i + 6]), __uint_as_float(v[i + 7]));
            *reinterpret_cast<uint4*>(o + out_offset(om, row, col)) = w;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(bar(B_ACCE + ab));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// 2-D bf16 tensor map over a row-major matrix [outer][inner] (row stride ld elements), box {64, box_outer}, 128B
// swizzle; out-of-range elements of a box read as zero (ragged M, N, K).
bool make_tmap_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, int64_t ld, uint32_t box_outer) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <bool A_MN, bool B_MN>
int launch_bf16(const GemmTmaps& tm, const OutMap& om, int64_t M, int64_t N, int64_t K, cudaStream_t s) {
  auto kern = gemm_bf16_kernel<A_MN, B_MN>;
  if (int e = set_max_dynamic_smem((const void*)kern, kGemmSmem)) return e;
  const int64_t tiles = ((M + kBM - 1) / kBM) * ((N + kBN - 1) / kBN);
  const int grid = (int)std::min<int64_t>(tiles, sm_count());
  if (grid <= 0) return 0;
  kern<<<grid, kGemmThreads, kGemmSmem, s>>>(tm, om, (int)M, (int)N, (int)K);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------- fp32 validation GEMM
// C[m][n] (+)= sum_k A(m, k) B(k, n), A(m, k) = a[m*sam + k*sak], B(k, n) = b[k*sbk + n*sbn]; 64 x 64 tiles, 16 x 16
// threads with 4 x 4 outputs each, true FP32 FMA in a fixed k order.
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ a, int64_t sam, int64_t sak,
                                                       const float* __restrict__ b, int64_t sbk, int64_t sbn,
                                                       OutMap om, int M, int N, int K) {
  __shared__ float As[16][64 + 1], Bs[16][64 + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int kk = i / 64, mm = i % 64;
      const int m = m0 + mm, n = n0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? a[(int64_t)m * sam + (int64_t)k * sak] : 0.f;
      Bs[kk][mm] = (n < N && k < K) ? b[(int64_t)k * sbk + (int64_t)n * sbn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(As[kk][ty * 4 + i], Bs[kk][tx * 4 + j], acc[i][j]);
    __syncthreads();
  }
  float* o = static_cast<float*>(om.out);
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m >= M || n >= N) continue;
      float* dst = o + out_offset(om, m, n);
      *dst = om.accumulate ? *dst + acc[i][j] : acc[i][j];
    }
}

int launch_f32(const float* a, int64_t sam, int64_t sak, const float* b, int64_t sbk, int64_t sbn, const OutMap& om,
               int64_t M, int64_t N, int64_t K, cudaStream_t s) {
  if (M <= 0 || N <= 0) return 0;
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
  gemm_f32_kernel<<<grid, 256, 0, s>>>(a, sam, sak, b, sbk, sbn, om, (int)M, (int)N, (int)K);
  return (int)cudaGetLastError();
}

OutMap plain_out(void* out, int64_t ld, bool fp32, bool accumulate) {
  OutMap o;
  o.out = out;
  o.ld = ld;
  o.fp32 = fp32 ? 1 : 0;
  o.accumulate = accumulate ? 1 : 0;
  return o;
}

}  // namespace

int launch_gemm_xw(int dtype_fp32, const void* X, int64_t ldx, const void* W, int64_t ldw, void* Y, int64_t ldy,
                   int64_t rows, int64_t k, int64_t n, const ScatterOut* scatter, cudaStream_t s) {
  OutMap om = plain_out(Y, ldy, dtype_fp32 != 0, false);
  if (scatter) {
    om.scatter = 1;
    om.d = scatter->d;
    om.Hq = scatter->Hq;
    om.Hkv = scatter->Hkv;
    om.hq = scatter->hq;
    om.hkv = scatter->hkv;
    om.peer_stride = scatter->peer_stride;
  }
  if (dtype_fp32)
    return launch_f32((const float*)X, ldx, 1, (const float*)W, ldw, 1, om, rows, n, k, s);
  GemmTmaps tm;
  bool ok = make_tmap_2d(&tm.a, X, (uint64_t)k, (uint64_t)rows, ldx, kBM);  // A = X [rows][k], K-major
  ok &= make_tmap_2d(&tm.b, W, (uint64_t)n, (uint64_t)k, ldw, 64);           // B^T = W [k][n], MN-major
  if (!ok) return -1;
  return launch_bf16<false, true>(tm, om, rows, n, k, s);
}

int launch_gemm_dx(int dtype_fp32, const void* dY, int64_t ldy, const void* W, int64_t ldw, void* dX, int64_t ldx,
                   int64_t rows, int64_t k, int64_t n, cudaStream_t s) {
  const OutMap om = plain_out(dX, ldx, dtype_fp32 != 0, false);
  if (dtype_fp32)  // dX(r, h) = sum_j dY(r, j) W(h, j)
    return launch_f32((const float*)dY, ldy, 1, (const float*)W, 1, ldw, om, rows, k, n, s);
  GemmTmaps tm;
  bool ok = make_tmap_2d(&tm.a, dY, (uint64_t)n, (uint64_t)rows, ldy, kBM);  // A = dY [rows][n], K-major
  ok &= make_tmap_2d(&tm.b, W, (uint64_t)n, (uint64_t)k, ldw, kBN);           // B = W [k][n] = [N][K], K-major
  if (!ok) return -1;
  return launch_bf16<false, false>(tm, om, rows, k, n, s);
}

int launch_gemm_dw(int dtype_fp32, const void* X, int64_t ldx, const void* dY, int64_t ldy, float* dW, int64_t rows,
                   int64_t k, int64_t n, bool accumulate, cudaStream_t s) {
  const OutMap om = plain_out(dW, n, true, accumulate);
  if (dtype_fp32)  // dW(h, j) = sum_r X(r, h) dY(r, j)
    return launch_f32((const float*)X, 1, ldx, (const float*)dY, ldy, 1, om, k, n, rows, s);
  GemmTmaps tm;
  bool ok = make_tmap_2d(&tm.a, X, (uint64_t)k, (uint64_t)rows, ldx, 64);   // A^T = X [rows][k] = [K][M], MN-major
  ok &= make_tmap_2d(&tm.b, dY, (uint64_t)n, (uint64_t)rows, ldy, 64);      // B^T = dY [rows][n] = [K][N], MN-major
  if (!ok) return -1;
  return launch_bf16<true, true>(tm, om, k, n, rows, s);
}

}  // namespace fpdt
