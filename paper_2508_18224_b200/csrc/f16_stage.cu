// fp16 staging of the value operand for the tensor-core P.V products.
//
// The forward kernels (K5 selected, the sliding-window and compressed
// branches) run O = P V with fp16 operands: P = exp(z - m) <= 2^8 and an fp16
// mantissa rounds P 8x finer than bf16, which keeps out -- and with it the
// backward's delta = sum out * dOut -- consistent with the backward's fp32 P
// (tools/emulate_bf16.py: bf16 P is the dominant source of elementwise
// parity violations in dQ).  V is staged once per call as
//     V16[t][kh][:] = fp16(V[t][kh][:] * s_kh),   s_kh = 2^(15 - k_kh),
// with max|V[:, kh, :]| = f 2^k_kh, f in [0.5, 1): every element lands in
// fp16's normal range whatever the input's magnitude (a bf16 V above 65504
// would overflow a plain conversion); consumers divide the result by s_kh.
// bf16 -> fp16 with a power-of-two scale is exact for all but the values
// 2^24 below the head's maximum.
#include "common.cuh"
#include <cuda_fp16.h>

namespace fsa {
namespace {

constexpr int kRowsPerBlock = 512;

__device__ __forceinline__ float scale_of(uint32_t max_bits) {
  const float m = __uint_as_float(max_bits);
  if (!(m > 0.f) || !isfinite(m)) return 1.f;
  int k;
  frexpf(m, &k);
  int e = 15 - k;
  e = e < -120 ? -120 : (e > 120 ? 120 : e);
  return ldexpf(1.f, e);
}

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// grid (row chunks, heads): block (c, kh) covers rows [c*512, (c+1)*512) of head kh;
// 8-element vectors, d/8 threads per row.
template <typename T>
__global__ void __launch_bounds__(256) absmax_kernel(const T* __restrict__ x, int64_t rows,
                                                     int64_t heads, int64_t d, uint32_t* mx) {
  const int64_t kh = blockIdx.y, vpr = d / 8;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
  const int64_t r1 = r0 + kRowsPerBlock < rows ? r0 + kRowsPerBlock : rows;
  float m = 0.f;
  for (int64_t e = threadIdx.x; e < (r1 - r0) * vpr; e += blockDim.x) {
    const int64_t r = r0 + e / vpr, c = (e % vpr) * 8;
    float v[8];
    load8(x + (r * heads + kh) * d + c, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) m = fmaxf(m, fabsf(v[i]));  // NaN ignored (fmaxf)
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, wm[w]);
    atomicMax(mx + kh, __float_as_uint(m));  // non-negative floats order as integers
  }
}

template <typename T>
__global__ void __launch_bounds__(256) to_f16_kernel(const T* __restrict__ x, int64_t rows,
                                                     int64_t heads, int64_t d,
                                                     const uint32_t* __restrict__ mx,
                                                     __half* __restrict__ y, float* vscale) {
  const int64_t kh = blockIdx.y, vpr = d / 8;
  const float s = scale_of(mx[kh]);
  if (blockIdx.x == 0 && threadIdx.x == 0) vscale[kh] = s;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
  const int64_t r1 = r0 + kRowsPerBlock < rows ? r0 + kRowsPerBlock : rows;
  for (int64_t e = threadIdx.x; e < (r1 - r0) * vpr; e += blockDim.x) {
    const int64_t r = r0 + e / vpr, c = (e % vpr) * 8;
    float v[8];
    load8(x + (r * heads + kh) * d + c, v);
    uint4 o;
    __half2* h = reinterpret_cast<__half2*>(&o);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(v[2 * i] * s, v[2 * i + 1] * s);
    *reinterpret_cast<uint4*>(y + (r * heads + kh) * d + c) = o;
  }
}

}  // namespace

// x [rows][heads][d] (bf16 or f32) -> y fp16, vscale[0, heads) = s_kh;
// vscale[heads, 2 heads) is scratch (the per-head max bits).
int stage_f16(int src_dtype, const void* x, int64_t rows, int64_t heads, int64_t d, void* y,
              float* vscale, cudaStream_t st) {
  FSA_REQUIRE(d % 8 == 0, "fp16 staging needs d %% 8 == 0 (d = %lld)", (long long)d);
  FSA_REQUIRE(src_dtype == FSA_DT_BF16 || src_dtype == FSA_DT_F32,
              "fp16 staging reads bf16 or f32 (dtype %d)", src_dtype);
  if (rows == 0 || heads == 0) return FSA_OK;
  uint32_t* mx = reinterpret_cast<uint32_t*>(vscale + heads);
  cudaMemsetAsync(mx, 0, sizeof(uint32_t) * heads, st);
  dim3 grid((unsigned)((rows + kRowsPerBlock - 1) / kRowsPerBlock), (unsigned)heads);
  if (src_dtype == FSA_DT_BF16) {
    absmax_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, rows, heads, d, mx);
    to_f16_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, rows, heads, d, mx,
                                                       (__half*)y, vscale);
  } else {
    absmax_kernel<float><<<grid, 256, 0, st>>>((const float*)x, rows, heads, d, mx);
    to_f16_kernel<float><<<grid, 256, 0, st>>>((const float*)x, rows, heads, d, mx, (__half*)y,
                                               vscale);
  }
  FSA_LAUNCH_CHECK("stage_f16");
  return FSA_OK;
}

}  // namespace fsa

extern "C" int fsa_stage_f16_ops(const fsa_shape* s, int dtype, const void* Q, const void* K,
                                 const void* V, const void* dOut, void* Q16, void* K16, void* V16,
                                 void* dO16, float* scales, void* stream) {
  // Q / dOut [N][h][d] are [N][h_K][g d]: one scale per kv group (the rows of
  // one backward item mix the group's heads, and dK^T / dV^T contract over them)
  FSA_REQUIRE(scales != nullptr, "stage_f16_ops: scales is required");
  FSA_REQUIRE(s->h_K > 0 && s->h % s->h_K == 0, "stage_f16_ops: h %% h_K != 0");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t g = s->h / s->h_K, hk = s->h_K;
  const void* src[4] = {Q, K, V, dOut};
  void* dst[4] = {Q16, K16, V16, dO16};
  const int64_t d[4] = {g * s->d_K, s->d_K, s->d_V, g * s->d_V};
  for (int i = 0; i < 4; ++i) {
    if (!src[i]) continue;
    FSA_REQUIRE(dst[i] != nullptr, "stage_f16_ops: operand %d has no destination", i);
    if (int rc = fsa::stage_f16(dtype, src[i], s->N, hk, d[i], dst[i], scales + 2 * hk * i, st))
      return rc;
  }
  return FSA_OK;
}

extern "C" int fsa_v_to_f16(const fsa_shape* s, int dtype, const void* V, void* V16, float* vscale,
                            void* stream) {
  return fsa::stage_f16(dtype, V, s->N, s->h_K, s->d_V, V16, vscale, (cudaStream_t)stream);
}
