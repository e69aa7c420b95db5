// HBM-bound reductions of the tensor-core path (d = 128, bf16 partials, T <= 32):
//   K6 merge (kv_major.py:207-242, fused LOCAL form): per (head j, token t) the
//      <= T per-block partials O_s / l_s (bf16) and (m_s, l_s) are combined in
//      ascending block order:  M = max m_s, w_s = l_s e^{m_s - M}, L = sum w_s,
//      out = sum_s w_s O_s / L, lse = M + ln L.
//   K9 dQ reduce (kv_major.py:326-340): dQ[t, j] = sum_s dq_s, ascending s.
// One warp per (j, t): lane k owns dims 4k..4k+3 (8-byte bf16 loads, 16-byte
// fp32 stores -> every partial row is one coalesced 256 B request); the slot
// statistics live one per lane and are reduced with shuffles.
#include "common.cuh"

namespace fsa {
namespace {

constexpr int kD = 128;

__device__ __forceinline__ float4 ld_bf16x4(const __nv_bfloat16* p) {
  const uint2 u = __ldcs(reinterpret_cast<const uint2*>(p));  // read once: evict first
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ int row_len(const int32_t* row, int T, int lane) {
  const int v = lane < T ? __ldg(row + lane) : -1;
  const unsigned live = __ballot_sync(0xffffffffu, v != -1);
  return __popc(live);  // entries are a prefix (validated selection)
}

__global__ void merge_bf16_kernel(const int32_t* __restrict__ idx, const __nv_bfloat16* __restrict__ obuf,
                                  const float2* __restrict__ ml, float* __restrict__ out,
                                  float* __restrict__ lse, float* __restrict__ m_out,
                                  float* __restrict__ l_out, int64_t N, int64_t h, int64_t g, int T) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= h * N) return;
  // consecutive warps take the g heads of one token (shared idx row)
  const int64_t t = wid / h, j = wid % h, kh = j / g;
  const int len = row_len(idx + (kh * N + t) * T, T, lane);
  const int64_t rb = (j * N + t) * (int64_t)T;
  float2 st = lane < len ? __ldg(ml + rb + lane) : make_float2(-INFINITY, 0.f);
  float M = st.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float w = lane < len ? st.y * __expf(st.x - M) : 0.f;
  float L = w;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  const __nv_bfloat16* src = obuf + rb * kD + lane * 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int s = 0;
  for (; s + 4 <= len; s += 4) {  // four independent 256 B rows in flight
    const float4 a = ld_bf16x4(src + (s + 0) * kD), b = ld_bf16x4(src + (s + 1) * kD);
    const float4 c = ld_bf16x4(src + (s + 2) * kD), d = ld_bf16x4(src + (s + 3) * kD);
    const float wa = __shfl_sync(0xffffffffu, w, s), wb = __shfl_sync(0xffffffffu, w, s + 1);
    const float wc = __shfl_sync(0xffffffffu, w, s + 2), wd = __shfl_sync(0xffffffffu, w, s + 3);
    acc.x += wa * a.x; acc.y += wa * a.y; acc.z += wa * a.z; acc.w += wa * a.w;
    acc.x += wb * b.x; acc.y += wb * b.y; acc.z += wb * b.z; acc.w += wb * b.w;
    acc.x += wc * c.x; acc.y += wc * c.y; acc.z += wc * c.z; acc.w += wc * c.w;
    acc.x += wd * d.x; acc.y += wd * d.y; acc.z += wd * d.z; acc.w += wd * d.w;
  }
  for (; s < len; ++s) {
    const float4 a = ld_bf16x4(src + s * kD);
    const float wa = __shfl_sync(0xffffffffu, w, s);
    acc.x += wa * a.x; acc.y += wa * a.y; acc.z += wa * a.z; acc.w += wa * a.w;
  }
  const float inv = 1.f / L;
  *reinterpret_cast<float4*>(out + (t * h + j) * kD + lane * 4) =
      make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  if (lane == 0) {
    if (lse) lse[j * N + t] = M + __logf(L);
    if (m_out) m_out[j * N + t] = M;
    if (l_out) l_out[j * N + t] = L;
  }
}

__global__ void dq_reduce_bf16_kernel(const int32_t* __restrict__ idx,
                                      const __nv_bfloat16* __restrict__ dq, float* __restrict__ dQ,
                                      int64_t N, int64_t h, int64_t g, int T) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= h * N) return;
  const int64_t t = wid / h, j = wid % h, kh = j / g;
  const int len = row_len(idx + (kh * N + t) * T, T, lane);
  const __nv_bfloat16* src = dq + ((j * N + t) * (int64_t)T) * kD + lane * 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int s = 0;
  for (; s + 4 <= len; s += 4) {
    const float4 a = ld_bf16x4(src + (s + 0) * kD), b = ld_bf16x4(src + (s + 1) * kD);
    const float4 c = ld_bf16x4(src + (s + 2) * kD), d = ld_bf16x4(src + (s + 3) * kD);
    acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
    acc.x += b.x; acc.y += b.y; acc.z += b.z; acc.w += b.w;
    acc.x += c.x; acc.y += c.y; acc.z += c.z; acc.w += c.w;
    acc.x += d.x; acc.y += d.y; acc.z += d.z; acc.w += d.w;
  }
  for (; s < len; ++s) {
    const float4 a = ld_bf16x4(src + s * kD);
    acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
  }
  *reinterpret_cast<float4*>(dQ + (t * h + j) * kD + lane * 4) = acc;
}

}  // namespace

bool fast_reduce_ok(const fsa_shape& s) { return s.d_V == kD && s.d_K == kD && s.T <= 32; }

int merge_bf16_fast(const fsa_shape* s, const int32_t* idx, const void* obuf, const void* ml,
                    void* out, void* lse, void* m_out, void* l_out, cudaStream_t st) {
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  merge_bf16_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      idx, (const __nv_bfloat16*)obuf, (const float2*)ml, (float*)out, (float*)lse, (float*)m_out,
      (float*)l_out, s->N, s->h, s->h / s->h_K, (int)s->T);
  FSA_LAUNCH_CHECK("merge_bf16");
  return FSA_OK;
}

int dq_reduce_bf16_fast(const fsa_shape* s, const int32_t* idx, const void* dq, void* dQ,
                        cudaStream_t st) {
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  dq_reduce_bf16_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      idx, (const __nv_bfloat16*)dq, (float*)dQ, s->N, s->h, s->h / s->h_K, (int)s->T);
  FSA_LAUNCH_CHECK("dq_reduce_bf16");
  return FSA_OK;
}

}  // namespace fsa
