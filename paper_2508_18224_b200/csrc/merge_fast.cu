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

// Gated-combine epilogue (branches.py:95-104): with cmb.out != null the warp
// also writes out = ((0 + tau0 out_cmp) + tau1 out_sel) + tau2 out_slide (bf16).
// kNarrow: out_cmp / out_slide are read and out (out_sel) written as bf16.
struct Combine {
  const void* out_cmp;
  const void* out_slide;
  const float* tau;
  __nv_bfloat16* out;
};

__device__ __forceinline__ void ld4(const void* p, int64_t e, bool narrow, float (&v)[4]) {
  if (narrow) {
    const float4 x = ld_bf16x4(reinterpret_cast<const __nv_bfloat16*>(p) + e);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else {
    const float4 x = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p) + e);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
}

template <int TMAX, bool kNarrow>  // TMAX >= T: partial rows held in registers
__global__ void __launch_bounds__(256) merge_bf16_kernel(
    const int32_t* __restrict__ idx, const __nv_bfloat16* __restrict__ obuf,
    const float2* __restrict__ ml, void* __restrict__ out, float* __restrict__ lse,
    float* __restrict__ m_out, float* __restrict__ l_out, int64_t N, int64_t h, int64_t g, int T,
    Combine cmb) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= h * N) return;
  // consecutive warps take the g heads of one token (shared idx row)
  const int64_t t = wid / h, j = wid % h, kh = j / g;
  const int len = row_len(idx + (kh * N + t) * T, T, lane);
  const int64_t rb = (j * N + t) * (int64_t)T;
  const __nv_bfloat16* src = obuf + rb * kD + lane * 4;
  // every partial row of this (head, token) is requested before the slot
  // statistics are reduced: one memory latency per warp, not two
  uint2 raw[TMAX];
#pragma unroll
  for (int s = 0; s < TMAX; ++s)
    if (s < len) raw[s] = __ldcs(reinterpret_cast<const uint2*>(src + s * kD));
  float2 st = lane < len ? __ldg(ml + rb + lane) : make_float2(-INFINITY, 0.f);
  float cm[4], cs[4], tw[3];
  if (cmb.out) {
    ld4(cmb.out_cmp, (t * h + j) * kD + lane * 4, kNarrow, cm);
    ld4(cmb.out_slide, (t * h + j) * kD + lane * 4, kNarrow, cs);
    tw[0] = __ldg(cmb.tau + t * 3);
    tw[1] = __ldg(cmb.tau + t * 3 + 1);
    tw[2] = __ldg(cmb.tau + t * 3 + 2);
  }
  float M = st.x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float w = lane < len ? st.y * __expf(st.x - M) : 0.f;
  float L = w;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int s = 0; s < TMAX; ++s) {  // ascending block order
    if (s < len) {
      const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[s].x));
      const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw[s].y));
      const float ws = __shfl_sync(0xffffffffu, w, s);
      acc.x += ws * a.x; acc.y += ws * a.y; acc.z += ws * b.x; acc.w += ws * b.y;
    }
  }
  const float inv = 1.f / L;
  const float4 o = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  if (kNarrow) {
    const __nv_bfloat162 p0 = __floats2bfloat162_rn(o.x, o.y), p1 = __floats2bfloat162_rn(o.z, o.w);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&p0);
    u.y = *reinterpret_cast<const uint32_t*>(&p1);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + (t * h + j) * kD + lane * 4) = u;
  } else {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + (t * h + j) * kD + lane * 4) = o;
  }
  if (cmb.out) {
    const float ov[4] = {o.x, o.y, o.z, o.w};
    float r[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float x = 0.f + tw[0] * cm[c];
      x = x + tw[1] * ov[c];
      r[c] = x + tw[2] * cs[c];
    }
    const __nv_bfloat162 p0 = __floats2bfloat162_rn(r[0], r[1]);
    const __nv_bfloat162 p1 = __floats2bfloat162_rn(r[2], r[3]);
    uint2 u;
    u.x = *reinterpret_cast<const uint32_t*>(&p0);
    u.y = *reinterpret_cast<const uint32_t*>(&p1);
    *reinterpret_cast<uint2*>(cmb.out + (t * h + j) * kD + lane * 4) = u;
  }
  if (lane == 0) {
    if (lse) lse[j * N + t] = M + __logf(L);
    if (m_out) m_out[j * N + t] = M;
    if (l_out) l_out[j * N + t] = L;
  }
}

__global__ void dq_reduce_bf16_kernel(const int32_t* __restrict__ idx,
                                      const __nv_bfloat16* __restrict__ dq, float* __restrict__ dQ,
                                      int64_t N, int64_t h, int64_t g, int T,
                                      const void* __restrict__ addend, int addend_bf16) {
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
  if (addend) {  // another branch's dQ rows (the sliding window), added once
    const int64_t e = (t * h + j) * kD + lane * 4;
    const float4 a = addend_bf16 ? ld_bf16x4(reinterpret_cast<const __nv_bfloat16*>(addend) + e)
                                 : __ldcs(reinterpret_cast<const float4*>(addend) + e / 4);
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
  auto kern = s->T <= 16 ? merge_bf16_kernel<16, false> : merge_bf16_kernel<32, false>;
  kern<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      idx, (const __nv_bfloat16*)obuf, (const float2*)ml, out, (float*)lse, (float*)m_out,
      (float*)l_out, s->N, s->h, s->h / s->h_K, (int)s->T, Combine{});
  FSA_LAUNCH_CHECK("merge_bf16");
  return FSA_OK;
}

int merge_combine_bf16_fast(const fsa_shape* s, const int32_t* idx, const void* obuf,
                            const void* ml, const void* out_cmp, const void* out_slide,
                            const void* tau, void* out_sel, void* lse, void* out, cudaStream_t st,
                            int narrow) {
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  Combine c{out_cmp, out_slide, (const float*)tau, (__nv_bfloat16*)out};
  auto kern = narrow ? (s->T <= 16 ? merge_bf16_kernel<16, true> : merge_bf16_kernel<32, true>)
                     : (s->T <= 16 ? merge_bf16_kernel<16, false> : merge_bf16_kernel<32, false>);
  kern<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      idx, (const __nv_bfloat16*)obuf, (const float2*)ml, out_sel, (float*)lse, nullptr,
      nullptr, s->N, s->h, s->h / s->h_K, (int)s->T, c);
  FSA_LAUNCH_CHECK("merge_combine_bf16");
  return FSA_OK;
}

int dq_reduce_bf16_fast(const fsa_shape* s, const int32_t* idx, const void* dq, void* dQ,
                        cudaStream_t st, const void* addend, int addend_bf16) {
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  dq_reduce_bf16_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      idx, (const __nv_bfloat16*)dq, (float*)dQ, s->N, s->h, s->h / s->h_K, (int)s->T, addend,
      addend_bf16);
  FSA_LAUNCH_CHECK("dq_reduce_bf16");
  return FSA_OK;
}

}  // namespace fsa
