// HBM-bound reductions of the tensor-core path (d = 128, fp16 partials):
//   K6 merge (kv_major.py:207-242, fused LOCAL form): per (head j, token t) the
//      <= T per-block partials O_s / l_s (fp16, in the scale s_kh of the V16
//      copy) and (m_s, l_s) are combined in ascending block order:
//      M = max m_s, w_s = l_s e^{m_s - M}, L = sum w_s,
//      out = (sum_s w_s O_s) / (L s_kh), lse = M + ln L.
//   K9 dQ reduce (kv_major.py:326-340): dQ[t, j] = sum_s dq_s 2^{-e_s},
//      ascending s, from fp16 rows with a per-row power-of-two exponent e_s.
// One warp per (j, t): lane k owns dims 4k..4k+3 (8-byte fp16 loads, 16-byte
// fp32 stores -> every partial row is one coalesced 256 B request); the slot
// statistics live one per lane and are reduced with shuffles.
// The partial rows are item-major (common.cuh, work plan): slot s of (kh, t)
// names block i = idx[kh][t][s] at list position p = pos[kh][t][s], i.e. row
// 128 (item[kh b + i] + p / tpi) + (p % tpi) g + hh of the buffers.
#include "common.cuh"
#include <cuda_fp16.h>

namespace fsa {
namespace {

constexpr int kD = 128;

__device__ __forceinline__ float4 h4(uint2 u) {
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ int row_len(const int32_t* row, int T, int lane) {
  int len = 0;
  for (int c = 0; c < T; c += 32) {  // entries are a prefix (validated selection)
    const int v = c + lane < T ? __ldg(row + c + lane) : -1;
    const int n = __popc(__ballot_sync(0xffffffffu, v != -1));
    len += n;
    if (n < 32) break;
  }
  return len;
}

// Gated-combine epilogue (branches.py:95-104): with cmb.out != null the warp
// also writes out = ((0 + tau0 out_cmp) + tau1 out_sel) + tau2 out_slide (bf16);
// out_cmp / out_slide in fp32.
struct Combine {
  const float* out_cmp;
  const float* out_slide;
  const float* tau;
  __nv_bfloat16* out;
};

// item-major partial rows (common.cuh, work plan)
struct ItemRows {
  const int32_t* item;   // item prefix per chunked task [ntask + 1]
  const int32_t* pos;    // sub-list position per (kh, t, slot) [h_K][N][T]
  const int32_t* cbase;  // task base of each token chunk within a kv head
  int64_t N;
  int C, nph, tpi, g;
  // row of slot s of (kh, t) -- its block blk -- for group head hh
  __device__ __forceinline__ int64_t row(int64_t kh, int64_t t, int T, int s, int blk, int hh) const {
    const int p = __ldg(pos + (kh * N + t) * T + s);
    const int64_t task = kh * nph + __ldg(cbase + t / C) + blk;
    const int it = __ldg(item + task) + p / tpi;
    return (int64_t)it * 128 + (int64_t)(p % tpi) * g + hh;
  }
};

template <int TMAX>  // TMAX >= T: partial rows held in registers
__global__ void __launch_bounds__(256) merge_f16_kernel(
    const int32_t* __restrict__ idx, const __half* __restrict__ obuf,
    const float2* __restrict__ ml, const float* __restrict__ vscale, float* __restrict__ out,
    float* __restrict__ lse, float* __restrict__ m_out, float* __restrict__ l_out, int64_t N,
    int64_t h, int64_t g, int T, Combine cmb, ItemRows ir) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= h * N) return;
  // consecutive warps take the g heads of one token (shared idx row)
  const int64_t t = wid / h, j = wid % h, kh = j / g;
  const int32_t* irow = idx + (kh * N + t) * T;
  const int len = row_len(irow, T, lane);
  const int64_t my = lane < len ? ir.row(kh, t, T, lane, __ldg(irow + lane), (int)(j - kh * g)) : 0;
  // every partial row of this (head, token) is requested before the slot
  // statistics are reduced: one memory latency per warp, not two
  uint2 raw[TMAX];
#pragma unroll
  for (int s = 0; s < TMAX; ++s) {
    const int64_t rs = __shfl_sync(0xffffffffu, my, s & 31);
    if (s < len) raw[s] = __ldcs(reinterpret_cast<const uint2*>(obuf + rs * kD + lane * 4));
  }
  float2 st = lane < len ? __ldg(ml + my) : make_float2(-INFINITY, 0.f);
  float4 cm = make_float4(0.f, 0.f, 0.f, 0.f), cs = cm;
  float tw[3];
  if (cmb.out) {
    cm = __ldcs(reinterpret_cast<const float4*>(cmb.out_cmp + (t * h + j) * kD) + lane);
    cs = __ldcs(reinterpret_cast<const float4*>(cmb.out_slide + (t * h + j) * kD) + lane);
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
      const float4 a = h4(raw[s]);
      const float ws = __shfl_sync(0xffffffffu, w, s);
      acc.x += ws * a.x; acc.y += ws * a.y; acc.z += ws * a.z; acc.w += ws * a.w;
    }
  }
  const float inv = 1.f / (L * __ldg(vscale + kh));
  const float4 o = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  reinterpret_cast<float4*>(out + (t * h + j) * kD)[lane] = o;
  if (cmb.out) {
    const float ov[4] = {o.x, o.y, o.z, o.w}, cv[4] = {cm.x, cm.y, cm.z, cm.w},
                sv[4] = {cs.x, cs.y, cs.z, cs.w};
    float r[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float x = 0.f + tw[0] * cv[c];
      x = x + tw[1] * ov[c];
      r[c] = x + tw[2] * sv[c];
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

// T > 32: the partials stream through in slot order (two passes over ml)
__global__ void __launch_bounds__(256) merge_f16_long_kernel(
    const int32_t* __restrict__ idx, const __half* __restrict__ obuf,
    const float2* __restrict__ ml, const float* __restrict__ vscale, float* __restrict__ out,
    float* __restrict__ lse, float* __restrict__ m_out, float* __restrict__ l_out, int64_t N,
    int64_t h, int64_t g, int T, Combine cmb, ItemRows ir) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= h * N) return;
  const int64_t t = wid / h, j = wid % h, kh = j / g;
  const int32_t* irow = idx + (kh * N + t) * T;
  const int len = row_len(irow, T, lane);
  const int hh = (int)(j - kh * g);
  float M = -INFINITY;
  for (int s = lane; s < len; s += 32) M = fmaxf(M, __ldg(ml + ir.row(kh, t, T, s, __ldg(irow + s), hh)).x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c = 0; c < len; c += 32) {
    const int64_t my = c + lane < len ? ir.row(kh, t, T, c + lane, __ldg(irow + c + lane), hh) : 0;
    const float2 st = c + lane < len ? __ldg(ml + my) : make_float2(-INFINITY, 0.f);
    const float w = c + lane < len ? st.y * __expf(st.x - M) : 0.f;
    const int n = len - c < 32 ? len - c : 32;
    for (int s = 0; s < n; ++s) {  // ascending block order
      const float ws = __shfl_sync(0xffffffffu, w, s);
      const int64_t rs = __shfl_sync(0xffffffffu, my, s);
      const float4 a = h4(__ldcs(reinterpret_cast<const uint2*>(obuf + rs * kD + lane * 4)));
      acc.x += ws * a.x; acc.y += ws * a.y; acc.z += ws * a.z; acc.w += ws * a.w;
      L += ws;
    }
  }
  const float inv = 1.f / (L * __ldg(vscale + kh));
  const float4 o = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  reinterpret_cast<float4*>(out + (t * h + j) * kD)[lane] = o;
  if (cmb.out) {
    const float4 cm = reinterpret_cast<const float4*>(cmb.out_cmp + (t * h + j) * kD)[lane];
    const float4 cs = reinterpret_cast<const float4*>(cmb.out_slide + (t * h + j) * kD)[lane];
    const float t0 = __ldg(cmb.tau + t * 3), t1 = __ldg(cmb.tau + t * 3 + 1),
                t2 = __ldg(cmb.tau + t * 3 + 2);
    const float ov[4] = {o.x, o.y, o.z, o.w}, cv[4] = {cm.x, cm.y, cm.z, cm.w},
                sv[4] = {cs.x, cs.y, cs.z, cs.w};
    float r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float x = 0.f + t0 * cv[k];
      x = x + t1 * ov[k];
      r[k] = x + t2 * sv[k];
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

// dq partial buffer (FSA_DT_F16R): fp16 rows [h][N][T][128] then 4 int8
// exponents per row (one per 32 columns) [h][N][T]; value = fp16 * 2^-e.
__global__ void __launch_bounds__(256) dq_reduce_f16r_kernel(
    const int32_t* __restrict__ idx, const __half* __restrict__ dq, const int32_t* __restrict__ dqe,
    float* __restrict__ dQ, int64_t N, int64_t h, int64_t g, int T, const float* __restrict__ addend) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= h * N) return;
  const int64_t t = wid / h, j = wid % h, kh = j / g;
  const int len = row_len(idx + (kh * N + t) * T, T, lane);
  const int64_t rb = (j * N + t) * (int64_t)T;
  const __half* src = dq + rb * kD + lane * 4;
  const int sh = 8 * (lane >> 3);  // this lane's 32-column chunk: exponent byte
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c = 0; c < len; c += 32) {
    const int32_t e4 = c + lane < len ? __ldg(dqe + rb + c + lane) : 0;
    const int n = len - c < 32 ? len - c : 32;
    int s = 0;
    for (; s + 4 <= n; s += 4) {  // four rows in flight per step
      uint2 r[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = __ldcs(reinterpret_cast<const uint2*>(src + (c + s + k) * kD));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t e = __shfl_sync(0xffffffffu, e4, s + k);
        const float m = ldexpf(1.f, -(int)(int8_t)(e >> sh));
        const float4 a = h4(r[k]);
        acc.x += a.x * m; acc.y += a.y * m; acc.z += a.z * m; acc.w += a.w * m;
      }
    }
    for (; s < n; ++s) {
      const int32_t e = __shfl_sync(0xffffffffu, e4, s);
      const float m = ldexpf(1.f, -(int)(int8_t)(e >> sh));
      const float4 a = h4(__ldcs(reinterpret_cast<const uint2*>(src + (c + s) * kD)));
      acc.x += a.x * m; acc.y += a.y * m; acc.z += a.z * m; acc.w += a.w * m;
    }
  }
  if (addend) {  // another branch's dQ rows (the sliding window), added once
    const float4 a = __ldcs(reinterpret_cast<const float4*>(addend + (t * h + j) * kD) + lane);
    acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w;
  }
  reinterpret_cast<float4*>(dQ + (t * h + j) * kD)[lane] = acc;
}

}  // namespace

bool fast_reduce_ok(const fsa_shape& s) { return s.d_V == kD && s.d_K == kD; }

ItemRows item_rows(const fsa_shape* s, const int32_t* work) {
  const PlanView v = plan_view(*s, work);
  ItemRows ir;
  ir.item = v.item;
  ir.pos = v.pos;
  ir.cbase = v.cbase;
  ir.N = s->N;
  ir.C = v.C;
  ir.nph = v.nph;
  ir.tpi = (int)plan_tpi(*s);
  ir.g = (int)(s->h / s->h_K);
  return ir;
}

int merge_f16_fast(const fsa_shape* s, const int32_t* idx, const int32_t* work, const void* obuf,
                   const void* ml, const float* vscale, void* out, void* lse, void* m_out,
                   void* l_out, cudaStream_t st, const void* out_cmp, const void* out_slide,
                   const void* tau, void* out_comb) {
  FSA_REQUIRE(vscale != nullptr, "merge: fp16 partials need the V16 scales (vscale)");
  FSA_REQUIRE(work != nullptr, "merge: item-major fp16 partials need the work plan");
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  Combine c{(const float*)out_cmp, (const float*)out_slide, (const float*)tau,
            (__nv_bfloat16*)out_comb};
  auto kern = s->T <= 16 ? merge_f16_kernel<16> : s->T <= 32 ? merge_f16_kernel<32> : merge_f16_long_kernel;
  kern<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      idx, (const __half*)obuf, (const float2*)ml, vscale, (float*)out, (float*)lse,
      (float*)m_out, (float*)l_out, s->N, s->h, s->h / s->h_K, (int)s->T, c, item_rows(s, work));
  FSA_LAUNCH_CHECK("merge_f16");
  return FSA_OK;
}

int dq_reduce_f16r(const fsa_shape* s, const int32_t* idx, const void* dq, void* dQ,
                   cudaStream_t st, const void* addend) {
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  const __half* rows16 = (const __half*)dq;
  const int32_t* ex = (const int32_t*)(rows16 + rows * s->T * kD);
  dq_reduce_f16r_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      idx, rows16, ex, (float*)dQ, s->N, s->h, s->h / s->h_K, (int)s->T, (const float*)addend);
  FSA_LAUNCH_CHECK("dq_reduce_f16r");
  return FSA_OK;
}

}  // namespace fsa
