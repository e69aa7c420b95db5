// KV compression (K1), importance scores (generic), gated combine (K12),
// finiteness check.  HBM-bound kernels; see DESIGN.md for their byte counts.
#include "common.cuh"

namespace fsa {

// ---------------------------------------------------------------------------
// K1 compress_kv: branches.py:34-44.  One CTA per (block i, kv head); threads
// over features.  Block means in the accumulator type.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void compress_kernel(const T* __restrict__ K, const T* __restrict__ V,
                                typename Acc<T>::type* __restrict__ Kc,
                                typename Acc<T>::type* __restrict__ Vc, int64_t B_K, int64_t h_K,
                                int64_t dK, int64_t dV) {
  // blockIdx.z: 0 = K, 1 = V (one launch); 8 independent row accumulators per
  // column keep 8 loads in flight (the block's 64 rows are 64 strided reads)
  using A = typename Acc<T>::type;
  const T* X = blockIdx.z ? V : K;
  A* Xc = blockIdx.z ? Vc : Kc;
  const int64_t d = blockIdx.z ? dV : dK;
  const int64_t i = blockIdx.x, kh = blockIdx.y, stride = h_K * d;
  const A inv = A(1) / A(B_K);
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    const T* p = X + ((i * B_K) * h_K + kh) * d + c;
    A a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t r = 0;
    for (; r + 8 <= B_K; r += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] += to_acc(p[(r + j) * stride]);
    }
    for (; r < B_K; ++r) a[0] += to_acc(p[r * stride]);
    const A acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    Xc[(i * h_K + kh) * d + c] = acc * inv;
  }
}

// running prefix means of rows 0..t, t < n_pref (branches.py:40-43): one block
// per (t, tensor), rows summed in order (the reference's cumsum order)
template <typename T>
__global__ void prefix_kernel(const T* __restrict__ K, const T* __restrict__ V,
                              typename Acc<T>::type* __restrict__ Kp,
                              typename Acc<T>::type* __restrict__ Vp, int64_t h_K, int64_t dK,
                              int64_t dV) {
  using A = typename Acc<T>::type;
  const T* X = blockIdx.y ? V : K;
  A* Xp = blockIdx.y ? Vp : Kp;
  const int64_t w = h_K * (blockIdx.y ? dV : dK), t = blockIdx.x;
  for (int64_t idx = threadIdx.x; idx < w; idx += blockDim.x) {
    A acc = 0;
    for (int64_t r = 0; r <= t; ++r) acc += to_acc(X[r * w + idx]);
    Xp[t * w + idx] = acc / A(t + 1);
  }
}

// ---------------------------------------------------------------------------
// importance scores: selection.py:105-120.  CTA = 32 tokens of one kv head x
// all b blocks (chunks of 64 blocks staged in smem).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void scores_kernel(const T* __restrict__ Q, const typename Acc<T>::type* __restrict__ Kc,
                              typename Acc<T>::type* __restrict__ S, fsa_shape s, int64_t b) {
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* qs = reinterpret_cast<A*>(smem_raw);          // [32][d+1]
  const int64_t d = s.d_K, dp = d + 1;
  A* ks = qs + 32 * dp;                             // [64][d+1]
  const int64_t kh = blockIdx.y, t0 = blockIdx.x * 32;
  const int64_t g = s.h / s.h_K;
  for (int64_t e = threadIdx.x; e < 32 * d; e += blockDim.x) {
    int64_t r = e / d, c = e % d, t = t0 + r;
    A acc = 0;
    if (t < s.N)
      for (int64_t hh = 0; hh < g; ++hh) acc += to_acc(Q[(t * s.h + kh * g + hh) * d + c]);
    qs[r * dp + c] = acc;
  }
  const A mul = A(s.scale) / A(g);
  for (int64_t i0 = 0; i0 < b; i0 += 64) {
    __syncthreads();
    for (int64_t e = threadIdx.x; e < 64 * d; e += blockDim.x) {
      int64_t r = e / d, c = e % d;
      ks[r * dp + c] = (i0 + r < b) ? Kc[((i0 + r) * s.h_K + kh) * d + c] : A(0);
    }
    __syncthreads();
    const int col = threadIdx.x % 64;
    for (int r = threadIdx.x / 64; r < 32; r += blockDim.x / 64) {
      int64_t t = t0 + r, i = i0 + col;
      if (t >= s.N || i >= b) continue;
      A acc = 0;
      for (int64_t c = 0; c < d; ++c) acc += qs[r * dp + c] * ks[col * dp + c];
      S[(kh * s.N + t) * b + i] = acc * mul;
    }
  }
}

// ---------------------------------------------------------------------------
// K12 gated combine: branches.py:95-104 (sum order ((0 + t0*a) + t1*b) + t2*c).
// ---------------------------------------------------------------------------
// Branch outputs arrive in the accumulator dtype; the combined output is
// written in TO (the input dtype, or the accumulator dtype).
template <typename A, typename TO>
__global__ void combine_kernel(const A* __restrict__ a, const A* __restrict__ bsel,
                               const A* __restrict__ c, const A* __restrict__ tau,
                               TO* __restrict__ out, int64_t N, int64_t row) {
  // one CTA per token row (grid-stride): no per-element index division
  for (int64_t t = blockIdx.x; t < N; t += gridDim.x) {
    const A t0 = tau[t * 3 + 0], t1 = tau[t * 3 + 1], t2 = tau[t * 3 + 2];
    const int64_t base = t * row;
    for (int64_t e = threadIdx.x; e < row; e += blockDim.x) {
      A acc = A(0) + t0 * a[base + e];
      acc = acc + t1 * bsel[base + e];
      acc = acc + t2 * c[base + e];
      out[base + e] = from_acc<TO>(acc);
    }
  }
}

// dOut_c = tau[:, c] * dOut (gate backward into one branch, branches.py:103)
template <typename T>
__global__ void gate_scale_kernel(const T* __restrict__ d, const typename Acc<T>::type* __restrict__ tau,
                                  int col, T* __restrict__ out, int64_t N, int64_t row) {
  for (int64_t t = blockIdx.x; t < N; t += gridDim.x) {
    const auto w = tau[t * 3 + col];
    const int64_t base = t * row;
    for (int64_t e = threadIdx.x; e < row; e += blockDim.x)
      out[base + e] = from_acc<T>(w * to_acc(d[base + e]));
  }
}

// Fused gate backward + delta for the two differentiated branches
// (branches.py:103 then kv_major.py:284 / oracle.py:102-131):
//   dO_sel = tau[t,1] dOut,  dO_slide = tau[t,2] dOut   (rounded to T)
//   delta_sel[j,t] = sum_v out_sel[t,j,v] dO_sel[t,j,v], delta_slide alike,
// from the ROUNDED branch cotangents (the values the backward kernels read).
// One warp per (token, head) row.
template <typename T>
__global__ void gate_backward_kernel(const T* __restrict__ dOut,
                                     const typename Acc<T>::type* __restrict__ tau,
                                     const typename Acc<T>::type* __restrict__ out_sel,
                                     const typename Acc<T>::type* __restrict__ out_slide,
                                     T* __restrict__ d_sel, T* __restrict__ d_slide,
                                     typename Acc<T>::type* __restrict__ delta_sel,
                                     typename Acc<T>::type* __restrict__ delta_slide, int64_t N,
                                     int64_t h, int64_t dv) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= N * h) return;
  const int64_t t = wid / h, j = wid - t * h;
  const A w1 = tau[t * 3 + 1], w2 = tau[t * 3 + 2];
  const int64_t base = wid * dv;
  A s1 = 0, s2 = 0;
  if constexpr (sizeof(T) == 2) {
    if ((dv & 127) == 0) {
      for (int64_t c = lane * 4; c < dv; c += 128) {
        const uint2 u = *reinterpret_cast<const uint2*>(dOut + base + c);
        const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
        const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        const float4 o1 = *reinterpret_cast<const float4*>(out_sel + base + c);
        const float4 o2 = *reinterpret_cast<const float4*>(out_slide + base + c);
        const __nv_bfloat162 a0 = __floats2bfloat162_rn(w1 * x.x, w1 * x.y);
        const __nv_bfloat162 a1 = __floats2bfloat162_rn(w1 * y.x, w1 * y.y);
        const __nv_bfloat162 b0 = __floats2bfloat162_rn(w2 * x.x, w2 * x.y);
        const __nv_bfloat162 b1 = __floats2bfloat162_rn(w2 * y.x, w2 * y.y);
        uint2 ua, ub;
        ua.x = *reinterpret_cast<const uint32_t*>(&a0);
        ua.y = *reinterpret_cast<const uint32_t*>(&a1);
        ub.x = *reinterpret_cast<const uint32_t*>(&b0);
        ub.y = *reinterpret_cast<const uint32_t*>(&b1);
        *reinterpret_cast<uint2*>(d_sel + base + c) = ua;
        *reinterpret_cast<uint2*>(d_slide + base + c) = ub;
        const float2 fa0 = __bfloat1622float2(a0), fa1 = __bfloat1622float2(a1);
        const float2 fb0 = __bfloat1622float2(b0), fb1 = __bfloat1622float2(b1);
        s1 += o1.x * fa0.x + o1.y * fa0.y + o1.z * fa1.x + o1.w * fa1.y;
        s2 += o2.x * fb0.x + o2.y * fb0.y + o2.z * fb1.x + o2.w * fb1.y;
      }
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) {
        delta_sel[j * N + t] = s1;
        delta_slide[j * N + t] = s2;
      }
      return;
    }
  }
  for (int64_t c = lane; c < dv; c += 32) {
    const A x = to_acc(dOut[base + c]);
    const T a = from_acc<T>(w1 * x), b = from_acc<T>(w2 * x);
    d_sel[base + c] = a;
    d_slide[base + c] = b;
    s1 += out_sel[base + c] * to_acc(a);
    s2 += out_slide[base + c] * to_acc(b);
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    delta_sel[j * N + t] = s1;
    delta_slide[j * N + t] = s2;
  }
}

template <typename T>
__global__ void finite_kernel(const T* __restrict__ x, int64_t n, int32_t* flag) {
  int bad = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite((double)to_acc(x[e]));
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename T>
int compress_impl(const fsa_shape* s, const void* K, const void* V, void* Kc, void* Vc, void* Kp,
                  void* Vp, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t b = s->N / s->B_K, n_pref = s->B_K - 1 < s->N ? s->B_K - 1 : s->N;
  if (b > 0) {
    dim3 grid((unsigned)b, (unsigned)s->h_K, 2);
    compress_kernel<T><<<grid, 128, 0, st>>>((const T*)K, (const T*)V, (A*)Kc, (A*)Vc, s->B_K,
                                             s->h_K, s->d_K, s->d_V);
  }
  if (n_pref > 0) {
    dim3 grid((unsigned)n_pref, 2);
    prefix_kernel<T><<<grid, 256, 0, st>>>((const T*)K, (const T*)V, (A*)Kp, (A*)Vp, s->h_K,
                                           s->d_K, s->d_V);
  }
  FSA_LAUNCH_CHECK("compress_kv");
  return FSA_OK;
}

template <typename T>
int scores_impl(const fsa_shape* s, const void* Q, const void* Kc, void* S, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t b = s->N / s->B_K;
  size_t smem = (size_t)(32 + 64) * (s->d_K + 1) * sizeof(A);
  FSA_REQUIRE(smem <= 200 * 1024, "importance scores: d_K=%lld too large", (long long)s->d_K);
  cudaFuncSetAttribute(scores_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)((s->N + 31) / 32), (unsigned)s->h_K);
  scores_kernel<T><<<grid, 256, smem, st>>>((const T*)Q, (const A*)Kc, (A*)S, *s, b);
  FSA_LAUNCH_CHECK("importance_scores");
  return FSA_OK;
}

template <typename T>
int combine_impl(const fsa_shape* s, const void* a, const void* b, const void* c, const void* tau,
                 void* out, int out_acc, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t row = s->h * s->d_V;
  int64_t blocks = s->N < 148 * 16 ? s->N : 148 * 16;
  if (blocks < 1) return FSA_OK;
  if (out_acc)
    combine_kernel<A, A><<<(unsigned)blocks, 256, 0, st>>>((const A*)a, (const A*)b, (const A*)c,
                                                          (const A*)tau, (A*)out, s->N, row);
  else
    combine_kernel<A, T><<<(unsigned)blocks, 256, 0, st>>>((const A*)a, (const A*)b, (const A*)c,
                                                          (const A*)tau, (T*)out, s->N, row);
  FSA_LAUNCH_CHECK("gated_combine");
  return FSA_OK;
}

template <typename T>
int gate_scale_impl(const fsa_shape* s, const void* d, const void* tau, int col, void* out,
                    cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t row = s->h * s->d_V;
  int64_t blocks = s->N < 148 * 16 ? s->N : 148 * 16;
  if (blocks < 1) return FSA_OK;
  gate_scale_kernel<T><<<(unsigned)blocks, 256, 0, st>>>((const T*)d, (const A*)tau, col, (T*)out,
                                                        s->N, row);
  FSA_LAUNCH_CHECK("gate_scale");
  return FSA_OK;
}

template <typename T>
int gate_backward_impl(const fsa_shape* s, const void* dOut, const void* tau, const void* out_sel,
                       const void* out_slide, void* d_sel, void* d_slide, void* delta_sel,
                       void* delta_slide, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t rows = s->N * s->h;
  if (rows == 0) return FSA_OK;
  gate_backward_kernel<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      (const T*)dOut, (const A*)tau, (const A*)out_sel, (const A*)out_slide, (T*)d_sel,
      (T*)d_slide, (A*)delta_sel, (A*)delta_slide, s->N, s->h, s->d_V);
  FSA_LAUNCH_CHECK("gate_backward");
  return FSA_OK;
}

// Gate backward folded into the branches' softmax statistics (tensor-core
// path): with d_c = tau_c[t] * dOut, every backward quantity of branch c is
// tau_c[t] times its value for the raw dOut (dP, dS, the dV product), and
// tau * exp(z - lse) = exp(z - (lse - ln tau)).  So the branch kernels take the
// raw dOut with lse_c - ln tau_c and delta_c = sum_v out_c * dOut -- no gated
// copies of dOut are written (nor rounded to bf16).  Warp per (token, head).
template <typename T, typename B = typename Acc<T>::type>  // B: branch-output element type
__global__ void gate_fold_kernel(const T* __restrict__ dOut, const typename Acc<T>::type* __restrict__ tau,
                                 const B* __restrict__ out_sel, const B* __restrict__ out_slide,
                                 const typename Acc<T>::type* __restrict__ lse_sel,
                                 const typename Acc<T>::type* __restrict__ lse_slide,
                                 typename Acc<T>::type* __restrict__ delta_sel,
                                 typename Acc<T>::type* __restrict__ delta_slide,
                                 typename Acc<T>::type* __restrict__ lse_sel_adj,
                                 typename Acc<T>::type* __restrict__ lse_slide_adj, int64_t N, int64_t h,
                                 int64_t dv) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= N * h) return;
  const int64_t t = wid / h, j = wid - t * h;
  const int64_t base = wid * dv;
  A s1 = 0, s2 = 0;
  for (int64_t c = lane; c < dv; c += 32) {
    const A x = to_acc(dOut[base + c]);
    s1 += A(to_acc(out_sel[base + c])) * x;
    s2 += A(to_acc(out_slide[base + c])) * x;
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    const int64_t r = j * N + t;
    delta_sel[r] = s1;
    delta_slide[r] = s2;
    lse_sel_adj[r] = lse_sel[r] - log_acc(tau[t * 3 + 1]);  // tau = 0: +inf, P = 0
    lse_slide_adj[r] = lse_slide[r] - log_acc(tau[t * 3 + 2]);
  }
}

// bf16 dOut, fp32 branch outputs, d_V = 128: a warp per (token, head) row,
// 16-byte branch-output loads and 8-byte dOut loads
__global__ void __launch_bounds__(256) gate_fold_d128_kernel(
    const __nv_bfloat16* __restrict__ dOut, const float* __restrict__ tau,
    const float* __restrict__ out_sel, const float* __restrict__ out_slide,
    const float* __restrict__ lse_sel, const float* __restrict__ lse_slide,
    float* __restrict__ delta_sel, float* __restrict__ delta_slide,
    float* __restrict__ lse_sel_adj, float* __restrict__ lse_slide_adj, int64_t N, int64_t h) {
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= N * h) return;
  const int64_t e = row * 128 + lane * 4;
  const uint2 x = __ldg(reinterpret_cast<const uint2*>(dOut + e));
  const float4 a = __ldcs(reinterpret_cast<const float4*>(out_sel + e));
  const float4 b = __ldcs(reinterpret_cast<const float4*>(out_slide + e));
  const float2 x0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x.x));
  const float2 x1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&x.y));
  float s1 = a.x * x0.x + a.y * x0.y + a.z * x1.x + a.w * x1.y;
  float s2 = b.x * x0.x + b.y * x0.y + b.z * x1.x + b.w * x1.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  if (lane == 0) {
    const int64_t t = row / h, j = row - t * h, r = j * N + t;
    delta_sel[r] = s1;
    delta_slide[r] = s2;
    lse_sel_adj[r] = lse_sel[r] - logf(tau[t * 3 + 1]);
    lse_slide_adj[r] = lse_slide[r] - logf(tau[t * 3 + 2]);
  }
}

template <typename T>
int gate_fold_impl(const fsa_shape* s, const void* dOut, const void* tau, const void* out_sel,
                   const void* out_slide, const void* lse_sel, const void* lse_slide, void* delta_sel,
                   void* delta_slide, void* lse_sel_adj, void* lse_slide_adj, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t rows = s->N * s->h;
  if (rows == 0) return FSA_OK;
  if (sizeof(T) == 2 && s->d_V == 128)
    gate_fold_d128_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
        (const __nv_bfloat16*)dOut, (const float*)tau, (const float*)out_sel,
        (const float*)out_slide, (const float*)lse_sel, (const float*)lse_slide,
        (float*)delta_sel, (float*)delta_slide, (float*)lse_sel_adj, (float*)lse_slide_adj, s->N, s->h);
  else
    gate_fold_kernel<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
        (const T*)dOut, (const A*)tau, (const A*)out_sel, (const A*)out_slide, (const A*)lse_sel,
        (const A*)lse_slide, (A*)delta_sel, (A*)delta_slide, (A*)lse_sel_adj, (A*)lse_slide_adj, s->N,
        s->h, s->d_V);
  FSA_LAUNCH_CHECK("gate_backward_fold");
  return FSA_OK;
}

template <typename T>
int finite_impl(const void* x, int64_t n, int32_t* flag, cudaStream_t st) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  finite_kernel<T><<<(unsigned)blocks, 256, 0, st>>>((const T*)x, n, flag);
  FSA_LAUNCH_CHECK("check_finite");
  return FSA_OK;
}

}  // namespace fsa

#define DISPATCH_DT(dt, FN, ...)                                            \
  switch (dt) {                                                             \
    case FSA_DT_F32: return fsa::FN<float>(__VA_ARGS__);                    \
    case FSA_DT_F64: return fsa::FN<double>(__VA_ARGS__);                   \
    case FSA_DT_BF16: return fsa::FN<__nv_bfloat16>(__VA_ARGS__);           \
    default: fsa::set_error("unsupported dtype %d", (int)dt); return FSA_ERR_INVALID; \
  }

extern "C" int fsa_compress_kv(const fsa_shape* s, int dtype, const void* K, const void* V,
                               void* K_cmp, void* V_cmp, void* K_prefix, void* V_prefix,
                               void* stream) {
  DISPATCH_DT(dtype, compress_impl, s, K, V, K_cmp, V_cmp, K_prefix, V_prefix, (cudaStream_t)stream);
}

extern "C" int fsa_importance_scores(const fsa_shape* s, int dtype, const void* Q, const void* K_cmp,
                                     void* scores, void* stream) {
  DISPATCH_DT(dtype, scores_impl, s, Q, K_cmp, scores, (cudaStream_t)stream);
}

extern "C" int fsa_gated_combine(const fsa_shape* s, int dtype, const void* out_cmp,
                                 const void* out_sel, const void* out_slide, const void* tau,
                                 void* out, int out_acc, void* stream) {
  DISPATCH_DT(dtype, combine_impl, s, out_cmp, out_sel, out_slide, tau, out, out_acc,
              (cudaStream_t)stream);
}

extern "C" int fsa_gate_scale(const fsa_shape* s, int dtype, const void* dOut, const void* tau,
                              int col, void* out, void* stream) {
  DISPATCH_DT(dtype, gate_scale_impl, s, dOut, tau, col, out, (cudaStream_t)stream);
}

extern "C" int fsa_gate_backward(const fsa_shape* s, int dtype, const void* dOut, const void* tau,
                                 const void* out_sel, const void* out_slide, void* d_sel,
                                 void* d_slide, void* delta_sel, void* delta_slide, void* stream) {
  DISPATCH_DT(dtype, gate_backward_impl, s, dOut, tau, out_sel, out_slide, d_sel, d_slide, delta_sel,
              delta_slide, (cudaStream_t)stream);
}

extern "C" int fsa_gate_backward_fold(const fsa_shape* s, int dtype, const void* dOut, const void* tau,
                                      const void* out_sel, const void* out_slide, const void* lse_sel,
                                      const void* lse_slide, void* delta_sel, void* delta_slide,
                                      void* lse_sel_adj, void* lse_slide_adj, void* stream) {
  DISPATCH_DT(dtype, gate_fold_impl, s, dOut, tau, out_sel, out_slide, lse_sel, lse_slide, delta_sel,
              delta_slide, lse_sel_adj, lse_slide_adj, (cudaStream_t)stream);
}

extern "C" int fsa_check_finite(int dtype, const void* x, int64_t n, int32_t* flag, void* stream) {
  if (n == 0) return FSA_OK;
  DISPATCH_DT(dtype, finite_impl, x, n, flag, (cudaStream_t)stream);
}
