// Compressed and sliding-window branches, generic SIMT path (f32/f64 and
// small bf16 shapes).  One warp per (query head, token); deterministic.
//   compressed fwd  branches.py:47-78
//   sliding fwd     branches.py:81-83 -> oracle.py:39-44, :64-74
//   sliding bwd     oracle.py:102-131 restricted to band_mask
#include "common.cuh"
#include "tc_plan.cuh"

namespace fsa {

template <typename T, typename KT>
__device__ __forceinline__ typename Acc<T>::type dot_row(const T* q, const KT* k, int64_t d) {
  typename Acc<T>::type acc = 0;
  for (int64_t c = 0; c < d; ++c) acc += to_acc(q[c]) * to_acc(k[c]);
  return acc;
}

// ---------------------------------------------------------------------------
// compressed attention: token t attends the (t+1)//B_K formed pooled rows;
// pending tokens copy their prefix row (branches.py:72-77).
// ---------------------------------------------------------------------------
template <typename T, typename O = typename Acc<T>::type>  // O: out element type
__global__ void cmp_fwd_generic(const T* __restrict__ Q, const typename Acc<T>::type* __restrict__ Kc,
                                const typename Acc<T>::type* __restrict__ Vc,
                                const typename Acc<T>::type* __restrict__ Kp,
                                const typename Acc<T>::type* __restrict__ Vp, O* __restrict__ out,
                                typename Acc<T>::type* __restrict__ lse, fsa_shape s,
                                int64_t ntok) {
  // ntok < N: only the first ntok tokens (the pending ones on the tensor-core path)
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.h * ntok) return;
  const int64_t j = wid / ntok, t = wid % ntok, g = s.h / s.h_K, kh = j / g;
  const int64_t dK = s.d_K, dV = s.d_V;
  const T* q = Q + (t * s.h + j) * dK;
  O* o = out + (t * s.h + j) * dV;
  const int64_t nf = (t + 1) / s.B_K;
  const A scale = A(s.scale);
  if (nf == 0) {
    const A* kp = Kp + (t * s.h_K + kh) * dK;
    A acc = 0;
    for (int64_t c = lane; c < dK; c += 32) acc += to_acc(q[c]) * kp[c];
    acc = warp_sum(acc);
    for (int64_t c = lane; c < dV; c += 32) o[c] = from_acc<O>(Vp[(t * s.h_K + kh) * dV + c]);
    if (lane == 0) lse[j * s.N + t] = acc * scale;
    return;
  }
  A m = neg_inf<A>();
  for (int64_t i = lane; i < nf; i += 32) m = fmax(m, dot_row<T, A>(q, Kc + (i * s.h_K + kh) * dK, dK) * scale);
  m = warp_max(m);
  A l = 0;
  for (int64_t c0 = 0; c0 < dV; c0 += 32) {
    A acc = 0;
    for (int64_t i0 = 0; i0 < nf; i0 += 32) {
      const int64_t i = i0 + lane;
      A p = 0;
      if (i < nf) p = exp_acc(dot_row<T, A>(q, Kc + (i * s.h_K + kh) * dK, dK) * scale - m);
      if (c0 == 0) l += p;
      const int64_t cnt = min((int64_t)32, nf - i0);
      for (int64_t k = 0; k < cnt; ++k) {
        const A pk = __shfl_sync(0xffffffffu, p, (int)k);
        if (c0 + lane < dV) acc += pk * Vc[((i0 + k) * s.h_K + kh) * dV + c0 + lane];
      }
    }
    if (c0 == 0) l = warp_sum(l);
    if (c0 + lane < dV) o[c0 + lane] = from_acc<O>(acc / l);
  }
  if (lane == 0) lse[j * s.N + t] = m + log_acc(l);
}

// ---------------------------------------------------------------------------
// sliding window forward: keys s in [t-W+1, t]
// ---------------------------------------------------------------------------
template <typename T>
__global__ void slide_fwd_generic(const T* __restrict__ Q, const T* __restrict__ K,
                                  const T* __restrict__ V, typename Acc<T>::type* __restrict__ out,
                                  typename Acc<T>::type* __restrict__ lse, fsa_shape s) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.h * s.N) return;
  const int64_t j = wid / s.N, t = wid % s.N, g = s.h / s.h_K, kh = j / g;
  const int64_t dK = s.d_K, dV = s.d_V;
  const int64_t lo = t - s.W + 1 > 0 ? t - s.W + 1 : 0, nk = t - lo + 1;
  const T* q = Q + (t * s.h + j) * dK;
  const A scale = A(s.scale);
  A m = neg_inf<A>();
  for (int64_t k = lane; k < nk; k += 32)
    m = fmax(m, dot_row<T, T>(q, K + ((lo + k) * s.h_K + kh) * dK, dK) * scale);
  m = warp_max(m);
  A l = 0;
  for (int64_t c0 = 0; c0 < dV; c0 += 32) {
    A acc = 0;
    for (int64_t k0 = 0; k0 < nk; k0 += 32) {
      const int64_t k = k0 + lane;
      A p = 0;
      if (k < nk) p = exp_acc(dot_row<T, T>(q, K + ((lo + k) * s.h_K + kh) * dK, dK) * scale - m);
      if (c0 == 0) l += p;
      const int64_t cnt = min((int64_t)32, nk - k0);
      for (int64_t kk = 0; kk < cnt; ++kk) {
        const A pk = __shfl_sync(0xffffffffu, p, (int)kk);
        if (c0 + lane < dV) acc += pk * to_acc(V[((lo + k0 + kk) * s.h_K + kh) * dV + c0 + lane]);
      }
    }
    if (c0 == 0) l = warp_sum(l);
    if (c0 + lane < dV) out[(t * s.h + j) * dV + c0 + lane] = acc / l;
  }
  if (lane == 0) lse[j * s.N + t] = m + log_acc(l);
}

// dQ: warp per (j, t)
template <typename T>
__global__ void slide_bwd_dq_generic(const T* __restrict__ Q, const T* __restrict__ K,
                                     const T* __restrict__ V, const T* __restrict__ dOut,
                                     const typename Acc<T>::type* __restrict__ lse,
                                     const typename Acc<T>::type* __restrict__ delta,
                                     typename Acc<T>::type* __restrict__ dQ, fsa_shape s) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.h * s.N) return;
  const int64_t j = wid / s.N, t = wid % s.N, g = s.h / s.h_K, kh = j / g;
  const int64_t dK = s.d_K, dV = s.d_V;
  const int64_t lo = t - s.W + 1 > 0 ? t - s.W + 1 : 0, nk = t - lo + 1;
  const T* q = Q + (t * s.h + j) * dK;
  const T* d = dOut + (t * s.h + j) * dV;
  const A scale = A(s.scale), lr = lse[j * s.N + t], dr = delta[j * s.N + t];
  for (int64_t c0 = 0; c0 < dK; c0 += 32) {
    A acc = 0;
    for (int64_t k0 = 0; k0 < nk; k0 += 32) {
      const int64_t k = k0 + lane;
      A dz = 0;
      if (k < nk) {
        const int64_t row = (lo + k) * s.h_K + kh;
        const A p = exp_acc(dot_row<T, T>(q, K + row * dK, dK) * scale - lr);
        dz = p * (dot_row<T, T>(d, V + row * dV, dV) - dr);
      }
      const int64_t cnt = min((int64_t)32, nk - k0);
      for (int64_t kk = 0; kk < cnt; ++kk) {
        const A z = __shfl_sync(0xffffffffu, dz, (int)kk);
        if (c0 + lane < dK) acc += z * to_acc(K[((lo + k0 + kk) * s.h_K + kh) * dK + c0 + lane]);
      }
    }
    if (c0 + lane < dK) dQ[(t * s.h + j) * dK + c0 + lane] = acc * scale;
  }
}

// dK/dV: warp per (kh, key s); queries t in [s, s+W-1], heads of the group
template <typename T>
__global__ void slide_bwd_dkdv_generic(const T* __restrict__ Q, const T* __restrict__ K,
                                       const T* __restrict__ V, const T* __restrict__ dOut,
                                       const typename Acc<T>::type* __restrict__ lse,
                                       const typename Acc<T>::type* __restrict__ delta,
                                       typename Acc<T>::type* __restrict__ dKo,
                                       typename Acc<T>::type* __restrict__ dVo, fsa_shape s) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.h_K * s.N) return;
  const int64_t kh = wid / s.N, sk = wid % s.N, g = s.h / s.h_K;
  const int64_t dK = s.d_K, dV = s.d_V;
  const int64_t hi = sk + s.W - 1 < s.N - 1 ? sk + s.W - 1 : s.N - 1, nq = hi - sk + 1;
  const T* kr = K + (sk * s.h_K + kh) * dK;
  const T* vr = V + (sk * s.h_K + kh) * dV;
  const A scale = A(s.scale);
  for (int64_t c0 = 0; c0 < (dK > dV ? dK : dV); c0 += 32) {
    A ak = 0, av = 0;
    for (int64_t hh = 0; hh < g; ++hh) {
      const int64_t j = kh * g + hh;
      for (int64_t q0 = 0; q0 < nq; q0 += 32) {
        const int64_t t = sk + q0 + lane;
        A p = 0, dz = 0;
        if (q0 + lane < nq) {
          p = exp_acc(dot_row<T, T>(Q + (t * s.h + j) * dK, kr, dK) * scale - lse[j * s.N + t]);
          dz = p * (dot_row<T, T>(dOut + (t * s.h + j) * dV, vr, dV) - delta[j * s.N + t]);
        }
        const int64_t cnt = min((int64_t)32, nq - q0);
        for (int64_t kk = 0; kk < cnt; ++kk) {
          const A pk = __shfl_sync(0xffffffffu, p, (int)kk);
          const A zk = __shfl_sync(0xffffffffu, dz, (int)kk);
          const int64_t tt = sk + q0 + kk;
          if (c0 + lane < dK) ak += zk * to_acc(Q[(tt * s.h + j) * dK + c0 + lane]);
          if (c0 + lane < dV) av += pk * to_acc(dOut[(tt * s.h + j) * dV + c0 + lane]);
        }
      }
    }
    if (c0 + lane < dK) dKo[(sk * s.h_K + kh) * dK + c0 + lane] = ak * scale;
    if (c0 + lane < dV) dVo[(sk * s.h_K + kh) * dV + c0 + lane] = av;
  }
}

template <typename T>
int cmp_fwd_impl(const fsa_shape* s, const void* Q, const void* Kc, const void* Vc, const void* Kp,
                 const void* Vp, void* out, void* lse, void* scores, void* workspace,
                 const void* Q16, const float* qscale, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int dt = sizeof(T) == 8 ? FSA_DT_F64 : (sizeof(T) == 4 ? FSA_DT_F32 : FSA_DT_BF16);
  const bool tc = tc_qo_supported(*s, dt) && workspace != nullptr;
  // tensor-core path: formed tokens on tcgen05 (its tile stores write the
  // pending rows as 0), then the < B_K - 1 pending ones here
  const int64_t ntok = tc ? (s->B_K - 1 < s->N ? s->B_K - 1 : s->N) : s->N;
  if (tc) {
    // scores for the formed blocks come from the tensor cores for every g:
    // a separate group-summed-query pass (bf16 hi/lo pairs, ~fp32 accurate)
    if (int rc = tc_cmp_fwd(s, Q, Q16, qscale, Kc, Vc, out, lse, scores, workspace, st)) return rc;
  }
  const int64_t rows = s->h * ntok;
  if (rows > 0)
    cmp_fwd_generic<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
        (const T*)Q, (const A*)Kc, (const A*)Vc, (const A*)Kp, (const A*)Vp, (A*)out, (A*)lse, *s,
        ntok);
  FSA_LAUNCH_CHECK("cmp_attn_fwd");
  if (!tc && scores) {
    return fsa_importance_scores(s, dt, Q, Kc, scores, st);
  }
  return FSA_OK;
}

template <typename T>
int slide_fwd_impl(const fsa_shape* s, const void* Q, const void* K, const void* V, void* out,
                   void* lse, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  slide_fwd_generic<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>((const T*)Q, (const T*)K,
                                                                   (const T*)V, (A*)out, (A*)lse, *s);
  FSA_LAUNCH_CHECK("slide_fwd");
  return FSA_OK;
}

template <typename T>
int slide_bwd_impl(const fsa_shape* s, const void* Q, const void* K, const void* V,
                   const void* dOut, const void* lse, const void* delta, void* dQ, void* dK,
                   void* dV, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t rows = s->h * s->N, krows = s->h_K * s->N;
  if (rows == 0) return FSA_OK;
  slide_bwd_dq_generic<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      (const T*)Q, (const T*)K, (const T*)V, (const T*)dOut, (const A*)lse, (const A*)delta,
      (A*)dQ, *s);
  slide_bwd_dkdv_generic<T><<<(unsigned)((krows + 7) / 8), 256, 0, st>>>(
      (const T*)Q, (const T*)K, (const T*)V, (const T*)dOut, (const A*)lse, (const A*)delta,
      (A*)dK, (A*)dV, *s);
  FSA_LAUNCH_CHECK("slide_bwd");
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

extern "C" int fsa_cmp_attn_fwd(const fsa_shape* s, int dtype, const void* Q, const void* K_cmp,
                                const void* V_cmp, const void* K_prefix, const void* V_prefix,
                                void* out, void* lse, void* scores, void* workspace,
                                const void* Q16, const float* qscale, void* stream) {
  DISPATCH_DT(dtype, cmp_fwd_impl, s, Q, K_cmp, V_cmp, K_prefix, V_prefix, out, lse, scores,
              workspace, Q16, qscale, (cudaStream_t)stream);
}

extern "C" size_t fsa_cmp_workspace_bytes(const fsa_shape* s) {
  return fsa::tc_cmp_workspace_bytes(s);
}

extern "C" int fsa_slide_fwd(const fsa_shape* s, int dtype, const void* Q, const void* K,
                             const void* V, const float* vscale, void* out, void* lse,
                             void* stream) {
  if (fsa::tc_qo_supported(*s, dtype))  // V: the fsa_v_to_f16 copy, vscale its scales
    return fsa::tc_slide_fwd(s, Q, K, V, vscale, out, lse, (cudaStream_t)stream);
  DISPATCH_DT(dtype, slide_fwd_impl, s, Q, K, V, out, lse, (cudaStream_t)stream);
}

extern "C" size_t fsa_slide_bwd_workspace_bytes(const fsa_shape* s, int dtype) {
  return fsa::tc_bwd_supported(*s, dtype) ? fsa::tc_slide_bwd_workspace_bytes(s) : 0;
}

extern "C" int fsa_slide_bwd(const fsa_shape* s, int dtype, const void* Q, const void* K,
                             const void* V, const void* dOut, const void* lse, const void* delta,
                             void* dQ, void* dK, void* dV, void* workspace, int accumulate,
                             const float* scales, void* stream) {
  if (fsa::tc_bwd_supported(*s, dtype)) {
    FSA_REQUIRE(workspace != nullptr, "slide_bwd: tensor-core path needs its workspace");
    FSA_REQUIRE(scales != nullptr,
                "slide_bwd: the tensor-core path reads the fsa_stage_f16_ops copies and their scales");
    return fsa::tc_slide_bwd(s, Q, K, V, dOut, lse, delta, dQ, dK, dV, workspace, accumulate,
                             fsa::f16_scales_of(scales, s->h_K), (cudaStream_t)stream);
  }
  FSA_REQUIRE(!accumulate, "slide_bwd: accumulate only on the tensor-core path");
  DISPATCH_DT(dtype, slide_bwd_impl, s, Q, K, V, dOut, lse, delta, dQ, dK, dV, (cudaStream_t)stream);
}
