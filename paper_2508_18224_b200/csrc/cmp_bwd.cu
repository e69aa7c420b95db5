// Compressed-branch backward and the full gate backward.
// The reference differentiates only the selected and sliding branches; these
// kernels add the gradient through the compressed branch (branches.py:34-78)
// and the gates (branches.py:95-104) so an NSA training step is complete.
// Parity is against the float64 oracle (oracle.compressed_backward /
// gate_grad, pinned to torch autograd) -- unpinned against the reference.
//
//   out_cmp[t] = softmax(q_t . K_cmp[:nf]^T * scale) V_cmp[:nf],  nf = (t+1) // B_K
//              = V_prefix[t] = mean(V[0..t])                       (nf = 0)
//   dQ[t]   += scale * sum_i dS[t,i] K_cmp[i]
//   dK_cmp  = scale * dS^T Q,  dV_cmp = P^T dOut     (per kv head, heads of the group)
//   dK[s]   += dK_cmp[s // B_K] / B_K,  dV[s] += dV_cmp[s // B_K] / B_K
//            + sum_{t=s}^{B_K-2} dOut[t] / (t+1)     (pending tokens' prefix means)
// Deterministic: every output element has one writer and a fixed order.
//
// bf16, d = 128: the tensor-core path.  dK_cmp / dV_cmp come from the FSA
// backward kernel (K8) in its compressed mode -- 64 pooled rows per task held
// in smem against a chunk of CH tokens, one partial slab per chunk, summed here
// in chunk order -- and dQ from the query-outer dQ kernel over the formed pooled
// rows (tc_slide_dq.cu).  Other dtypes / shapes use the generic kernels below.
#include "tc_plan.cuh"

namespace fsa {
namespace {

template <typename T, typename KT>
__device__ __forceinline__ typename Acc<T>::type dotr(const T* q, const KT* k, int64_t d) {
  typename Acc<T>::type acc = 0;
  for (int64_t c = 0; c < d; ++c) acc += to_acc(q[c]) * to_acc(k[c]);
  return acc;
}

// dQ += (warp per (j, t), formed tokens)
template <typename T>
__global__ void cmp_bwd_dq_generic(const T* __restrict__ Q, const typename Acc<T>::type* __restrict__ Kc,
                                   const typename Acc<T>::type* __restrict__ Vc,
                                   const T* __restrict__ dOut,
                                   const typename Acc<T>::type* __restrict__ lse,
                                   const typename Acc<T>::type* __restrict__ delta,
                                   typename Acc<T>::type* __restrict__ dQ, fsa_shape s) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.h * s.N) return;
  const int64_t j = wid / s.N, t = wid % s.N, g = s.h / s.h_K, kh = j / g;
  const int64_t nf = (t + 1) / s.B_K, dK = s.d_K, dV = s.d_V;
  if (nf == 0) return;
  const T* q = Q + (t * s.h + j) * dK;
  const T* d = dOut + (t * s.h + j) * dV;
  const A scale = A(s.scale), lr = lse[j * s.N + t], dr = delta[j * s.N + t];
  for (int64_t c0 = 0; c0 < dK; c0 += 32) {
    A acc = 0;
    for (int64_t k0 = 0; k0 < nf; k0 += 32) {
      const int64_t i = k0 + lane;
      A dz = 0;
      if (i < nf) {
        const A p = exp_acc(dotr<T, A>(q, Kc + (i * s.h_K + kh) * dK, dK) * scale - lr);
        dz = p * (dotr<T, A>(d, Vc + (i * s.h_K + kh) * dV, dV) - dr);
      }
      const int64_t cnt = min((int64_t)32, nf - k0);
      for (int64_t kk = 0; kk < cnt; ++kk) {
        const A z = __shfl_sync(0xffffffffu, dz, (int)kk);
        if (c0 + lane < dK) acc += z * Kc[((k0 + kk) * s.h_K + kh) * dK + c0 + lane];
      }
    }
    if (c0 + lane < dK) dQ[(t * s.h + j) * dK + c0 + lane] += acc * scale;
  }
}

// dK_cmp / dV_cmp (warp per (kh, pooled row i)): queries t >= B_K (i+1) - 1
template <typename T>
__global__ void cmp_bwd_dkdv_generic(const T* __restrict__ Q, const typename Acc<T>::type* __restrict__ Kc,
                                     const typename Acc<T>::type* __restrict__ Vc,
                                     const T* __restrict__ dOut,
                                     const typename Acc<T>::type* __restrict__ lse,
                                     const typename Acc<T>::type* __restrict__ delta,
                                     typename Acc<T>::type* __restrict__ dKc,
                                     typename Acc<T>::type* __restrict__ dVc, fsa_shape s) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t b = s.N / s.B_K;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.h_K * b) return;
  const int64_t kh = wid / b, i = wid % b, g = s.h / s.h_K, dK = s.d_K, dV = s.d_V;
  const int64_t t0 = s.B_K * (i + 1) - 1, nq = s.N - t0;
  const A* kr = Kc + (i * s.h_K + kh) * dK;
  const A* vr = Vc + (i * s.h_K + kh) * dV;
  const A scale = A(s.scale);
  for (int64_t c0 = 0; c0 < (dK > dV ? dK : dV); c0 += 32) {
    A ak = 0, av = 0;
    for (int64_t hh = 0; hh < g; ++hh) {
      const int64_t j = kh * g + hh;
      for (int64_t q0 = 0; q0 < nq; q0 += 32) {
        const int64_t t = t0 + q0 + lane;
        A p = 0, dz = 0;
        if (q0 + lane < nq) {
          p = exp_acc(dotr<T, A>(Q + (t * s.h + j) * dK, kr, dK) * scale - lse[j * s.N + t]);
          dz = p * (dotr<T, A>(dOut + (t * s.h + j) * dV, vr, dV) - delta[j * s.N + t]);
        }
        const int64_t cnt = min((int64_t)32, nq - q0);
        for (int64_t kk = 0; kk < cnt; ++kk) {
          const A pk = __shfl_sync(0xffffffffu, p, (int)kk);
          const A zk = __shfl_sync(0xffffffffu, dz, (int)kk);
          const int64_t tt = t0 + q0 + kk;
          if (c0 + lane < dK) ak += zk * to_acc(Q[(tt * s.h + j) * dK + c0 + lane]);
          if (c0 + lane < dV) av += pk * to_acc(dOut[(tt * s.h + j) * dV + c0 + lane]);
        }
      }
    }
    if (c0 + lane < dK) dKc[(i * s.h_K + kh) * dK + c0 + lane] = ak * scale;
    if (c0 + lane < dV) dVc[(i * s.h_K + kh) * dV + c0 + lane] = av;
  }
}

// pooling backward (+ the pending tokens' prefix means): warp per (s, kh)
template <typename T>
__global__ void cmp_pool_bwd(const typename Acc<T>::type* __restrict__ dKc,
                             const typename Acc<T>::type* __restrict__ dVc,
                             const T* __restrict__ dOut, typename Acc<T>::type* __restrict__ dK,
                             typename Acc<T>::type* __restrict__ dV, fsa_shape s,
                             const typename Acc<T>::type* __restrict__ tau = nullptr) {
  // tau != null: dOut is the raw cotangent and the gate (tau[t, 0]) applies here
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.N * s.h_K) return;
  const int64_t sk = wid / s.h_K, kh = wid % s.h_K, i = sk / s.B_K, g = s.h / s.h_K;
  const int64_t n_pref = s.B_K - 1 < s.N ? s.B_K - 1 : s.N;
  const A inv = A(1) / A(s.B_K);
  for (int64_t c = lane; c < s.d_K; c += 32)
    dK[(sk * s.h_K + kh) * s.d_K + c] += dKc[(i * s.h_K + kh) * s.d_K + c] * inv;
  for (int64_t c = lane; c < s.d_V; c += 32) {
    A acc = dVc[(i * s.h_K + kh) * s.d_V + c] * inv;
    for (int64_t t = sk; t < n_pref; ++t) {
      A sum = 0;
      for (int64_t hh = 0; hh < g; ++hh) sum += to_acc(dOut[(t * s.h + kh * g + hh) * s.d_V + c]);
      if (tau) sum *= tau[t * 3];
      acc += sum / A(t + 1);
    }
    dV[(sk * s.h_K + kh) * s.d_V + c] += acc;
  }
}

// Gate backward for all three branches + their deltas + dtau: warp per token.
//   d_c = tau[t,c] dOut (rounded to T), delta_c[j,t] = sum_v out_c * d_c,
//   dtau[t,c] = sum_{j,v} out_c * dOut            (branches.py:103)
template <typename T, typename B = typename Acc<T>::type>  // B: branch-output element type
__global__ void gate_backward_full_kernel(const T* __restrict__ dOut,
                                          const typename Acc<T>::type* __restrict__ tau,
                                          const B* __restrict__ o0, const B* __restrict__ o1,
                                          const B* __restrict__ o2,
                                          T* __restrict__ d0, T* __restrict__ d1, T* __restrict__ d2,
                                          typename Acc<T>::type* __restrict__ del0,
                                          typename Acc<T>::type* __restrict__ del1,
                                          typename Acc<T>::type* __restrict__ del2,
                                          typename Acc<T>::type* __restrict__ dtau, int64_t N,
                                          int64_t h, int64_t dv) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= N) return;
  const A w0 = tau[t * 3], w1 = tau[t * 3 + 1], w2 = tau[t * 3 + 2];
  A g0 = 0, g1 = 0, g2 = 0;
  for (int64_t j = 0; j < h; ++j) {
    const int64_t base = (t * h + j) * dv;
    A s0 = 0, s1 = 0, s2 = 0;
    for (int64_t c = lane; c < dv; c += 32) {
      const A x = to_acc(dOut[base + c]);
      const A a0 = to_acc(o0[base + c]), a1 = to_acc(o1[base + c]), a2 = to_acc(o2[base + c]);
      const T r0 = from_acc<T>(w0 * x), r1 = from_acc<T>(w1 * x), r2 = from_acc<T>(w2 * x);
      d0[base + c] = r0;
      d1[base + c] = r1;
      d2[base + c] = r2;
      s0 += a0 * to_acc(r0);
      s1 += a1 * to_acc(r1);
      s2 += a2 * to_acc(r2);
      g0 += a0 * x;
      g1 += a1 * x;
      g2 += a2 * x;
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      del0[j * N + t] = s0;
      del1[j * N + t] = s1;
      del2[j * N + t] = s2;
    }
  }
  g0 = warp_sum(g0);
  g1 = warp_sum(g1);
  g2 = warp_sum(g2);
  if (lane == 0) {
    dtau[t * 3] = g0;
    dtau[t * 3 + 1] = g1;
    dtau[t * 3 + 2] = g2;
  }
}

// sum of a pooled row's per-chunk partial slabs, in chunk order (tensor-core path)
__global__ void cmp_slab_reduce(const float* __restrict__ dKp, const float* __restrict__ dVp,
                                float* __restrict__ dKc, float* __restrict__ dVc, int64_t b,
                                int64_t h_K, int64_t B_K, int64_t CH, int64_t nch, int64_t cstride) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // (j, kh, c), c fastest
  if (e >= b * h_K * 128) return;
  const int64_t j = e / (h_K * 128);
  const int64_t first = ((j / 64) * 64 + 1) * B_K - 1;  // first token of the tile's chunks
  float ak = 0.f, av = 0.f;
  for (int64_t q = first / CH; q < nch; ++q) {
    ak += __ldcs(dKp + q * cstride + e);
    av += __ldcs(dVp + q * cstride + e);
  }
  dKc[e] = ak;
  dVc[e] = av;
}

__global__ void f32_to_bf16(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

bool tc_cmp_bwd_ok(const fsa_shape& s) { return tc_qo_supported(s, FSA_DT_BF16) && s.N * s.h < (1ll << 31); }

struct CmpWs {  // tensor-core path workspace
  __half *kc16, *vc16;   // fp16 staged K_cmp / V_cmp (their own per-kv-head scales)
  float *kcs, *vcs;      // [2 h_K] each: scales, scratch
  __half *q16, *o16;     // staged Q / dOut (fsa_cmp_bwd only; the fold entry gets them)
  float* qos;            // [8 h_K]: the fsa_stage_f16_ops scale blocks (s_Q, s_dO used)
  float *dKp, *dVp, *dKc, *dVc;
  int32_t* counter;
  int64_t CH, nch, cstride;
  size_t bytes;
};
CmpWs cmp_ws(const fsa_shape& s, void* base, bool stage_qo) {
  CmpWs w{};
  const int64_t b = s.N / s.B_K, n = b * s.h_K * 128;
  w.CH = cmp_chunk_tokens(&s);
  w.nch = (s.N + w.CH - 1) / w.CH;
  w.cstride = ((b + 63) / 64) * 64 * s.h_K * 128;
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* r = p + off; off += (bytes + 255) & ~size_t(255); return r; };
  w.kc16 = (__half*)take(n * 2);
  w.vc16 = (__half*)take(n * 2);
  w.kcs = (float*)take(2 * s.h_K * 4);
  w.vcs = (float*)take(2 * s.h_K * 4);
  if (stage_qo) {
    w.q16 = (__half*)take(s.N * s.h * s.d_K * 2);
    w.o16 = (__half*)take(s.N * s.h * s.d_V * 2);
    w.qos = (float*)take(8 * s.h_K * 4);  // fsa_stage_f16_ops scale blocks
  }
  w.dKp = (float*)take(w.nch * w.cstride * 4);
  w.dVp = (float*)take(w.nch * w.cstride * 4);
  w.dKc = (float*)take(n * 4);
  w.dVc = (float*)take(n * 4);
  w.counter = (int32_t*)take(256);
  w.bytes = off + 256;
  return w;
}

// Q16 / dO16 / qos: the fsa_stage_f16_ops copies of Q and dOut and their scales
// (sq, so: per kv head); dOut: the raw bf16 cotangent (the
// pending tokens' prefix-mean gradients read it)
int cmp_bwd_tc(const fsa_shape* s, const void* Q16, const void* Kc, const void* Vc,
               const void* dOut, const void* dO16, const float* sq, const float* so,
               const void* tau, const void* lse, const void* delta, void* dQ, void* dK, void* dV,
               const CmpWs& w, cudaStream_t st) {
  const int64_t b = s->N / s->B_K, n = b * s->h_K * 128;
  if (n > 0) {
    if (int rc = stage_f16(FSA_DT_F32, Kc, b, s->h_K, 128, w.kc16, w.kcs, st)) return rc;
    if (int rc = stage_f16(FSA_DT_F32, Vc, b, s->h_K, 128, w.vc16, w.vcs, st)) return rc;
    const F16Scales sc{sq, w.kcs, w.vcs, so};
    if (int rc = tc_cmp_dq(s, Q16, w.kc16, w.vc16, dO16, lse, delta, dQ, sc, st)) return rc;
    if (int rc = tc_cmp_bwd_kv(s, Q16, w.kc16, w.vc16, dO16, lse, delta, w.dKp, w.dVp, w.counter,
                               sc, st))
      return rc;
    cmp_slab_reduce<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w.dKp, w.dVp, w.dKc, w.dVc, b, s->h_K,
                                                               s->B_K, w.CH, w.nch, w.cstride);
    FSA_LAUNCH_CHECK("cmp_slab_reduce");
  }
  const int64_t pr = s->N * s->h_K;
  if (pr > 0)
    cmp_pool_bwd<__nv_bfloat16><<<(unsigned)((pr + 7) / 8), 256, 0, st>>>(
        w.dKc, w.dVc, (const __nv_bfloat16*)dOut, (float*)dK, (float*)dV, *s, (const float*)tau);
  FSA_LAUNCH_CHECK("cmp_pool_bwd");
  return FSA_OK;
}

// tau non-null: the gate is folded in (lse = lse_adj, dOut raw; tau gates the
// pending tokens' prefix-mean gradients).  Q16 / dO16 / scales: the
// fsa_stage_f16_ops copies for the tensor-core path (null: staged here, into
// a workspace sized for it).
template <typename T>
int cmp_bwd_impl(const fsa_shape* s, const void* Q, const void* Kc, const void* Vc, const void* dOut,
                 const void* tau, const void* lse, const void* delta, void* dQ, void* dK, void* dV,
                 void* ws, const void* Q16, const void* dO16, const float* scales, cudaStream_t st) {
  using A = typename Acc<T>::type;
  if (sizeof(T) == 2 && tc_cmp_bwd_ok(*s)) {
    const bool stage = Q16 == nullptr;
    const CmpWs w = cmp_ws(*s, ws, stage);
    const float *sq, *so;
    if (stage) {
      if (int rc = fsa_stage_f16_ops(s, FSA_DT_BF16, Q, nullptr, nullptr, dOut, w.q16, nullptr,
                                     nullptr, w.o16, w.qos, st))
        return rc;
      Q16 = w.q16;
      dO16 = w.o16;
      sq = w.qos;
      so = w.qos + 6 * s->h_K;
    } else {
      FSA_REQUIRE(dO16 != nullptr && scales != nullptr, "cmp_bwd: Q16 given without dO16 / scales");
      const F16Scales sc = f16_scales_of(scales, s->h_K);
      sq = sc.q;
      so = sc.o;
    }
    return cmp_bwd_tc(s, Q16, Kc, Vc, dOut, dO16, sq, so, tau, lse, delta, dQ, dK, dV, w, st);
  }
  const int64_t b = s->N / s->B_K;
  A* dKc = (A*)ws;
  A* dVc = dKc + b * s->h_K * s->d_K;
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  cmp_bwd_dq_generic<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(
      (const T*)Q, (const A*)Kc, (const A*)Vc, (const T*)dOut, (const A*)lse, (const A*)delta,
      (A*)dQ, *s);
  const int64_t kr = s->h_K * b;
  if (kr > 0)
    cmp_bwd_dkdv_generic<T><<<(unsigned)((kr + 7) / 8), 256, 0, st>>>(
        (const T*)Q, (const A*)Kc, (const A*)Vc, (const T*)dOut, (const A*)lse, (const A*)delta,
        dKc, dVc, *s);
  const int64_t pr = s->N * s->h_K;
  cmp_pool_bwd<T><<<(unsigned)((pr + 7) / 8), 256, 0, st>>>(dKc, dVc, (const T*)dOut, (A*)dK,
                                                           (A*)dV, *s, (const A*)tau);
  FSA_LAUNCH_CHECK("cmp_bwd");
  return FSA_OK;
}

// The full gate backward folded into the three branches' statistics (the
// tensor-core NSA step with full=True): delta_c = sum_v out_c * dOut, lse_c_adj
// = lse_c - ln tau_c[t] -- the branch kernels then take the raw dOut -- and
// dtau[t, c] = sum_{j,v} out_c * dOut.  Warp per token (deterministic dtau).
template <typename T, typename B>
__global__ void gate_fold3_kernel(const T* __restrict__ dOut, const typename Acc<T>::type* __restrict__ tau,
                                  const B* __restrict__ o0, const B* __restrict__ o1,
                                  const B* __restrict__ o2, const typename Acc<T>::type* __restrict__ l0,
                                  const typename Acc<T>::type* __restrict__ l1,
                                  const typename Acc<T>::type* __restrict__ l2,
                                  typename Acc<T>::type* __restrict__ del0,
                                  typename Acc<T>::type* __restrict__ del1,
                                  typename Acc<T>::type* __restrict__ del2,
                                  typename Acc<T>::type* __restrict__ la0,
                                  typename Acc<T>::type* __restrict__ la1,
                                  typename Acc<T>::type* __restrict__ la2,
                                  typename Acc<T>::type* __restrict__ dtau, int64_t N, int64_t h,
                                  int64_t dv) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= N) return;
  const A w0 = tau[t * 3], w1 = tau[t * 3 + 1], w2 = tau[t * 3 + 2];
  const A lw0 = log_acc(w0), lw1 = log_acc(w1), lw2 = log_acc(w2);
  A g0 = 0, g1 = 0, g2 = 0;
  for (int64_t j = 0; j < h; ++j) {
    const int64_t base = (t * h + j) * dv;
    A s0 = 0, s1 = 0, s2 = 0;
    if constexpr (sizeof(T) == 2 && sizeof(B) == 2) {
      if (dv == 128) {  // 4 features per lane: 8-byte loads of dOut and the three outputs
        const int64_t e = base + lane * 4;
        const uint2 ux = *reinterpret_cast<const uint2*>(dOut + e);
        const uint2 u0 = *reinterpret_cast<const uint2*>(o0 + e);
        const uint2 u1 = *reinterpret_cast<const uint2*>(o1 + e);
        const uint2 u2 = *reinterpret_cast<const uint2*>(o2 + e);
        const __nv_bfloat162* px = reinterpret_cast<const __nv_bfloat162*>(&ux);
        const __nv_bfloat162* p0 = reinterpret_cast<const __nv_bfloat162*>(&u0);
        const __nv_bfloat162* p1 = reinterpret_cast<const __nv_bfloat162*>(&u1);
        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&u2);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float2 x = __bfloat1622float2(px[k]), a = __bfloat1622float2(p0[k]),
                       b = __bfloat1622float2(p1[k]), c2 = __bfloat1622float2(p2[k]);
          s0 += a.x * x.x + a.y * x.y;
          s1 += b.x * x.x + b.y * x.y;
          s2 += c2.x * x.x + c2.y * x.y;
        }
      } else {
        for (int64_t c = lane; c < dv; c += 32) {
          const A x = to_acc(dOut[base + c]);
          s0 += A(to_acc(o0[base + c])) * x;
          s1 += A(to_acc(o1[base + c])) * x;
          s2 += A(to_acc(o2[base + c])) * x;
        }
      }
    } else {
      for (int64_t c = lane; c < dv; c += 32) {
        const A x = to_acc(dOut[base + c]);
        s0 += A(to_acc(o0[base + c])) * x;
        s1 += A(to_acc(o1[base + c])) * x;
        s2 += A(to_acc(o2[base + c])) * x;
      }
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    g0 += s0;
    g1 += s1;
    g2 += s2;
    if (lane == 0) {
      const int64_t r = j * N + t;
      del0[r] = s0;
      del1[r] = s1;
      del2[r] = s2;
      la0[r] = l0[r] - lw0;  // tau = 0: +inf, the branch's P = 0
      la1[r] = l1[r] - lw1;
      la2[r] = l2[r] - lw2;
    }
  }
  if (lane == 0) {
    dtau[t * 3] = g0;
    dtau[t * 3 + 1] = g1;
    dtau[t * 3 + 2] = g2;
  }
}

template <typename T>
int gate_fold3_impl(const fsa_shape* s, const void* dOut, const void* tau, const void* o0,
                    const void* o1, const void* o2, const void* l0, const void* l1, const void* l2,
                    void* del0, void* del1, void* del2, void* la0, void* la1, void* la2, void* dtau,
                    cudaStream_t st) {
  using A = typename Acc<T>::type;
  if (s->N == 0) return FSA_OK;
  const unsigned grid = (unsigned)((s->N + 7) / 8);
  gate_fold3_kernel<T, A><<<grid, 256, 0, st>>>(
        (const T*)dOut, (const A*)tau, (const A*)o0, (const A*)o1, (const A*)o2, (const A*)l0,
        (const A*)l1, (const A*)l2, (A*)del0, (A*)del1, (A*)del2, (A*)la0, (A*)la1, (A*)la2,
        (A*)dtau, s->N, s->h, s->d_V);
  FSA_LAUNCH_CHECK("gate_backward_full_fold");
  return FSA_OK;
}

template <typename T>
int gate_bwd_full_impl(const fsa_shape* s, const void* dOut, const void* tau, const void* o0,
                       const void* o1, const void* o2, void* d0, void* d1, void* d2, void* del0,
                       void* del1, void* del2, void* dtau, cudaStream_t st) {
  using A = typename Acc<T>::type;
  if (s->N == 0) return FSA_OK;
  gate_backward_full_kernel<T><<<(unsigned)((s->N + 7) / 8), 256, 0, st>>>(
        (const T*)dOut, (const A*)tau, (const A*)o0, (const A*)o1, (const A*)o2, (T*)d0, (T*)d1,
        (T*)d2, (A*)del0, (A*)del1, (A*)del2, (A*)dtau, s->N, s->h, s->d_V);
  FSA_LAUNCH_CHECK("gate_backward_full");
  return FSA_OK;
}

}  // namespace
}  // namespace fsa

#define DISPATCH_DT(dt, FN, ...)                                            \
  switch (dt) {                                                             \
    case FSA_DT_F32: return fsa::FN<float>(__VA_ARGS__);                    \
    case FSA_DT_F64: return fsa::FN<double>(__VA_ARGS__);                   \
    case FSA_DT_BF16: return fsa::FN<__nv_bfloat16>(__VA_ARGS__);           \
    default: fsa::set_error("unsupported dtype %d", (int)dt); return FSA_ERR_INVALID; \
  }

extern "C" size_t fsa_cmp_bwd_workspace_bytes(const fsa_shape* s, int dtype) {
  const size_t acc = dtype == FSA_DT_F64 ? 8 : 4;
  if (dtype == FSA_DT_BF16 && fsa::tc_cmp_bwd_ok(*s)) return fsa::cmp_ws(*s, nullptr, true).bytes;
  return (size_t)(s->N / s->B_K) * s->h_K * (s->d_K + s->d_V) * acc + 256;
}

extern "C" int fsa_cmp_bwd(const fsa_shape* s, int dtype, const void* Q, const void* K_cmp,
                           const void* V_cmp, const void* dOut, const void* lse, const void* delta,
                           void* dQ, void* dK, void* dV, void* workspace, void* stream) {
  FSA_REQUIRE(workspace != nullptr, "cmp_bwd: workspace required");
  DISPATCH_DT(dtype, cmp_bwd_impl, s, Q, K_cmp, V_cmp, dOut, nullptr, lse, delta, dQ, dK, dV,
              workspace, nullptr, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" size_t fsa_cmp_bwd_fold_workspace_bytes(const fsa_shape* s, int dtype) {
  if (dtype == FSA_DT_BF16 && fsa::tc_cmp_bwd_ok(*s)) return fsa::cmp_ws(*s, nullptr, false).bytes;
  return fsa_cmp_bwd_workspace_bytes(s, dtype);
}

extern "C" int fsa_cmp_bwd_fold(const fsa_shape* s, int dtype, const void* Q, const void* K_cmp,
                                const void* V_cmp, const void* dOut, const void* tau,
                                const void* lse_adj, const void* delta, void* dQ, void* dK, void* dV,
                                const void* Q16, const void* dO16, const float* scales,
                                void* workspace, void* stream) {
  FSA_REQUIRE(workspace != nullptr, "cmp_bwd: workspace required");
  FSA_REQUIRE(tau != nullptr, "cmp_bwd_fold: tau required");
  if (dtype == FSA_DT_BF16 && fsa::tc_cmp_bwd_ok(*s))
    FSA_REQUIRE(Q16 != nullptr && dO16 != nullptr && scales != nullptr,
                "cmp_bwd_fold: the tensor-core path reads the fsa_stage_f16_ops copies of Q and dOut");
  DISPATCH_DT(dtype, cmp_bwd_impl, s, Q, K_cmp, V_cmp, dOut, tau, lse_adj, delta, dQ, dK, dV,
              workspace, Q16, dO16, scales, (cudaStream_t)stream);
}

extern "C" int fsa_gate_backward_full(const fsa_shape* s, int dtype, const void* dOut,
                                      const void* tau, const void* out_cmp, const void* out_sel,
                                      const void* out_slide, void* d_cmp, void* d_sel,
                                      void* d_slide, void* delta_cmp, void* delta_sel,
                                      void* delta_slide, void* dtau, void* stream) {
  DISPATCH_DT(dtype, gate_bwd_full_impl, s, dOut, tau, out_cmp, out_sel, out_slide, d_cmp, d_sel,
              d_slide, delta_cmp, delta_sel, delta_slide, dtau, (cudaStream_t)stream);
}

extern "C" int fsa_gate_backward_full_fold(const fsa_shape* s, int dtype, const void* dOut,
                                           const void* tau, const void* out_cmp, const void* out_sel,
                                           const void* out_slide, const void* lse_cmp,
                                           const void* lse_sel, const void* lse_slide,
                                           void* delta_cmp, void* delta_sel, void* delta_slide,
                                           void* lse_cmp_adj, void* lse_sel_adj, void* lse_slide_adj,
                                           void* dtau, void* stream) {
  DISPATCH_DT(dtype, gate_fold3_impl, s, dOut, tau, out_cmp, out_sel, out_slide, lse_cmp, lse_sel,
              lse_slide, delta_cmp, delta_sel, delta_slide, lse_cmp_adj, lse_sel_adj, lse_slide_adj,
              dtau, (cudaStream_t)stream);
}
