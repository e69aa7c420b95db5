// FSA selected attention, generic SIMT path (any d_K/d_V/B_K that fits in
// shared memory; f32, f64 and bf16 inputs).  The bf16 d=128/B_K=64 hot path
// runs on tcgen05 tensor cores instead (tc_sel_fwd.cu / tc_sel_bwd.cu); this
// file serves the fp32 / fp64 configurations and the small shapes of the
// reference's own tests.
//
//   fwd task (kv head kh, block i)   kv_major.py:152-204, _core.pyx:49-94
//   merge    (kh, token t)           kv_major.py:137-149, :207-242
//   delta    (head j, token t)       kv_major.py:284
//   bwd task (kh, i)                 kv_major.py:297-324, _core.pyx:97-131
//   dq reduce (j, t)                 kv_major.py:326-340
#include "common.cuh"
#include "tc_plan.cuh"

namespace fsa {

template <typename A> struct Pair { A m, l; };

// ---------------------------------------------------------------------------
// forward block pass: one CTA per (block i, kv head kh); K_i/V_i staged once
// and reused by all g heads of every gathered row.
// ---------------------------------------------------------------------------
template <typename T, int kMode>
__global__ void __launch_bounds__(128)
sel_fwd_generic(const T* __restrict__ Q, const T* __restrict__ K, const T* __restrict__ V,
                const int32_t* __restrict__ offsets, const int32_t* __restrict__ qlist,
                const typename Acc<T>::type* __restrict__ m_global,
                typename Acc<T>::type* __restrict__ obuf, typename Acc<T>::type* __restrict__ ml,
                fsa_shape s) {
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t i = blockIdx.x, kh = blockIdx.y;
  const int64_t b = s.N / s.B_K, g = s.h / s.h_K;
  const int64_t beg = offsets[kh * (b + 1) + i], n = offsets[kh * (b + 1) + i + 1] - beg;
  if (n == 0) return;  // early return: no loads (kv_major.py:188-189)
  const int64_t dK = s.d_K, dV = s.d_V, BK = s.B_K, dKp = dK + 1;
  A* Ks = reinterpret_cast<A*>(smem_raw);  // [BK][dK+1]
  A* Vs = Ks + BK * dKp;                   // [BK][dV]
  A* wbuf = Vs + BK * dV;                  // per warp: q[dK], p[BK]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  A* qw = wbuf + warp * (dK + BK);
  A* pw = qw + dK;
  for (int64_t e = threadIdx.x; e < BK * dK; e += blockDim.x) {
    const int64_t r = e / dK, c = e % dK;
    Ks[r * dKp + c] = to_acc(K[((i * BK + r) * s.h_K + kh) * dK + c]);
  }
  for (int64_t e = threadIdx.x; e < BK * dV; e += blockDim.x) {
    const int64_t r = e / dV, c = e % dV;
    Vs[r * dV + c] = to_acc(V[((i * BK + r) * s.h_K + kh) * dV + c]);
  }
  __syncthreads();
  const int64_t TT = s.T;
  const A scale = A(s.scale);
  for (int64_t r = warp; r < n * g; r += blockDim.x >> 5) {
    const int32_t ent = qlist[kh * s.N * TT + beg + r / g];
    const int64_t t = ent / TT, slot = ent % TT, j = kh * g + r % g;
    const int64_t vis = min(t - i * BK + 1, BK);
    for (int64_t c = lane; c < dK; c += 32) qw[c] = to_acc(Q[(t * s.h + j) * dK + c]);
    __syncwarp();
    A mloc = neg_inf<A>();
    for (int64_t c = lane; c < BK; c += 32) {
      A z = neg_inf<A>();
      if (c < vis) {
        A acc = 0;
        for (int64_t k = 0; k < dK; ++k) acc += qw[k] * Ks[c * dKp + k];
        z = acc * scale;
      }
      pw[c] = z;
      mloc = fmax(mloc, z);
    }
    mloc = warp_max(mloc);
    const A shift = (kMode == FSA_FWD_GLOBAL) ? m_global[j * s.N + t] : mloc;
    A lsum = 0;
    for (int64_t c = lane; c < BK; c += 32) {
      const A p = exp_acc(pw[c] - shift);
      pw[c] = p;
      lsum += p;
    }
    lsum = warp_sum(lsum);
    __syncwarp();
    const int64_t orow = (j * s.N + t) * TT + slot;
    if (kMode != FSA_FWD_GLOBAL && lane == 0) {
      ml[orow * 2 + 0] = mloc;
      ml[orow * 2 + 1] = lsum;
    }
    if (kMode != FSA_FWD_STATS) {
      const A inv = (kMode == FSA_FWD_LOCAL) ? A(1) / lsum : A(1);
      for (int64_t c = lane; c < dV; c += 32) {
        A acc = 0;
        for (int64_t k = 0; k < vis; ++k) acc += pw[k] * Vs[k * dV + c];
        obuf[orow * dV + c] = acc * inv;
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// merge: one warp per (kv head, token); the g heads are handled in turn so the
// shared-max variant (kv_major.py:141-146) sees the whole group.
// ---------------------------------------------------------------------------
template <typename T, typename OB>
__global__ void merge_generic(int mode, const int32_t* __restrict__ idx, const OB* __restrict__ obuf,
                              const typename Acc<T>::type* __restrict__ ml,
                              const typename Acc<T>::type* __restrict__ m_global,
                              const typename Acc<T>::type* __restrict__ l_global, typename Acc<T>::type* __restrict__ out,
                              typename Acc<T>::type* __restrict__ lse,
                              typename Acc<T>::type* __restrict__ m_out,
                              typename Acc<T>::type* __restrict__ l_out, int shared_max, fsa_shape s) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.h_K * s.N) return;
  const int64_t kh = wid / s.N, t = wid % s.N, TT = s.T, g = s.h / s.h_K, dV = s.d_V;
  const int32_t* row = idx + (kh * s.N + t) * TT;
  int64_t len = 0;
  while (len < TT && row[len] != -1) ++len;
  A gmax = neg_inf<A>();
  for (int64_t hh = 0; hh < g; ++hh) {
    const int64_t j = kh * g + hh;
    const int64_t rb = (j * s.N + t) * TT;
    if (mode == FSA_MERGE_STATS) {
      A m = neg_inf<A>(), l = 0;
      for (int64_t k = 0; k < len; ++k) {
        const A mp = ml[(rb + k) * 2], lp = ml[(rb + k) * 2 + 1];
        const A mn = fmax(m, mp);
        l = l * exp_acc(m - mn) + lp * exp_acc(mp - mn);
        m = mn;
      }
      if (lane == 0) {
        m_out[j * s.N + t] = m;
        l_out[j * s.N + t] = l;
      }
      gmax = fmax(gmax, m);
    } else if (mode == FSA_MERGE_LOCAL) {
      A M = neg_inf<A>();
      for (int64_t k = 0; k < len; ++k) M = fmax(M, ml[(rb + k) * 2]);
      A L = 0;
      for (int64_t k = 0; k < len; ++k) L += ml[(rb + k) * 2 + 1] * exp_acc(ml[(rb + k) * 2] - M);
      const A invL = A(1) / L;
      for (int64_t c = lane; c < dV; c += 32) {
        A acc = 0;
        for (int64_t k = 0; k < len; ++k) {
          const A w = ml[(rb + k) * 2 + 1] * exp_acc(ml[(rb + k) * 2] - M);
          acc += w * to_acc(obuf[(rb + k) * dV + c]);
        }
        out[(t * s.h + j) * dV + c] = acc * invL;
      }
      if (lane == 0) {
        if (lse) lse[j * s.N + t] = M + log_acc(L);
        if (m_out) m_out[j * s.N + t] = M;
        if (l_out) l_out[j * s.N + t] = L;
      }
    } else {  // FSA_MERGE_REDUCE
      const A l = l_global[j * s.N + t], m = m_global[j * s.N + t];
      for (int64_t c = lane; c < dV; c += 32) {
        A acc = 0;
        for (int64_t k = 0; k < len; ++k) acc += to_acc(obuf[(rb + k) * dV + c]);
        out[(t * s.h + j) * dV + c] = acc / l;
      }
      if (lane == 0 && lse) lse[j * s.N + t] = m + log_acc(l);
    }
  }
  if (mode == FSA_MERGE_STATS && shared_max && lane == 0) {
    for (int64_t hh = 0; hh < g; ++hh) {
      const int64_t o = (kh * g + hh) * s.N + t;
      l_out[o] = l_out[o] * exp_acc(m_out[o] - gmax);
      m_out[o] = gmax;
    }
  }
}

template <typename T>
__global__ void delta_kernel(const typename Acc<T>::type* __restrict__ out, const T* __restrict__ dOut,
                             typename Acc<T>::type* __restrict__ delta, fsa_shape s) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.h * s.N) return;
  const int64_t j = wid / s.N, t = wid % s.N;
  const A* o = out + (t * s.h + j) * s.d_V;
  const T* d = dOut + (t * s.h + j) * s.d_V;
  A acc = 0;
  for (int64_t c = lane; c < s.d_V; c += 32) acc += to_acc(o[c]) * to_acc(d[c]);
  acc = warp_sum(acc);
  if (lane == 0) delta[j * s.N + t] = acc;
}

// ---------------------------------------------------------------------------
// backward: one CTA per (block i, kv head kh), rows processed in list order by
// the whole CTA so every dK/dV element has one owner thread and a fixed
// accumulation order (deterministic, no atomics).
// ---------------------------------------------------------------------------
template <typename T, bool kStage>
__global__ void __launch_bounds__(128)
sel_bwd_generic(const T* __restrict__ Q, const T* __restrict__ K, const T* __restrict__ V,
                const T* __restrict__ dOut, const typename Acc<T>::type* __restrict__ lse,
                const typename Acc<T>::type* __restrict__ delta,
                const int32_t* __restrict__ offsets, const int32_t* __restrict__ qlist,
                typename Acc<T>::type* __restrict__ dq_buf, typename Acc<T>::type* __restrict__ dK,
                typename Acc<T>::type* __restrict__ dV, fsa_shape s) {
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t i = blockIdx.x, kh = blockIdx.y;
  const int64_t b = s.N / s.B_K, g = s.h / s.h_K, TT = s.T;
  const int64_t dKd = s.d_K, dVd = s.d_V, BK = s.B_K;
  const int64_t beg = offsets[kh * (b + 1) + i], n = offsets[kh * (b + 1) + i + 1] - beg;
  if (n == 0) {
    for (int64_t e = threadIdx.x; e < BK * dKd; e += blockDim.x)
      dK[((i * BK + e / dKd) * s.h_K + kh) * dKd + e % dKd] = 0;
    for (int64_t e = threadIdx.x; e < BK * dVd; e += blockDim.x)
      dV[((i * BK + e / dVd) * s.h_K + kh) * dVd + e % dVd] = 0;
    return;
  }
  // kStage: K_i/V_i staged in smem; otherwise (large f64 tiles) read through L1
  A* Ks = reinterpret_cast<A*>(smem_raw);              // [BK][dK+1]
  A* Vs = Ks + (kStage ? BK * (dKd + 1) : 0);          // [BK][dV+1]
  A* dKs = Vs + (kStage ? BK * (dVd + 1) : 0);         // [BK][dK]
  A* dVs = dKs + BK * dKd;                 // [BK][dV]
  A* qs = dVs + BK * dVd;                  // [dK]
  A* dos = qs + dKd;                       // [dV]
  A* ps = dos + dVd;                       // [BK]
  A* dzs = ps + BK;                        // [BK]
  const T* Kg = K + (i * BK * s.h_K + kh) * dKd;  // row r at Kg + r*h_K*dK
  const T* Vg = V + (i * BK * s.h_K + kh) * dVd;
  auto kv = [&](int64_t r, int64_t c) -> A {
    return kStage ? Ks[r * (dKd + 1) + c] : to_acc(Kg[r * s.h_K * dKd + c]);
  };
  auto vv = [&](int64_t r, int64_t c) -> A {
    return kStage ? Vs[r * (dVd + 1) + c] : to_acc(Vg[r * s.h_K * dVd + c]);
  };
  for (int64_t e = threadIdx.x; e < BK * dKd; e += blockDim.x) {
    const int64_t r = e / dKd, c = e % dKd;
    if (kStage) Ks[r * (dKd + 1) + c] = to_acc(Kg[r * s.h_K * dKd + c]);
    dKs[e] = 0;
  }
  for (int64_t e = threadIdx.x; e < BK * dVd; e += blockDim.x) {
    const int64_t r = e / dVd, c = e % dVd;
    if (kStage) Vs[r * (dVd + 1) + c] = to_acc(Vg[r * s.h_K * dVd + c]);
    dVs[e] = 0;
  }
  const A scale = A(s.scale);
  for (int64_t r = 0; r < n * g; ++r) {
    const int32_t ent = qlist[kh * s.N * TT + beg + r / g];
    const int64_t t = ent / TT, slot = ent % TT, j = kh * g + r % g;
    const int64_t vis = min(t - i * BK + 1, BK);
    __syncthreads();
    for (int64_t c = threadIdx.x; c < dKd; c += blockDim.x) qs[c] = to_acc(Q[(t * s.h + j) * dKd + c]);
    for (int64_t c = threadIdx.x; c < dVd; c += blockDim.x)
      dos[c] = to_acc(dOut[(t * s.h + j) * dVd + c]);
    __syncthreads();
    const A lrow = lse[j * s.N + t], drow = delta[j * s.N + t];
    for (int64_t c = threadIdx.x; c < BK; c += blockDim.x) {
      A p = 0, dz = 0;
      if (c < vis) {
        A z = 0, dp = 0;
        for (int64_t k = 0; k < dKd; ++k) z += qs[k] * kv(c, k);
        for (int64_t k = 0; k < dVd; ++k) dp += dos[k] * vv(c, k);
        p = exp_acc(z * scale - lrow);
        dz = p * (dp - drow);
      }
      ps[c] = p;
      dzs[c] = dz;
    }
    __syncthreads();
    A* dqr = dq_buf + ((j * s.N + t) * TT + slot) * dKd;
    for (int64_t c = threadIdx.x; c < dKd; c += blockDim.x) {
      A acc = 0;
      for (int64_t k = 0; k < vis; ++k) acc += dzs[k] * kv(k, c);
      dqr[c] = acc * scale;
    }
    for (int64_t e = threadIdx.x; e < BK * dKd; e += blockDim.x)
      dKs[e] += dzs[e / dKd] * qs[e % dKd] * scale;
    for (int64_t e = threadIdx.x; e < BK * dVd; e += blockDim.x)
      dVs[e] += ps[e / dVd] * dos[e % dVd];
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < BK * dKd; e += blockDim.x)
    dK[((i * BK + e / dKd) * s.h_K + kh) * dKd + e % dKd] = dKs[e];
  for (int64_t e = threadIdx.x; e < BK * dVd; e += blockDim.x)
    dV[((i * BK + e / dVd) * s.h_K + kh) * dVd + e % dVd] = dVs[e];
}

template <typename T, typename DB>
__global__ void dq_reduce_kernel(const int32_t* __restrict__ idx, const DB* __restrict__ dq_buf,
                                 typename Acc<T>::type* __restrict__ dQ, fsa_shape s) {
  using A = typename Acc<T>::type;
  const int lane = threadIdx.x & 31;
  const int64_t wid = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= s.h * s.N) return;
  const int64_t j = wid / s.N, t = wid % s.N, TT = s.T, g = s.h / s.h_K, kh = j / g;
  const int32_t* row = idx + (kh * s.N + t) * TT;
  int64_t len = 0;
  while (len < TT && row[len] != -1) ++len;
  const int64_t rb = (j * s.N + t) * TT;
  for (int64_t c = lane; c < s.d_K; c += 32) {
    A acc = 0;
    for (int64_t k = 0; k < len; ++k) acc += to_acc(dq_buf[(rb + k) * s.d_K + c]);
    dQ[(t * s.h + j) * s.d_K + c] = acc;
  }
}

// ---------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------
template <typename T>
int sel_fwd_impl(const fsa_shape* s, int mode, const void* Q, const void* K, const void* V,
                 const int32_t* offsets, const int32_t* qlist, const void* m_global, void* obuf,
                 void* ml, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t b = s->N / s->B_K;
  size_t smem = sizeof(A) * (size_t)(s->B_K * (s->d_K + 1 + s->d_V) + 4 * (s->d_K + s->B_K));
  FSA_REQUIRE(smem <= 220 * 1024, "selected forward: B_K=%lld d=%lld exceeds shared memory",
              (long long)s->B_K, (long long)s->d_K);
  auto kern = mode == FSA_FWD_LOCAL ? sel_fwd_generic<T, FSA_FWD_LOCAL>
            : mode == FSA_FWD_STATS ? sel_fwd_generic<T, FSA_FWD_STATS>
                                    : sel_fwd_generic<T, FSA_FWD_GLOBAL>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)b, (unsigned)s->h_K);
  kern<<<grid, 128, smem, st>>>((const T*)Q, (const T*)K, (const T*)V, offsets, qlist,
                                (const A*)m_global, (A*)obuf, (A*)ml, *s);
  FSA_LAUNCH_CHECK("sel_fwd");
  return FSA_OK;
}

template <typename T>
int merge_impl(const fsa_shape* s, int mode, const int32_t* idx, const int32_t* work,
               const void* obuf, int obuf_dtype, const void* ml, const void* mg, const void* lg,
               void* out, void* lse, void* m_out, void* l_out, int shared_max, const float* vscale,
               cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t rows = s->h_K * s->N;
  if (rows == 0) return FSA_OK;
  const unsigned grid = (unsigned)((rows + 7) / 8);
  if (obuf_dtype == FSA_DT_F16) {  // the tensor-core path's fp16 partials (LOCAL mode only)
    FSA_REQUIRE(mode == FSA_MERGE_LOCAL && fast_reduce_ok(*s) && sizeof(A) == 4,
                "merge_fwd: fp16 partials only in LOCAL mode with d = 128");
    return merge_f16_fast(s, idx, work, obuf, ml, vscale, out, lse, m_out, l_out, st);
  }
  {
    merge_generic<T, A><<<grid, 256, 0, st>>>(mode, idx, (const A*)obuf, (const A*)ml, (const A*)mg,
                                              (const A*)lg, (A*)out, (A*)lse, (A*)m_out, (A*)l_out,
                                              shared_max, *s);
  }
  FSA_LAUNCH_CHECK("merge_fwd");
  return FSA_OK;
}

template <typename T>
int delta_impl(const fsa_shape* s, const void* out, const void* dOut, void* delta, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  delta_kernel<T><<<(unsigned)((rows + 7) / 8), 256, 0, st>>>((const A*)out, (const T*)dOut,
                                                              (A*)delta, *s);
  FSA_LAUNCH_CHECK("bwd_delta");
  return FSA_OK;
}

template <typename T>
int sel_bwd_impl(const fsa_shape* s, const void* Q, const void* K, const void* V, const void* dOut,
                 const void* lse, const void* delta, const int32_t* offsets, const int32_t* qlist,
                 void* dq_buf, void* dK, void* dV, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t b = s->N / s->B_K;
  const size_t acc_elems = (size_t)(s->B_K * (s->d_K + s->d_V) + s->d_K + s->d_V + 2 * s->B_K);
  const size_t stage_elems = (size_t)(s->B_K * (s->d_K + 1 + s->d_V + 1));
  const bool stage = sizeof(A) * (acc_elems + stage_elems) <= 220 * 1024;
  const size_t smem = sizeof(A) * (acc_elems + (stage ? stage_elems : 0));
  FSA_REQUIRE(smem <= 220 * 1024, "selected backward: B_K=%lld d=%lld exceeds shared memory",
              (long long)s->B_K, (long long)s->d_K);
  auto kern = stage ? sel_bwd_generic<T, true> : sel_bwd_generic<T, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)b, (unsigned)s->h_K);
  kern<<<grid, 128, smem, st>>>((const T*)Q, (const T*)K, (const T*)V,
                                              (const T*)dOut, (const A*)lse, (const A*)delta,
                                              offsets, qlist, (A*)dq_buf, (A*)dK, (A*)dV, *s);
  FSA_LAUNCH_CHECK("sel_bwd");
  return FSA_OK;
}

template <typename T>
int dq_reduce_impl(const fsa_shape* s, const int32_t* idx, const void* dq_buf, int dqbuf_dtype,
                   void* dQ, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t rows = s->h * s->N;
  if (rows == 0) return FSA_OK;
  const unsigned grid = (unsigned)((rows + 7) / 8);
  if (dqbuf_dtype == FSA_DT_F16R) {
    FSA_REQUIRE(fast_reduce_ok(*s) && sizeof(A) == 4, "dq_reduce: fp16 partials need d = 128");
    return dq_reduce_f16r(s, idx, dq_buf, dQ, st);
  }
  dq_reduce_kernel<T, A><<<grid, 256, 0, st>>>(idx, (const A*)dq_buf, (A*)dQ, *s);
  FSA_LAUNCH_CHECK("dq_reduce");
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

extern "C" int fsa_sel_fwd(const fsa_shape* s, int dtype, int mode, const void* Q, const void* K,
                           const void* V, const int32_t* offsets, const int32_t* qlist,
                           const int32_t* work, const void* m_global, void* obuf, int obuf_dtype,
                           void* ml, void* stream) {
  if (mode < FSA_FWD_LOCAL || mode > FSA_FWD_GLOBAL) {
    fsa::set_error("sel_fwd: bad mode %d", mode);
    return FSA_ERR_INVALID;
  }
  if (obuf_dtype == FSA_DT_F16) {  // V is the fsa_v_to_f16 copy
    if (mode != FSA_FWD_LOCAL || !fsa::tc_fwd_supported(*s, dtype)) {
      fsa::set_error("sel_fwd: fp16 partial buffer only on the tensor-core LOCAL path");
      return FSA_ERR_INVALID;
    }
    return fsa::tc_sel_fwd(s, Q, K, V, offsets, qlist, work, obuf, ml, (cudaStream_t)stream);
  }
  DISPATCH_DT(dtype, sel_fwd_impl, s, mode, Q, K, V, offsets, qlist, m_global, obuf, ml,
              (cudaStream_t)stream);
}

extern "C" int fsa_sel_fwd_phase(const fsa_shape* s, int mode, const void* Q, const void* K,
                                 const void* V16, const float* vscale, const int32_t* offsets,
                                 const int32_t* qlist, const int32_t* work, const float* m_global,
                                 float* obuf, float* ml, void* stream) {
  FSA_REQUIRE(fsa::tc_fwd_supported(*s, FSA_DT_BF16),
              "sel_fwd_phase: tensor-core shapes only (bf16, d = 128, B_K = 64)");
  FSA_REQUIRE(mode == FSA_FWD_STATS || mode == FSA_FWD_GLOBAL, "sel_fwd_phase: bad mode %d", mode);
  FSA_REQUIRE(work != nullptr, "sel_fwd_phase: needs the work plan");
  if (mode == FSA_FWD_STATS) {
    FSA_REQUIRE(ml != nullptr, "sel_fwd_phase STATS: ml is required");
  } else {
    FSA_REQUIRE(obuf && m_global && V16 && vscale, "sel_fwd_phase GLOBAL: obuf, m_global, V16 and vscale are required");
  }
  return fsa::tc_sel_fwd(s, Q, K, V16, offsets, qlist, work, obuf, ml, (cudaStream_t)stream, mode,
                         m_global, vscale);
}

extern "C" int fsa_merge_fwd(const fsa_shape* s, int dtype, int mode, const int32_t* idx,
                             const int32_t* work, const void* obuf, int obuf_dtype, const void* ml,
                             const void* m_global, const void* l_global, void* out, void* lse,
                             void* m_out, void* l_out, int shared_max, const float* vscale,
                             void* stream) {
  if (mode == FSA_MERGE_STATS && (!m_out || !l_out)) {
    fsa::set_error("merge_fwd: STATS mode needs m_out and l_out");
    return FSA_ERR_INVALID;
  }
  DISPATCH_DT(dtype, merge_impl, s, mode, idx, work, obuf, obuf_dtype, ml, m_global, l_global, out,
              lse, m_out, l_out, shared_max, vscale, (cudaStream_t)stream);
}

extern "C" int fsa_merge_combine_fwd(const fsa_shape* s, int dtype, const int32_t* idx,
                                     const int32_t* work, const void* obuf, int obuf_dtype,
                                     const void* ml,
                                     const float* vscale, const void* out_cmp,
                                     const void* out_slide, const void* tau, void* out_sel,
                                     void* lse, void* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == FSA_DT_BF16 && obuf_dtype == FSA_DT_F16 && fsa::fast_reduce_ok(*s))
    return fsa::merge_f16_fast(s, idx, work, obuf, ml, vscale, out_sel, lse, nullptr, nullptr, st,
                               out_cmp, out_slide, tau, out);
  int rc = fsa_merge_fwd(s, dtype, FSA_MERGE_LOCAL, idx, work, obuf, obuf_dtype, ml, nullptr,
                         nullptr, out_sel, lse, nullptr, nullptr, 0, vscale, stream);
  if (rc) return rc;
  return fsa_gated_combine(s, dtype, out_cmp, out_sel, out_slide, tau, out, 0, stream);
}

extern "C" int fsa_bwd_delta(const fsa_shape* s, int dtype, const void* out, const void* dOut,
                             void* delta, void* stream) {
  DISPATCH_DT(dtype, delta_impl, s, out, dOut, delta, (cudaStream_t)stream);
}

extern "C" int fsa_sel_bwd(const fsa_shape* s, int dtype, const void* Q, const void* K,
                           const void* V, const void* dOut, const void* lse, const void* delta,
                           const int32_t* offsets, const int32_t* qlist, const int32_t* work,
                           void* dq_buf, int dqbuf_dtype, void* dK, void* dV,
                           const float* scales, void* stream) {
  if (fsa::tc_bwd_supported(*s, dtype)) {  // dq_buf: FSA_DT_F16R rows + exponents
    FSA_REQUIRE(scales != nullptr,
                "sel_bwd: the tensor-core path reads the fsa_stage_f16_ops copies and their scales");
    return fsa::tc_sel_bwd(s, Q, K, V, dOut, lse, delta, offsets, qlist, work, dq_buf, dqbuf_dtype,
                           dK, dV, fsa::f16_scales_of(scales, s->h_K), (cudaStream_t)stream);
  }
  FSA_REQUIRE(dqbuf_dtype == (dtype == FSA_DT_F64 ? FSA_DT_F64 : FSA_DT_F32),
              "sel_bwd: dq buffer dtype mismatch");
  DISPATCH_DT(dtype, sel_bwd_impl, s, Q, K, V, dOut, lse, delta, offsets, qlist, dq_buf, dK, dV,
              (cudaStream_t)stream);
}

extern "C" int fsa_dq_reduce_add(const fsa_shape* s, int dtype, const int32_t* idx,
                                 const void* dq_buf, int dqbuf_dtype, const void* addend, void* dQ,
                                 void* stream) {
  if (dtype == FSA_DT_BF16 && dqbuf_dtype == FSA_DT_F16R && fsa::fast_reduce_ok(*s))
    return fsa::dq_reduce_f16r(s, idx, dq_buf, dQ, (cudaStream_t)stream, addend);
  fsa::set_error("dq_reduce_add: only the bf16 tensor-core configuration (fp16 partials, d = 128)");
  return FSA_ERR_UNSUPPORTED;
}

extern "C" int fsa_dq_reduce(const fsa_shape* s, int dtype, const int32_t* idx, const void* dq_buf,
                             int dqbuf_dtype, void* dQ, void* stream) {
  DISPATCH_DT(dtype, dq_reduce_impl, s, idx, dq_buf, dqbuf_dtype, dQ, (cudaStream_t)stream);
}
