// NSA query-major selected-attention forward (the paper's baseline schedule,
// query_major.py:45-69, _core.pyx:134-181): one task per (kv head, token)
// batches the group's g query heads and walks the token's selected KV blocks
// in ascending order with an online softmax; the own (partially causal) block
// is loaded in full and masked by position.
//
// This is the FSA-vs-NSA comparison point, on CUDA
// cores: each task is g rows, far below the M = 64/128 a tcgen05 MMA needs --
// exactly the under-utilisation the FSA KV-block-major order removes.  One
// warp per task; lanes own keys for Q.K and features for P.V.
#include "common.cuh"

namespace fsa {
namespace {

template <typename T, int kMaxG, int kNQ>  // kMaxG >= g heads, kNQ * 32 >= d_V
__global__ void __launch_bounds__(128) qm_fwd_kernel(const T* __restrict__ Q, const T* __restrict__ K,
                                                     const T* __restrict__ V,
                                                     const int32_t* __restrict__ idx,
                                                     typename Acc<T>::type* __restrict__ out,
                                                     typename Acc<T>::type* __restrict__ lse,
                                                     fsa_shape s) {
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t task = blockIdx.x * 4ll + wib;  // (kh, t), t fastest
  if (task >= s.h_K * s.N) return;
  const int64_t kh = task / s.N, t = task % s.N;
  const int g = (int)(s.h / s.h_K), dK = (int)s.d_K, dV = (int)s.d_V, BK = (int)s.B_K;
  A* qs = reinterpret_cast<A*>(smem_raw) + (int64_t)wib * g * dK;  // this warp's g query rows
  for (int e = lane; e < g * dK; e += 32) {
    const int hh = e / dK, c = e % dK;
    qs[e] = to_acc(Q[(t * s.h + kh * g + hh) * dK + c]);
  }
  __syncwarp();
  A m[kMaxG], l[kMaxG], o[kMaxG][kNQ];  // o: features lane + 32 q
#pragma unroll
  for (int hh = 0; hh < kMaxG; ++hh) {
    m[hh] = neg_inf<A>();
    l[hh] = A(0);
#pragma unroll
    for (int q = 0; q < kNQ; ++q) o[hh][q] = A(0);
  }
  const int32_t* row = idx + (kh * s.N + t) * s.T;
  for (int slot = 0; slot < (int)s.T; ++slot) {
    const int i = row[slot];
    if (i < 0) break;
    for (int k0 = 0; k0 < BK; k0 += 32) {  // 32 keys of the block at a time
      const int key = k0 + lane;
      const int64_t pos = (int64_t)i * BK + key;
      const bool vis = key < BK && pos <= t;
      A z[kMaxG];
#pragma unroll
      for (int hh = 0; hh < kMaxG; ++hh) z[hh] = A(0);
      if (vis) {
        const T* kr = K + (pos * s.h_K + kh) * dK;
        for (int c = 0; c < dK; ++c) {
          const A kv = to_acc(kr[c]);
#pragma unroll
          for (int hh = 0; hh < kMaxG; ++hh)
            if (hh < g) z[hh] += qs[hh * dK + c] * kv;
        }
      }
#pragma unroll
      for (int hh = 0; hh < kMaxG; ++hh) {
        if (hh >= g) break;
        const A zz = vis ? z[hh] * A(s.scale) : neg_inf<A>();
        const A bm = warp_max(zz);
        if (bm == neg_inf<A>()) continue;  // no visible key in this chunk
        const A mn = m[hh] > bm ? m[hh] : bm;
        const A f = exp_acc(m[hh] - mn);
        const A p = vis ? exp_acc(zz - mn) : A(0);
        l[hh] = l[hh] * f + warp_sum(p);
        m[hh] = mn;
#pragma unroll
        for (int q = 0; q < kNQ; ++q) o[hh][q] *= f;
        z[hh] = p;
      }
      // O += P V: lanes over features, keys broadcast
      const int nk = min(32, BK - k0);
      for (int kk = 0; kk < nk; ++kk) {
        const int64_t p2 = (int64_t)i * BK + k0 + kk;
        if (p2 > t) break;
        const T* vr = V + (p2 * s.h_K + kh) * dV;
        A vv[kNQ];
#pragma unroll
        for (int q = 0; q < kNQ; ++q) vv[q] = (lane + 32 * q < dV) ? to_acc(vr[lane + 32 * q]) : A(0);
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
          if (hh >= g) break;
          const A pk = __shfl_sync(0xffffffffu, z[hh], kk);
#pragma unroll
          for (int q = 0; q < kNQ; ++q) o[hh][q] += pk * vv[q];
        }
      }
    }
  }
#pragma unroll
  for (int hh = 0; hh < kMaxG; ++hh) {
    if (hh >= g) break;
    const int64_t j = kh * g + hh;
    const A inv = A(1) / l[hh];
#pragma unroll
    for (int q = 0; q < kNQ; ++q)
      if (lane + 32 * q < dV) out[(t * s.h + j) * dV + lane + 32 * q] = o[hh][q] * inv;
    if (lane == 0) lse[j * s.N + t] = m[hh] + log_acc(l[hh]);
  }
}

template <typename T, int G, int NQ>
int qm_launch(const fsa_shape* s, const void* Q, const void* K, const void* V, const int32_t* idx,
              void* out, void* lse, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t g = s->h / s->h_K;
  const size_t smem = (size_t)4 * g * s->d_K * sizeof(A);
  FSA_REQUIRE(smem <= 200 * 1024, "query-major forward: g*d_K too large");
  cudaFuncSetAttribute(qm_fwd_kernel<T, G, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t tasks = s->h_K * s->N;
  if (tasks == 0) return FSA_OK;
  qm_fwd_kernel<T, G, NQ><<<(unsigned)((tasks + 3) / 4), 128, smem, st>>>(
      (const T*)Q, (const T*)K, (const T*)V, idx, (A*)out, (A*)lse, *s);
  FSA_LAUNCH_CHECK("qm_fwd");
  return FSA_OK;
}

template <typename T, int G>
int qm_fwd_nq(const fsa_shape* s, const void* Q, const void* K, const void* V, const int32_t* idx,
              void* out, void* lse, cudaStream_t st) {
  if (s->d_V <= 64) return qm_launch<T, G, 2>(s, Q, K, V, idx, out, lse, st);
  if (s->d_V <= 128) return qm_launch<T, G, 4>(s, Q, K, V, idx, out, lse, st);
  return qm_launch<T, G, 8>(s, Q, K, V, idx, out, lse, st);
}

template <typename T>
int qm_fwd_impl(const fsa_shape* s, const void* Q, const void* K, const void* V, const int32_t* idx,
                void* out, void* lse, cudaStream_t st) {
  const int64_t g = s->h / s->h_K;
  FSA_REQUIRE(g <= 16, "query-major forward: g=%lld > 16", (long long)g);
  FSA_REQUIRE(s->d_V <= 256, "query-major forward: d_V=%lld > 256", (long long)s->d_V);
  if (g <= 2) return qm_fwd_nq<T, 2>(s, Q, K, V, idx, out, lse, st);
  if (g <= 4) return qm_fwd_nq<T, 4>(s, Q, K, V, idx, out, lse, st);
  if (g <= 8) return qm_fwd_nq<T, 8>(s, Q, K, V, idx, out, lse, st);
  return qm_fwd_nq<T, 16>(s, Q, K, V, idx, out, lse, st);
}


// Query-major backward (query_major.py:72-99, _core.pyx:184-241): the same
// (kv head, token) tasks recompute P = exp(z - lse) for the token's selected
// blocks, accumulate the g rows' dQ in the warp's shared memory, and scatter
// dK / dV rows with atomics -- many tasks select the same block, so a
// query-major schedule has no single writer per KV row.  That scatter (and
// its non-deterministic summation order) is the cost the FSA KV-block-major
// backward removes.  Lanes own keys for the score products and features for
// the row updates; the g heads are summed in registers before each atomic.
template <typename T, int kMaxG>
__global__ void __launch_bounds__(128) qm_bwd_kernel(const T* __restrict__ Q, const T* __restrict__ K,
                                                     const T* __restrict__ V, const T* __restrict__ dOut,
                                                     const int32_t* __restrict__ idx,
                                                     const typename Acc<T>::type* __restrict__ lse,
                                                     const typename Acc<T>::type* __restrict__ delta,
                                                     typename Acc<T>::type* __restrict__ dQ,
                                                     typename Acc<T>::type* __restrict__ gK,
                                                     typename Acc<T>::type* __restrict__ gV, fsa_shape s) {
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t task = blockIdx.x * 4ll + wib;  // (kh, t), t fastest
  if (task >= s.h_K * s.N) return;
  const int64_t kh = task / s.N, t = task % s.N;
  const int g = (int)(s.h / s.h_K), dK = (int)s.d_K, dV = (int)s.d_V, BK = (int)s.B_K;
  const A sc = A(s.scale);
  A* qs = reinterpret_cast<A*>(smem_raw) + (int64_t)wib * g * (2 * dK + dV);
  A* dos = qs + g * dK;
  A* dqs = dos + g * dV;
  for (int e = lane; e < g * dK; e += 32) {
    const int hh = e / dK, c = e % dK;
    qs[e] = to_acc(Q[(t * s.h + kh * g + hh) * dK + c]);
    dqs[e] = A(0);
  }
  for (int e = lane; e < g * dV; e += 32) {
    const int hh = e / dV, c = e % dV;
    dos[e] = to_acc(dOut[(t * s.h + kh * g + hh) * dV + c]);
  }
  A lz[kMaxG], dl[kMaxG];
#pragma unroll
  for (int hh = 0; hh < kMaxG; ++hh) {
    lz[hh] = hh < g ? lse[(kh * g + hh) * s.N + t] : A(0);
    dl[hh] = hh < g ? delta[(kh * g + hh) * s.N + t] : A(0);
  }
  __syncwarp();
  const int32_t* row = idx + (kh * s.N + t) * s.T;
  for (int slot = 0; slot < (int)s.T; ++slot) {
    const int i = row[slot];
    if (i < 0) break;
    if ((int64_t)i * BK > t) continue;
    for (int k0 = 0; k0 < BK; k0 += 32) {
      const int key = k0 + lane;
      const int64_t pos = (int64_t)i * BK + key;
      const bool vis = key < BK && pos <= t;
      A p[kMaxG], ds[kMaxG];
#pragma unroll
      for (int hh = 0; hh < kMaxG; ++hh) p[hh] = ds[hh] = A(0);
      if (vis) {
        const T* kr = K + (pos * s.h_K + kh) * dK;
        for (int c = 0; c < dK; ++c) {
          const A kv = to_acc(kr[c]);
#pragma unroll
          for (int hh = 0; hh < kMaxG; ++hh)
            if (hh < g) p[hh] += qs[hh * dK + c] * kv;
        }
        const T* vr = V + (pos * s.h_K + kh) * dV;
        for (int c = 0; c < dV; ++c) {
          const A vv = to_acc(vr[c]);
#pragma unroll
          for (int hh = 0; hh < kMaxG; ++hh)
            if (hh < g) ds[hh] += dos[hh * dV + c] * vv;
        }
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
          if (hh >= g) break;
          p[hh] = exp_acc(p[hh] * sc - lz[hh]);
          ds[hh] = p[hh] * (ds[hh] - dl[hh]);
        }
      }
      const int nk = min(32, BK - k0);
      for (int kk = 0; kk < nk; ++kk) {
        const int64_t p2 = (int64_t)i * BK + k0 + kk;
        if (p2 > t) break;
        A pk[kMaxG], dk[kMaxG];
#pragma unroll
        for (int hh = 0; hh < kMaxG; ++hh) {
          pk[hh] = __shfl_sync(0xffffffffu, p[hh], kk);
          dk[hh] = __shfl_sync(0xffffffffu, ds[hh], kk);
        }
        const T* kr = K + (p2 * s.h_K + kh) * dK;
        A* dkr = gK + (p2 * s.h_K + kh) * dK;
        for (int c = lane; c < dK; c += 32) {
          const A kv = to_acc(kr[c]);
          A acc = A(0);
#pragma unroll
          for (int hh = 0; hh < kMaxG; ++hh) {
            if (hh >= g) break;
            dqs[hh * dK + c] += sc * dk[hh] * kv;
            acc += dk[hh] * qs[hh * dK + c];
          }
          atomicAdd(dkr + c, sc * acc);
        }
        A* dvr = gV + (p2 * s.h_K + kh) * dV;
        for (int c = lane; c < dV; c += 32) {
          A acc = A(0);
#pragma unroll
          for (int hh = 0; hh < kMaxG; ++hh) {
            if (hh >= g) break;
            acc += pk[hh] * dos[hh * dV + c];
          }
          atomicAdd(dvr + c, acc);
        }
      }
    }
  }
  __syncwarp();
  for (int e = lane; e < g * dK; e += 32) {
    const int hh = e / dK, c = e % dK;
    dQ[(t * s.h + kh * g + hh) * dK + c] = dqs[e];
  }
}

template <typename T, int G>
int qm_bwd_launch(const fsa_shape* s, const void* Q, const void* K, const void* V, const void* dOut,
                  const int32_t* idx, const void* lse, const void* delta, void* dQ, void* dK, void* dV,
                  cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t g = s->h / s->h_K;
  const size_t smem = (size_t)4 * g * (2 * s->d_K + s->d_V) * sizeof(A);
  FSA_REQUIRE(smem <= 200 * 1024, "query-major backward: g*(2 d_K + d_V) too large");
  cudaFuncSetAttribute(qm_bwd_kernel<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t tasks = s->h_K * s->N;
  if (tasks == 0) return FSA_OK;
  qm_bwd_kernel<T, G><<<(unsigned)((tasks + 3) / 4), 128, smem, st>>>(
      (const T*)Q, (const T*)K, (const T*)V, (const T*)dOut, idx, (const A*)lse, (const A*)delta,
      (A*)dQ, (A*)dK, (A*)dV, *s);
  FSA_LAUNCH_CHECK("qm_bwd");
  return FSA_OK;
}

template <typename T>
int qm_bwd_impl(const fsa_shape* s, const void* Q, const void* K, const void* V, const void* dOut,
                const int32_t* idx, const void* lse, const void* delta, void* dQ, void* dK, void* dV,
                cudaStream_t st) {
  using A = typename Acc<T>::type;
  const int64_t g = s->h / s->h_K;
  FSA_REQUIRE(g <= 16, "query-major backward: g=%lld > 16", (long long)g);
  cudaMemsetAsync(dK, 0, (size_t)(s->N * s->h_K * s->d_K) * sizeof(A), st);
  cudaMemsetAsync(dV, 0, (size_t)(s->N * s->h_K * s->d_V) * sizeof(A), st);
  if (g <= 2) return qm_bwd_launch<T, 2>(s, Q, K, V, dOut, idx, lse, delta, dQ, dK, dV, st);
  if (g <= 4) return qm_bwd_launch<T, 4>(s, Q, K, V, dOut, idx, lse, delta, dQ, dK, dV, st);
  if (g <= 8) return qm_bwd_launch<T, 8>(s, Q, K, V, dOut, idx, lse, delta, dQ, dK, dV, st);
  return qm_bwd_launch<T, 16>(s, Q, K, V, dOut, idx, lse, delta, dQ, dK, dV, st);
}

}  // namespace
}  // namespace fsa

extern "C" int fsa_qm_fwd(const fsa_shape* s, int dtype, const void* Q, const void* K, const void* V,
                          const int32_t* idx, void* out, void* lse, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (dtype) {
    case FSA_DT_F32: return fsa::qm_fwd_impl<float>(s, Q, K, V, idx, out, lse, st);
    case FSA_DT_F64: return fsa::qm_fwd_impl<double>(s, Q, K, V, idx, out, lse, st);
    case FSA_DT_BF16: return fsa::qm_fwd_impl<__nv_bfloat16>(s, Q, K, V, idx, out, lse, st);
    default: fsa::set_error("qm_fwd: unsupported dtype %d", dtype); return FSA_ERR_INVALID;
  }
}

extern "C" int fsa_qm_bwd(const fsa_shape* s, int dtype, const void* Q, const void* K, const void* V,
                          const void* dOut, const int32_t* idx, const void* lse, const void* delta,
                          void* dQ, void* dK, void* dV, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (dtype) {
    case FSA_DT_F32: return fsa::qm_bwd_impl<float>(s, Q, K, V, dOut, idx, lse, delta, dQ, dK, dV, st);
    case FSA_DT_F64: return fsa::qm_bwd_impl<double>(s, Q, K, V, dOut, idx, lse, delta, dQ, dK, dV, st);
    case FSA_DT_BF16:
      return fsa::qm_bwd_impl<__nv_bfloat16>(s, Q, K, V, dOut, idx, lse, delta, dQ, dK, dV, st);
    default: fsa::set_error("qm_bwd: unsupported dtype %d", dtype); return FSA_ERR_INVALID;
  }
}
