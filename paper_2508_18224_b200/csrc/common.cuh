// Shared device helpers for the FSA / NSA sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <math.h>

#include "../../include/fsa_b200.h"

namespace fsa {

// ---------------------------------------------------------------------------
// element / accumulator traits: f32 -> f32 acc, f64 -> f64 acc, bf16 -> f32 acc
// ---------------------------------------------------------------------------
template <typename T> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ float to_acc(float x) { return x; }
__device__ __forceinline__ double to_acc(double x) { return x; }
__device__ __forceinline__ float to_acc(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_acc(float x);
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <typename T> __device__ __forceinline__ T from_acc(double x);
template <> __device__ __forceinline__ double from_acc<double>(double x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(double x) { return __double2bfloat16(x); }

__device__ __forceinline__ float exp_acc(float x) { return expf(x); }
__device__ __forceinline__ double exp_acc(double x) { return exp(x); }
__device__ __forceinline__ float log_acc(float x) { return logf(x); }
__device__ __forceinline__ double log_acc(double x) { return log(x); }

template <typename A> __device__ __forceinline__ A neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return -INFINITY; }
template <> __device__ __forceinline__ double neg_inf<double>() { return -(double)INFINITY; }

// ---------------------------------------------------------------------------
// warp reductions
// ---------------------------------------------------------------------------
template <typename A> __device__ __forceinline__ A warp_max(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <typename A> __device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------------------
// host-side error plumbing
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);

// ---------------------------------------------------------------------------
// Work plan of the tensor-core selected branch (fsa_build_inverse's `work`,
// int32): [0, ntask] the item prefix over head-major tasks (task = kh * b + i;
// an item is <= 128 rows = tpi tokens x g heads), [ntask + 1] the persistent
// kernels' scheduler counter, then from plan_pos_offset the position of every
// live selection entry (kh, t, slot) in its task's query list.  Item n owns
// rows [128 n, 128 n + 128) of the partial buffers (obuf / ml / dq partials):
// row 128 n + (p % tpi) g + hh for list position p and group head hh.
// ---------------------------------------------------------------------------
__host__ __device__ inline int64_t plan_ntask(const fsa_shape& s) { return s.h_K * (s.N / s.B_K); }
__host__ __device__ inline int64_t plan_pos_offset(const fsa_shape& s) {
  return ((plan_ntask(s) + 2 + 31) / 32) * 32;
}
__host__ __device__ inline int64_t plan_tpi(const fsa_shape& s) {
  const int64_t g = s.h / s.h_K;
  return g >= 128 ? 1 : 128 / g;
}
// item count bound: a valid selection has <= min(t / B_K + 1, T) entries per
// token, so nnz <= B_K * sum_j min(j + 1, T) per kv head, and every task adds
// at most one partial item
inline int64_t plan_max_items(const fsa_shape& s) {
  const int64_t b = s.N / s.B_K, T = s.T;
  const int64_t cols = b <= T ? b * (b + 1) / 2 : T * (T + 1) / 2 + (b - T) * T;
  const int64_t nnz = s.B_K * cols, tpi = plan_tpi(s);
  return s.h_K * ((nnz + tpi - 1) / tpi + b);
}

}  // namespace fsa

#define FSA_REQUIRE(cond, ...)            \
  do {                                    \
    if (!(cond)) {                        \
      ::fsa::set_error(__VA_ARGS__);      \
      return FSA_ERR_INVALID;             \
    }                                     \
  } while (0)

#define FSA_LAUNCH_CHECK(what)                          \
  do {                                                  \
    int _rc = ::fsa::check_launch(what);                \
    if (_rc) return _rc;                                \
  } while (0)
