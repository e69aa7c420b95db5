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
// int32), token-chunked: the tokens are cut into chunks of C (a multiple of
// 256) and a task is (kv head kh, chunk c, block i) -- the entries of block
// i's query list whose token lies in chunk c (a contiguous sub-list: lists are
// token-sorted).  Tasks are numbered kh-major, then chunk, then block, the
// order the persistent kernels claim them, so at any time every CTA gathers
// query rows of the same C tokens of one kv head (an L2-resident working set
// for small C; measured not to pay, so C = N by default).  Chunk c holds the blocks
// that a token of it can select, i < bic(c) = min(b, (min((c+1) C, N) - 1) / B_K + 1).
//
//   [0] C  [1] nc  [2] tasks per kv head  [3] scheduler counter
//   [64, 64 + nc)            task base of chunk c within a kv head
//   item  [ntask + 1]        exclusive prefix of item counts (an item is <= 128
//                            rows = tpi tokens x g heads); item n owns rows
//                            [128 n, 128 n + 128) of the partial buffers
//   tbeg  [ntask]            first entry of the task in the kv head's qlist
//   tn    [ntask]            entries of the task
//   tki   [ntask]            kh * b + i
//   pos   [h_K][N][T]        position of entry (kh, t, slot) in its task's
//                            sub-list: its row is 128 (item[task] + p / tpi)
//                            + (p % tpi) g + hh
// ---------------------------------------------------------------------------
constexpr int kPlanMaxChunks = 64;
constexpr int64_t kPlanHeader = 128;
__host__ __device__ inline int64_t plan_tpi(const fsa_shape& s) {
  const int64_t g = s.h / s.h_K;
  return g >= 128 ? 1 : 128 / g;
}
// C (inverse.cu): N by default (one chunk); FSA_CHUNK_TOKENS overrides it
int64_t plan_chunk_tokens(const fsa_shape& s);
__host__ __device__ inline int64_t plan_bic(const fsa_shape& s, int64_t C, int64_t c) {
  const int64_t b = s.N / s.B_K;
  const int64_t tend = (c + 1) * C < s.N ? (c + 1) * C : s.N;
  const int64_t n = (tend - 1) / s.B_K + 1;
  return n < b ? n : b;
}
inline int64_t plan_nchunks(const fsa_shape& s) {
  const int64_t C = plan_chunk_tokens(s);
  return s.N <= 0 ? 0 : (s.N + C - 1) / C;
}
inline int64_t plan_tasks_per_head(const fsa_shape& s) {
  const int64_t C = plan_chunk_tokens(s), nc = plan_nchunks(s);
  int64_t n = 0;
  for (int64_t c = 0; c < nc; ++c) n += plan_bic(s, C, c);
  return n;
}
inline int64_t plan_ntask(const fsa_shape& s) { return s.h_K * plan_tasks_per_head(s); }
inline int64_t align32(int64_t x) { return (x + 31) / 32 * 32; }
inline int64_t plan_item_offset(const fsa_shape&) { return kPlanHeader; }
inline int64_t plan_tbeg_offset(const fsa_shape& s) { return align32(kPlanHeader + plan_ntask(s) + 1); }
inline int64_t plan_tn_offset(const fsa_shape& s) { return plan_tbeg_offset(s) + align32(plan_ntask(s)); }
inline int64_t plan_tki_offset(const fsa_shape& s) { return plan_tn_offset(s) + align32(plan_ntask(s)); }
inline int64_t plan_pos_offset(const fsa_shape& s) { return plan_tki_offset(s) + align32(plan_ntask(s)); }
// device view of a plan (built by fsa_build_inverse)
struct PlanView {
  const int32_t *item, *tbeg, *tn, *tki, *pos, *cbase;
  int32_t* counter;
  int32_t C, nph;
};
inline PlanView plan_view(const fsa_shape& s, const int32_t* work) {
  PlanView v;
  v.item = work + plan_item_offset(s);
  v.tbeg = work + plan_tbeg_offset(s);
  v.tn = work + plan_tn_offset(s);
  v.tki = work + plan_tki_offset(s);
  v.pos = work + plan_pos_offset(s);
  v.cbase = work + 64;
  v.counter = const_cast<int32_t*>(work) + 3;
  v.C = (int32_t)plan_chunk_tokens(s);
  v.nph = (int32_t)plan_tasks_per_head(s);
  return v;
}
// item count bound: a valid selection has <= min(t / B_K + 1, T) entries per
// token, so nnz <= B_K * sum_j min(j + 1, T) per kv head, and every task adds
// at most one partial item
inline int64_t plan_max_items(const fsa_shape& s) {
  const int64_t b = s.N / s.B_K, T = s.T;
  const int64_t cols = b <= T ? b * (b + 1) / 2 : T * (T + 1) / 2 + (b - T) * T;
  const int64_t nnz = s.B_K * cols, tpi = plan_tpi(s);
  return s.h_K * ((nnz + tpi - 1) / tpi + plan_tasks_per_head(s));
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
