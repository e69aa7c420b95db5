// Persistent-kernel task scheduling shared by the tcgen05 FSA kernels.
//
// Tasks are (kv head, KV block) pairs in head-major order: task = kh * b + i.
// CTAs claim whole tasks from a global atomic counter (dynamic, so heavy and
// light blocks balance), which keeps every CTA inside the same kv head at the
// same time: the gathered query (and dOut) rows of one kv group -- 33.5 MB of
// Q at 32K tokens -- stay resident in the 126 MB L2 while all blocks of that
// head are processed.  Within a head, early blocks (the heaviest: they are
// causal for every later token) come first.  A whole task stays on one CTA,
// so the backward's dK/dV for a block has a single writer (deterministic).
//
// One producer thread claims tasks into a 4-deep shared-memory ring guarded by
// mbarriers; every consumer thread reads each entry once and arrives.
#pragma once
#include "tc_common.cuh"

namespace fsa {
namespace tc {

constexpr int kRingDepth = 4;

struct Ring {
  uint32_t full0, empty0;  // mbarrier addresses of slot 0 (8 B apart)
  volatile int32_t* slots;
  __device__ uint32_t full(int k) const { return full0 + 8u * (uint32_t)(k & (kRingDepth - 1)); }
  __device__ uint32_t empty(int k) const { return empty0 + 8u * (uint32_t)(k & (kRingDepth - 1)); }

  // producer side: claim the next task (or -1 once all are taken)
  __device__ void produce(int k, int32_t* counter, int64_t ntask) const {
    mbar_wait(empty(k), (uint32_t)(((k / kRingDepth) & 1) ^ 1));
    int32_t t = atomicAdd(counter, 1);
    slots[k & (kRingDepth - 1)] = (t < ntask) ? t : -1;
    mbar_arrive(full(k));
  }
  // consumer side, non-blocking: false if slot k is not filled yet
  __device__ bool try_consume(int k, int32_t& t) const {
    if (!mbar_test(full(k), (uint32_t)((k / kRingDepth) & 1))) return false;
    t = slots[k & (kRingDepth - 1)];
    mbar_arrive(empty(k));
    return true;
  }
  // warp-wide non-blocking consumer: all lanes read the slot, one arrives
  __device__ bool try_consume_warp(int k, int32_t& t) const {
    if (!mbar_test_warp(full(k), (uint32_t)((k / kRingDepth) & 1))) return false;
    t = slots[k & (kRingDepth - 1)];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(empty(k));
    return true;
  }
  // warp-wide blocking consumer: lane 0 waits, all lanes read, lane 0 arrives
  __device__ int32_t consume_warp(int k) const {
    if ((threadIdx.x & 31) == 0) mbar_wait(full(k), (uint32_t)((k / kRingDepth) & 1));
    __syncwarp();
    const int32_t t = slots[k & (kRingDepth - 1)];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(empty(k));
    return t;
  }
  // consumer side
  __device__ int32_t consume(int k) const {
    mbar_wait(full(k), (uint32_t)((k / kRingDepth) & 1));
    const int32_t t = slots[k & (kRingDepth - 1)];
    mbar_arrive(empty(k));
    return t;
  }
};

// Static description of a task's rows.
struct TaskRows {
  int64_t i, kh, beg, ntok;  // block, kv head, CSR start, number of attending tokens
  int nitems;                // ceil(ntok / tpi)
};

__device__ __forceinline__ TaskRows task_rows(int32_t task, const int32_t* offsets, int64_t b,
                                              int tpi) {
  TaskRows r;
  r.kh = task / b;
  r.i = task % b;
  const int32_t* off = offsets + r.kh * (b + 1) + r.i;
  r.beg = off[0];
  r.ntok = off[1] - off[0];
  r.nitems = (int)((r.ntok + tpi - 1) / tpi);
  return r;
}

}  // namespace tc
}  // namespace fsa
