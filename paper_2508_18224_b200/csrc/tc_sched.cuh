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

// A claimed task, decoded once by the producer (its descriptor loads are
// global-memory latency: the consumers read it from shared memory instead).
struct TaskSlot {
  int32_t task;   // -1: no more tasks
  int32_t kh, i;  // kv head, KV block
  int32_t beg;    // first row: CSR entry (selected) or token (window / compressed)
  int32_t ntok;   // rows (tokens) of the task
  int32_t ibase;  // item base in the partial buffers (work plan), if any
  int32_t pad0, pad1;
};
constexpr uint32_t kRingBytes = kRingDepth * sizeof(TaskSlot);

struct Ring {
  uint32_t full0, empty0;  // mbarrier addresses of slot 0 (8 B apart)
  volatile TaskSlot* slots;
  __device__ uint32_t full(int k) const { return full0 + 8u * (uint32_t)(k & (kRingDepth - 1)); }
  __device__ uint32_t empty(int k) const { return empty0 + 8u * (uint32_t)(k & (kRingDepth - 1)); }

  // producer side: claim the next task (or -1 once all are taken) and decode
  // it with dec(task, slot) into the ring
  template <class Dec>
  __device__ void produce(int k, int32_t* counter, int64_t ntask, Dec dec) const {
    mbar_wait(empty(k), (uint32_t)(((k / kRingDepth) & 1) ^ 1));
    const int32_t t = atomicAdd(counter, 1);
    TaskSlot ts{};
    ts.task = (t < ntask) ? t : -1;
    if (ts.task >= 0) dec(t, ts);
    volatile TaskSlot& d = slots[k & (kRingDepth - 1)];
    d.task = ts.task;
    d.kh = ts.kh;
    d.i = ts.i;
    d.beg = ts.beg;
    d.ntok = ts.ntok;
    d.ibase = ts.ibase;
    mbar_arrive(full(k));
  }
  __device__ TaskSlot read(int k) const {
    const volatile TaskSlot& d = slots[k & (kRingDepth - 1)];
    TaskSlot ts;
    ts.task = d.task;
    ts.kh = d.kh;
    ts.i = d.i;
    ts.beg = d.beg;
    ts.ntok = d.ntok;
    ts.ibase = d.ibase;
    ts.pad0 = ts.pad1 = 0;
    return ts;
  }
  // warp-wide non-blocking consumer: false if slot k is not filled yet
  __device__ bool try_consume_warp(int k, TaskSlot& ts) const {
    if (!mbar_test_warp(full(k), (uint32_t)((k / kRingDepth) & 1))) return false;
    ts = read(k);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(empty(k));
    return true;
  }
  // warp-wide blocking consumer: lane 0 waits, all lanes read, lane 0 arrives
  __device__ TaskSlot consume_warp(int k) const {
    if ((threadIdx.x & 31) == 0) mbar_wait(full(k), (uint32_t)((k / kRingDepth) & 1));
    __syncwarp();
    const TaskSlot ts = read(k);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(empty(k));
    return ts;
  }
  // consumer side
  __device__ TaskSlot consume(int k) const {
    mbar_wait(full(k), (uint32_t)((k / kRingDepth) & 1));
    const TaskSlot ts = read(k);
    mbar_arrive(empty(k));
    return ts;
  }
};

// Static description of a task's rows.
struct TaskRows {
  int64_t i, kh, beg, ntok;  // block, kv head, CSR start, number of attending tokens
  int nitems;                // ceil(ntok / tpi)
};

__device__ __forceinline__ TaskRows rows_of_slot(const TaskSlot& ts, int tpi) {
  TaskRows r;
  r.kh = ts.kh;
  r.i = ts.i;
  r.beg = ts.beg;
  r.ntok = ts.ntok;
  r.nitems = (int)((r.ntok + tpi - 1) / tpi);
  return r;
}

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
