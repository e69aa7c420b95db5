// FSA selected-attention backward on tcgen05 tensor cores (K8), bf16,
// d = 128, B_K = 64.  Replaces kv_major.py:297-324 / _core.pyx:97-131 and the
// per-group dK/dV head sum (kv_major.py:342-354): one task = one (kv head,
// block i); all g query heads of every gathered row are processed against
// K_i / V_i held in shared memory, and dK_i, dV_i accumulate in TMEM across
// the whole task (single writer, fixed order -> deterministic).
//
// Per 128-row item (TPI tokens x g heads), rows = gathered (token, slot):
//   S   = Q K^T          M128 N64  K128   TMEM stage s, cols [0, 64)
//   dP  = dO V^T         M128 N64  K128   TMEM stage s, cols [64, 128)
//   P   = exp(S*scale - lse),  dS = P * (dP - delta)      (softmax warps, fp16 -> smem)
//   dV^T += dO^T P       M128(d) N64 K128(rows)  TMEM accumulator
//   dK^T += Q^T dS       M128(d) N64 K128(rows)  TMEM accumulator
//   dQ_i  = dS K         M128 N128 K64  -> TMEM stage s (over the consumed S/dP)
//                                        -> fp16 partial row of dq_buf with a
//                                           power-of-two exponent per 32 columns
// dq partial rows are slot-indexed [h][N][T] (the dQ reduce then reads each
// token's rows contiguously; item-major tiles measured no faster here and a
// 1.6x slower reduce).
// dQ partials are summed over the token's selected blocks in ascending block
// order by the dq_reduce kernel (kv_major.py:326-340).
//
// Every product runs fp16 x fp16 -> fp32 on the fsa_stage_f16_ops copies
// Q16 = Q s_Q, K16 = K s_K, V16 = V s_V, dO16 = dO s_dO (power-of-two scales
// per kv head, max |x s| in [2^14, 2^15)): S and dP come out exact as with
// bf16 operands, while P and dS are rounded to 11 bits instead of 8 -- the
// rounding behind elementwise dQ / dK / dV errors (tools/emulate_bf16.py).
// Stored operands:  P16 = P 2^15 (P <= 1),  dS16 = P (dP16 - delta s_V s_dO) 2^-23,
// where |dP16|, |delta s_V s_dO| <= 128 2^15 2^15 (|out| <= max|V|), so
// |dS16| <= 2^15 < 65504 for any input scale; the epilogues divide the scales out.
//
// Roles: warps 0-7 two softmax warpgroups that ping-pong over items (wg owns
// items n with n % 2 == wg and its own Q/dO, S/dP and P/dS stages; after its
// item's products land it stages the dQ epilogue in its now-free P/dS smem),
// warps 8-11 loaders: K_i / V_i of each task by 3-D TMA boxes (one lane),
// the item's gathered Q / dO rows by cp.async (one item's gather kept in
// flight; TMA tile::gather4 measured ~70 cycles per 512 B request -- too slow
// for 64 KB items), warp 12 the MMA issuer (S/dP of item n+1 issued ahead of
// the products of item n).
// Tasks are claimed dynamically, head-major (tc_sched.cuh).  The sliding
// branch's backward runs the same kernel with each block's contiguous token
// window as its rows and a band mask (oracle.py:102-131).
#include "tc_plan.cuh"
#include "tc_sched.cuh"

namespace fsa {
namespace {

using namespace tc;

constexpr int kD = 128, kBK = 64, kRows = 128;
// 8 softmax warps + loader warps + 1 MMA warp.  The selected mode gathers with
// 4 cp.async loader warps (13 warps: 128 registers); the window / compressed
// modes load by TMA from one lane, so one loader warp (10 warps: 168 registers)
template <int SL> constexpr int loader_warps() { return SL == 0 ? 4 : 1; }
template <int SL> constexpr int threads_of() { return (9 + loader_warps<SL>()) * 32; }

constexpr uint32_t kTile = kRows * kD * 2;  // 32768: [2 halves][128][128 B]
constexpr uint32_t kOffQ = 0;               // Q[2]
constexpr uint32_t kOffDO = 2 * kTile;      // dO[2]
constexpr uint32_t kOffK = 4 * kTile;       // K [2 halves][64][128 B] = 16384
constexpr uint32_t kOffV = kOffK + 16384;
constexpr uint32_t kOffP = kOffV + 16384;   // P[2]  [128][128 B]
constexpr uint32_t kOffDS = kOffP + 32768;  // dS[2] [128][128 B]
constexpr uint32_t kOffBar = kOffDS + 32768;
enum {
  // smem stages (Q/dO, P/dS) by item parity; TMEM stages (S|dP, then dQ) by item mod 3
  B_QDF = 0, B_QDE = 2, B_KVF = 4, B_KVE = 5, B_SDF = 6, B_SDE = 9, B_PDF = 12, B_DQF = 14,
  B_KAF = 17, B_KAE = 18, B_RF = 19, B_RE = 23,
  B_DE = 27,  // selected mode: dO stage free (after the dV product), ahead of Q (QDE)
  kNumBars = 29
};
constexpr uint32_t kOffRing = kOffBar + kNumBars * 8;
constexpr uint32_t kOffTmem = kOffRing + kRingBytes;
constexpr uint32_t kSmemBytes = kOffTmem + 16 + 1024;

// TMEM columns: stage t (= item mod 3) at 128 t (S | dP, later dQ), dK^T 384, dV^T 448.
// The third stage lets S/dP of item n+2 run while item n's dQ is read out.
constexpr int kTStages = 3;
constexpr uint32_t kColDK = 384, kColDV = 448;

constexpr uint32_t kIdS = idesc_f16(128, 64, false, false);  // S, dP
constexpr uint32_t kIdKV = idesc_f16(128, 64, true, true);   // dV^T, dK^T
constexpr uint32_t kIdQ = idesc_f16(128, 128, false, true);  // dQ
constexpr float kP16 = 32768.f;             // P16 = P 2^15
constexpr float kDS16 = 1.f / 8388608.f;    // dS16 = P (dP16 - delta16) 2^-23

struct Params {
  CUtensorMap tmQ, tmO;  // sliding / compressed modes: TMA token boxes of Q / dO
  CUtensorMap tmK, tmV;  // every mode: the task's 64 key rows (TMA boxes)
  CUtensorMap tmDQ;                 // dq partial rows [h N T][128] fp16 (scatter4 stores)
  long long* trace;  // debug timeline (CTA 0, first 256 items), null in production
  const __half *Q, *K, *V, *dO;  // the fp16 staged copies (fsa_stage_f16_ops)
  F16Scales sc;                   // their per-kv-head scales
  const float *lse, *delta;
  const int32_t *offsets, *qlist;
  int32_t* counter;
  __half* dq;         // [h][N][T][128] fp16 rows (FSA_DT_F16R) ...
  int32_t* dqe;       // ... and 4 int8 exponents per row (one per 32 columns): value = x * 2^-e
  float *dK, *dV;     // [N][h_K][128]
  int64_t N, h, h_K, T, b, g, ntask;
  int64_t W;   // sliding mode: window; T is then the number of window slots
  // compressed mode (slide == 2): keys = 64 pooled rows of K_cmp / V_cmp (bf16),
  // rows = a chunk of CH consecutive tokens; dK/dV (the pooled rows' gradients)
  // go to a per-chunk partial slab of cstride floats (tc_cmp_bwd sums them)
  int64_t cmpBK, CH, nct, nch, cstride;
  int tpi, slide, accumulate;  // accumulate: dK/dV += (sliding branch onto the selected one)
  int no_dq;                   // sliding mode: dQ comes from the query-outer kernel (tc_slide_dq.cu)
  FastDiv fdT;
  float scale, scale_log2;
};

#ifdef FSA_TRACE
#define K8_TRACE(item, slot)                                                        \
  do {                                                                              \
    if (p.trace && blockIdx.x == 0 && (item) < 256) p.trace[(item) * 16 + (slot)] = clock64(); \
  } while (0)
#else
#define K8_TRACE(item, slot) \
  do {                     \
  } while (0)
#endif

// Rows of a task: the selected mode reads them from the inverse CSR; the
// sliding mode uses the contiguous window of tokens [64 i, 64 i + 63 + W - 1].
template <int SL>
__device__ __forceinline__ TaskRows rows_of(const Params& p, int32_t task) {
  if (SL == 0) return task_rows(task, p.offsets, p.b, p.tpi);
  TaskRows r;
  if (SL == 2) {  // task = (kv head, pooled-row tile, token chunk), chunk fastest
    const int64_t per = p.nct * p.nch;
    r.kh = task / per;
    r.i = (task % per) / p.nch;
    const int64_t q = task % p.nch, first = (r.i * kBK + 1) * p.cmpBK - 1;
    r.beg = q * p.CH > first ? q * p.CH : first;
    const int64_t end = (q + 1) * p.CH < p.N ? (q + 1) * p.CH : p.N;
    r.ntok = end > r.beg ? end - r.beg : 0;
    r.nitems = (int)((r.ntok + p.tpi - 1) / p.tpi);
    return r;
  }
  r.kh = task / p.b;
  r.i = task % p.b;
  r.beg = r.i * kBK;
  const int64_t end = r.beg + kBK + p.W - 1 < p.N ? r.beg + kBK + p.W - 1 : p.N;
  r.ntok = end - r.beg;
  r.nitems = (int)((r.ntok + p.tpi - 1) / p.tpi);
  return r;
}
// query-list entry at position pos of a task (selected mode; loaded ahead of use)
template <int SL>
__device__ __forceinline__ int32_t entry_at(const Params& p, const TaskRows& tr, int64_t pos) {
  return (SL != 0 || pos >= tr.ntok) ? 0 : __ldg(p.qlist + tr.kh * p.N * p.T + tr.beg + pos);
}
// token and slot of list position pos of a task (ent = entry_at(pos))
template <int SL>
__device__ __forceinline__ void token_of(const Params& p, const TaskRows& tr, int64_t pos,
                                         int32_t ent, int64_t& t, int64_t& slot) {
  if (SL == 0) {
    t = p.fdT.div((uint32_t)ent);
    slot = ent - t * p.T;
  } else if (SL == 2) {
    t = tr.beg + pos;
    slot = 0;
  } else {
    t = tr.beg + pos;
    const int64_t first = (t - p.W + 1 > 0 ? t - p.W + 1 : 0) / kBK;
    slot = tr.i - first;
  }
}

// FIFO of non-empty tasks handed from the MMA thread's look-ahead iterator
struct TaskFifo {
  TaskRows task[4];
  int head = 0, tail = 0;
  __device__ void push(const TaskRows& t) { task[tail++ & 3] = t; }
  __device__ TaskRows pop() { return task[head++ & 3]; }
};

// kMode: 0 selected (gathered rows, dq partials), 1 sliding window, 2 compressed
// (compile-time: each mode carries only its own code -- instruction-cache footprint)
template <int SL>
__global__ void __launch_bounds__(threads_of<SL>(), 1) tc_sel_bwd_kernel(const __grid_constant__ Params p) {
  constexpr int kLoaders = 32 * loader_warps<SL>();  // loader threads
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int k) { return sb + kOffBar + 8u * (uint32_t)k; };
  Ring ring{bar(B_RF), bar(B_RE), reinterpret_cast<volatile TaskSlot*>(smem + kOffRing)};
  auto decode = [&](int32_t t, TaskSlot& ts) {
    const TaskRows r = rows_of<SL>(p, t);
    ts.kh = (int32_t)r.kh;
    ts.i = (int32_t)r.i;
    ts.beg = (int32_t)r.beg;
    ts.ntok = (int32_t)r.ntok;
  };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool ACC = SL == 1 && p.accumulate;  // dK/dV += (only the sliding mode reads them back)

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(B_QDF + s), kLoaders);
      mbar_init(bar(B_QDE + s), 1);
      mbar_init(bar(B_DE + s), 1);
      mbar_init(bar(B_PDF + s), 128);
    }
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(bar(B_SDF + s), 1);
      mbar_init(bar(B_SDE + s), 128);
      mbar_init(bar(B_DQF + s), 1);
    }
    mbar_init(bar(B_KVF), kLoaders);
    mbar_init(bar(B_KVE), 1);
    mbar_init(bar(B_KAF), 1);
    mbar_init(bar(B_KAE), 128);
    for (int k = 0; k < kRingDepth; ++k) {
      mbar_init(bar(B_RF + k), 1);
      mbar_init(bar(B_RE + k), 8 + kLoaders + 1);  // 8 softmax warps + loader threads + MMA warp
    }
    fence_mbar_init();
  }
  if (SL != 0) {
    // TMA boxes fill g * tpi rows of a Q / dO tile; zero the rest once (they
    // carry P = dS = 0, but stale shared memory may hold NaN patterns and
    // 0 * NaN would poison the dK / dV row sums)
    const int used = (int)(p.g * p.tpi);
    for (int e = threadIdx.x; e < 2 * 2 * 2 * (kRows - used) * 8; e += (int)blockDim.x) {
      const int c = e & 7, rr = used + (e >> 3) % (kRows - used), t = (e >> 3) / (kRows - used);
      const uint32_t base = (t & 4 ? kOffDO : kOffQ) + (uint32_t)((t >> 1) & 1) * kTile + (uint32_t)(t & 1) * 16384u;
      *reinterpret_cast<uint4*>(smem + base + rr * 128u + c * 16u) = make_uint4(0u, 0u, 0u, 0u);
    }
    fence_proxy_async();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8 && warp < 8 + loader_warps<SL>()) {
    // ================================================================ loaders
    const int lr = threadIdx.x - 256;
    const int kt = lr / (int)p.g, hh = lr % (int)p.g;
    int64_t n = 0, kseq = 0;
    // The newest gather stays in flight (unpublished) while the next one is
    // issued; any wait that could block first publishes it.
    uint32_t pend = 0;      // QDF barrier of the in-flight Q/dO gather
    int64_t pend_n = 0;     // (trace) its item
    auto publish = [&]() {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      fence_proxy_async();
      if (pend) {
        mbar_arrive(pend);
        if (lr == 0) K8_TRACE(pend_n, 14);  // gather landed (published)
      }
      pend = 0;
    };
    if (SL != 0) {
      // Sliding mode: an item's rows are TPI consecutive tokens x g heads and
      // the task's keys 64 consecutive rows -> TMA boxes (one lane issues,
      // the other loader threads just arrive).
      const uint32_t box = 64u * (uint32_t)(p.g * p.tpi) * 2u;
      for (int k = 0;; ++k) {
        if (lr == 0) ring.produce(k, p.counter, p.ntask, decode);
        const TaskSlot ts = ring.consume(k);
        if (ts.task < 0) break;
        const TaskRows tr = rows_of_slot(ts, p.tpi);
        if (tr.nitems == 0) continue;
        mbar_spin(bar(B_KVE), (uint32_t)((kseq & 1) ^ 1));
        if (lr == 0) {
          mbar_arrive_expect_tx(bar(B_KVF), 32768u);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            tma_load_3d(sb + kOffK + hf * 8192u, &p.tmK, hf * 64, (int)tr.kh, (int)(tr.i * kBK), bar(B_KVF));
            tma_load_3d(sb + kOffV + hf * 8192u, &p.tmV, hf * 64, (int)tr.kh, (int)(tr.i * kBK), bar(B_KVF));
          }
        } else {
          mbar_arrive(bar(B_KVF));
        }
        for (int c = 0; c < tr.nitems; ++c, ++n) {
          const int s = (int)(n & 1);
          mbar_spin(bar(B_QDE + s), (uint32_t)(((n >> 1) & 1) ^ 1));
          if (lr == 0) {
            const int t0 = (int)(tr.beg + (int64_t)c * p.tpi);
            mbar_arrive_expect_tx(bar(B_QDF + s), 4u * box);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              tma_load_3d(sb + kOffQ + s * kTile + hf * 16384u, &p.tmQ, hf * 64, (int)(tr.kh * p.g), t0, bar(B_QDF + s));
              tma_load_3d(sb + kOffDO + s * kTile + hf * 16384u, &p.tmO, hf * 64, (int)(tr.kh * p.g), t0, bar(B_QDF + s));
            }
          } else {
            mbar_arrive(bar(B_QDF + s));
          }
        }
        ++kseq;
      }
    } else
    for (int k = 0;; ++k) {
      publish();  // nothing in flight across the task ring
      if (lr == 0) ring.produce(k, p.counter, p.ntask, decode);
      const TaskSlot ts = ring.consume(k);
      if (ts.task < 0) break;
      const TaskRows tr = rows_of_slot(ts, p.tpi);
      if (tr.nitems == 0) continue;
      mbar_spin(bar(B_KVE), (uint32_t)((kseq & 1) ^ 1));
      // K_i / V_i: the block's 64 contiguous key rows of this kv head, one 3-D
      // TMA box per 64-column half (loaded once per task, FSA's amortisation)
      if (lr == 0) {
        mbar_arrive_expect_tx(bar(B_KVF), 32768u);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          tma_load_3d(sb + kOffK + hf * 8192u, &p.tmK, hf * 64, (int)tr.kh, (int)(tr.i * kBK), bar(B_KVF));
          tma_load_3d(sb + kOffV + hf * 8192u, &p.tmV, hf * 64, (int)tr.kh, (int)(tr.i * kBK), bar(B_KVF));
        }
      } else {
        mbar_arrive(bar(B_KVF));
      }
      int32_t ent_next = kt < p.tpi ? entry_at<SL>(p, tr, kt) : 0;
      for (int c = 0; c < tr.nitems; ++c, ++n) {
        const int s = (int)(n & 1);
        const int64_t pos = (int64_t)c * p.tpi + kt;
        const bool ok = kt < p.tpi && pos < tr.ntok;
        const int32_t ent = ent_next;
        ent_next = kt < p.tpi ? entry_at<SL>(p, tr, pos + p.tpi) : 0;
        const uint32_t par = (uint32_t)(((n >> 1) & 1) ^ 1);
        int64_t row = 0;
        if (ok) {
          int64_t t, slot;
          token_of<SL>(p, tr, pos, ent, t, slot);
          row = t * p.h + tr.kh * p.g + hh;
        }
        if (lr == 0) K8_TRACE(n, 15);  // loader ready for this item (before the stage waits)
        // the dO half of the stage frees first (after the dV product): gather it
        // while the dK / dQ products still read Q
        if (!mbar_test(bar(B_DE + s), par)) {
          publish();
          mbar_spin(bar(B_DE + s), par);
        }
        warp_gather_rows32(sb + kOffDO + s * kTile, 16384u, lr & ~31, p.dO + row * kD, ok, lane);
        if (!mbar_test(bar(B_QDE + s), par)) {
          publish();
          mbar_spin(bar(B_QDE + s), par);
        }
        warp_gather_rows32(sb + kOffQ + s * kTile, 16384u, lr & ~31, p.Q + row * kD, ok, lane);
        asm volatile("cp.async.commit_group;" ::: "memory");
        // everything but this gather has landed: publish the previous one
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        fence_proxy_async();
        if (pend) {
          mbar_arrive(pend);
          if (lr == 0) K8_TRACE(pend_n, 14);  // gather landed (published)
        }
        pend = bar(B_QDF + s);
        pend_n = n;
        if (lr == 0) K8_TRACE(n, 0);  // gather issued
        {  // L2 prefetch of the next item's rows: its gather waits for a free stage
           // (-2 % at 128K where the rows miss L2; neutral at 32K)
          const int64_t pos1 = pos + p.tpi;
          if (kt < p.tpi && pos1 < tr.ntok) {
            int64_t t1, slot1;
            token_of<SL>(p, tr, pos1, ent_next, t1, slot1);
            const int64_t row1 = t1 * p.h + tr.kh * p.g + hh;
            prefetch_l2(p.Q + row1 * kD);
            prefetch_l2(p.Q + row1 * kD + 64);
            prefetch_l2(p.dO + row1 * kD);
            prefetch_l2(p.dO + row1 * kD + 64);
          }
        }
      }
      ++kseq;
    }
    publish();
  } else if (warp == 8 + loader_warps<SL>()) {
    // ================================================================ MMA issuer
    // Two independent in-order streams, polled without blocking:
    //   S stream : S/dP of item m (needs its Q/dO gather, the task's K/V, and
    //              a free S/dP TMEM stage -- at most 2 items ahead of P);
    //   P stream : products of item m (needs the softmax's P/dS of item m).
    // Products never wait for the next item's gather, so a stage is released
    // (and its next gather started) as soon as the softmax is done with it.
    // The whole warp runs the (warp-uniform) state machine so descriptors live
    // in uniform registers; one elected lane issues each MMA / commit.
    {
      const uint32_t tK = tmem + kColDK, tV = tmem + kColDV;
      TaskFifo fifo;
      int ka = 0, a_c = 0, a_n = 0;  // ring index, item in task, items in task
      int a_kseq = -1, ns = 0;       // K/V sequence of the S stream, next S item
      bool a_done = false;
      TaskRows b_tr{};
      int b_c = 0;
      int kseq_b = -1, np = 0;       // next products item
      long long idle_since = 0;
      for (;;) {
        bool progressed = false;
        auto s_stream = [&]() {
        if (!a_done && ns < np + 2) {
          bool have = a_c < a_n;
          while (!have) {
            TaskSlot t;
            if (!ring.try_consume_warp(ka, t)) break;
            ++ka;
            if (t.task < 0) {
              a_done = true;
              break;
            }
            const TaskRows tr = rows_of_slot(t, p.tpi);
            if (tr.nitems == 0) continue;
            a_c = 0;
            a_n = tr.nitems;
            ++a_kseq;
            fifo.push(tr);
            have = true;
          }
          if (have) {
            const int s = ns & 1, tm = ns % kTStages;
            if (mbar_test_warp(bar(B_KVF), (uint32_t)(a_kseq & 1)) &&
                mbar_test_warp(bar(B_QDF + s), (uint32_t)((ns >> 1) & 1)) &&
                mbar_test_warp(bar(B_SDE + tm), (uint32_t)(((ns / kTStages) & 1) ^ 1))) {
              tc_fence_after();
              const uint32_t q = sb + kOffQ + s * kTile, o = sb + kOffDO + s * kTile;
              const uint32_t tS = tmem + 128u * (uint32_t)tm;
              if (elect_one()) {
                K8_TRACE(ns, 12);  // S/dP issue starts
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  const uint32_t ko = (k >> 2) * 16384u + (k & 3) * 32u, kk = (k >> 2) * 8192u + (k & 3) * 32u;
                  mma_bf16(tS, desc_kmajor(q + ko), desc_kmajor(sb + kOffK + kk), kIdS, k > 0);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  const uint32_t ko = (k >> 2) * 16384u + (k & 3) * 32u, kk = (k >> 2) * 8192u + (k & 3) * 32u;
                  mma_bf16(tS + 64, desc_kmajor(o + ko), desc_kmajor(sb + kOffV + kk), kIdS, k > 0);
                }
                mma_commit(bar(B_SDF + tm));
                K8_TRACE(ns, 1);  // S/dP issued
              }
              __syncwarp();
#ifdef FSA_TRACE
              if (p.trace && blockIdx.x == 0 && ns < 256 && (p.trace[255 * 16 + 15] & 1)) {
                // debug probe: raw S/dP completion latency (serialises the issuer)
                if (lane == 0) {
                  while (!mbar_test(bar(B_SDF + tm), (uint32_t)((ns / kTStages) & 1))) {}
                  K8_TRACE(ns, 13);
                }
                __syncwarp();
              }
#endif
              ++a_c;
              ++ns;
              progressed = true;
            }
          }
        }
        };
        auto p_stream = [&]() {
        if (np < ns) {
          const bool first = np == 0 || b_c + 1 >= b_tr.nitems;
          const int s = np & 1, tm = np % kTStages;
          const bool ready = mbar_test_warp(bar(B_PDF + s), (uint32_t)((np >> 1) & 1)) &&
                             (!first || mbar_test_warp(bar(B_KAE), (uint32_t)(((kseq_b + 1) & 1) ^ 1)));
          if (ready) {
            if (first) {
              b_tr = fifo.pop();
              b_c = 0;
              ++kseq_b;
            } else {
              ++b_c;
            }
            const bool last = b_c + 1 == b_tr.nitems;
            tc_fence_after();
            const uint32_t q = sb + kOffQ + s * kTile, o = sb + kOffDO + s * kTile;
            const uint32_t pp = sb + kOffP + s * 16384u, ds = sb + kOffDS + s * 16384u;
            if (elect_one()) {
              K8_TRACE(np, 8);  // products ready (seen by the MMA warp)
#pragma unroll
              for (int k = 0; k < 8; ++k)
                mma_bf16(tV, desc_mnmajor(o + k * 2048u, 16384u), desc_mnmajor(pp + k * 2048u, 8192u),
                         kIdKV, (first && k == 0) ? 0u : 1u);
              if constexpr (SL == 0) mma_commit(bar(B_DE + s));  // dO read: its half of the stage is free
#pragma unroll
              for (int k = 0; k < 8; ++k)
                mma_bf16(tK, desc_mnmajor(q + k * 2048u, 16384u), desc_mnmajor(ds + k * 2048u, 8192u),
                         kIdKV, (first && k == 0) ? 0u : 1u);
              if (SL == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_bf16(tmem + 128u * (uint32_t)tm, desc_kmajor(ds + k * 32u),
                           desc_mnmajor(sb + kOffK + k * 2048u, 8192u), kIdQ, k > 0);
              }
              mma_commit(bar(B_DQF + tm));
              K8_TRACE(np, 4);  // products issued
              mma_commit(bar(B_QDE + s));
              if (last) {
                mma_commit(bar(B_KAF));
                mma_commit(bar(B_KVE));
              }
            }
            __syncwarp();
            ++np;
            progressed = true;
          }
        }
        };
        // products first: they free the item's Q/dO stage, the scarce resource
        // (2 stages); S/dP first measured 3.5-6 % slower
        p_stream();
        s_stream();
        if (a_done && np == ns) break;
        // watchdog: trap instead of hanging if neither stream can move for seconds
        // (polling hot or with a 16 ns nap measured the same as 64 ns)
        if (progressed) {
          idle_since = 0;
        } else if (idle_since == 0) {
          __nanosleep(64);  // yield issue slots to the softmax warps sharing this SMSP
          idle_since = clock64();
        } else if (__nanosleep(64), clock64() - idle_since > (1ll << 34)) {
          mbar_stuck(bar(B_SDF), 0);
        }
      }
    }
  } else {
    // ================================================================ softmax warpgroups
    const int wg = warp >> 2;
    const int r = threadIdx.x & 127;
    const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
    const int kt = r / (int)p.g, hh = r % (int)p.g;
    int64_t n = 0, kseq = 0;
    auto kv_epilogue = [&](const TaskRows& tr, int64_t ks) {
      mbar_spin_warp(bar(B_KAF), (uint32_t)(ks & 1));
      tc_fence_after();
      const int64_t slab = SL == 2 ? (tr.beg / p.CH) * p.cstride : 0;
      float* dk = p.dK + slab + ((tr.i * kBK) * p.h_K + tr.kh) * kD + r;
      float* dv = p.dV + slab + ((tr.i * kBK) * p.h_K + tr.kh) * kD + r;
      const int64_t ks_ = p.h_K * kD;  // key stride
      const float sv = p.sc.v[tr.kh], so = p.sc.o[tr.kh];
      const float mul_k = p.scale / (kDS16 * p.sc.q[tr.kh] * sv * so), mul_v = 1.f / (kP16 * so);
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // dK keys 16 at a time, then dV (register budget)
        float* dst = (q < 4 ? dk : dv) + (int64_t)(q & 3) * 16 * ks_;
        const float mul = q < 4 ? mul_k : mul_v;
        float v[16], old[16];
        if (ACC) {  // batch the 16 loads: one memory latency per chunk
#pragma unroll
          for (int c = 0; c < 16; ++c) old[c] = __ldcg(dst + c * ks_);
        }
        tmem_ld16(tmem + lb + (q < 4 ? kColDK : kColDV) + (q & 3) * 16, v);
        tmem_wait_ld();
        if (ACC) {
#pragma unroll
          for (int c = 0; c < 16; ++c) dst[c * ks_] = old[c] + v[c] * mul;
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c) dst[c * ks_] = v[c] * mul;
        }
      }
      tc_fence_before();
      mbar_arrive(bar(B_KAE));
    };
    for (int k = 0;; ++k) {
      const TaskSlot ts = ring.consume_warp(k);
      if (ts.task < 0) break;
      const TaskRows tr = rows_of_slot(ts, p.tpi);
      if (ACC && tr.nitems > 0) {
        // the block's dK/dV rows are read back (+=) at the end of the task:
        // pull them into L2 now (512 lines of 128 B over the 256 softmax threads)
        const int x = threadIdx.x;  // 0..255
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int line = x + 256 * h2, key = (line >> 2) & 63, part = line & 3;
          const float* base = (line < 256 ? p.dK : p.dV) + ((tr.i * kBK + key) * p.h_K + tr.kh) * kD;
          prefetch_l2(base + part * 32);
        }
      }
      if (tr.nitems == 0) {  // no attending rows: the block's gradients are zero
        if (ACC || wg != 0 || SL == 2) continue;  // (compressed: slab not read)
        float* dk = p.dK + ((tr.i * kBK) * p.h_K + tr.kh) * kD + r;
        float* dv = p.dV + ((tr.i * kBK) * p.h_K + tr.kh) * kD + r;
        for (int key = 0; key < kBK; ++key) {
          dk[key * p.h_K * kD] = 0.f;
          dv[key * p.h_K * kD] = 0.f;
        }
        continue;
      }
      // Per-row inputs of this warpgroup's items (every other item), loaded
      // ahead: the list entry two own items ahead, the token's lse / delta
      // (scattered [h][N] reads, mostly HBM misses) one own item ahead -- the
      // loads would otherwise sit between the S/dP landing and the softmax.
      const int c0 = (int)((wg - n) & 1);
      auto row_t = [&](int64_t pos, int32_t ent, int64_t& t, int64_t& slot) -> bool {
        if (kt >= p.tpi || pos >= tr.ntok) return false;
        token_of<SL>(p, tr, pos, ent, t, slot);
        return true;
      };
      auto stats_of = [&](int64_t pos, int32_t ent, float& lz, float& dz) {
        int64_t t, slot;
        lz = dz = 0.f;
        if (row_t(pos, ent, t, slot)) {
          const int64_t j = tr.kh * p.g + hh;
          lz = __ldg(p.lse + j * p.N + t);
          dz = __ldg(p.delta + j * p.N + t);
        }
      };
      // fp16 operand scales of this kv head: S16 = S s_Q s_K, dP16 = dP s_V s_dO
      const float sl2 = p.scale_log2 / (p.sc.q[tr.kh] * p.sc.k[tr.kh]);
      const float d16 = p.sc.v[tr.kh] * p.sc.o[tr.kh];
      const float mul_q = p.scale / (kDS16 * p.sc.k[tr.kh] * d16);  // dQ = scale dS K
      int32_t ent_a = kt < p.tpi ? entry_at<SL>(p, tr, (int64_t)c0 * p.tpi + kt) : 0;        // item c
      int32_t ent_b = kt < p.tpi ? entry_at<SL>(p, tr, (int64_t)(c0 + 2) * p.tpi + kt) : 0;  // item c + 2
      float lse_a, dl_a;
      stats_of((int64_t)c0 * p.tpi + kt, ent_a, lse_a, dl_a);
      for (int c = 0; c < tr.nitems; ++c, ++n) {
        if ((int)(n & 1) != wg) continue;
        const int s = (int)(n & 1);
        const int64_t pos = (int64_t)c * p.tpi + kt;
        const int32_t ent = ent_a;
        const float lse_raw = lse_a, dl = dl_a;
        int klo = 0, khi = -1;  // visible keys of the block: [klo, khi]
        int64_t drow = -1;
        int64_t t, slot;
        const bool ok = row_t(pos, ent, t, slot);
        if (ok) {
          drow = ((tr.kh * p.g + hh) * p.N + t) * p.T + slot;
          // compressed mode: pooled row j is formed for t iff j < (t + 1) / B_K
          const int64_t hi = (SL == 2 ? (t + 1) / p.cmpBK - 1 : t) - tr.i * kBK;
          khi = hi < kBK - 1 ? (int)hi : kBK - 1;
          if (SL == 1) {
            const int64_t lo = t - p.W + 1 - tr.i * kBK;
            klo = lo > 0 ? (int)lo : 0;
          }
        }
        const float lse_r = lse_raw * 1.4426950408889634f;
        const float dl16 = dl * d16;
        const bool full = __all_sync(0xffffffffu, klo == 0 && khi == kBK - 1);
        const int tm = (int)(n % kTStages);
        const uint32_t tpar = (uint32_t)((n / kTStages) & 1);
        mbar_spin_warp(bar(B_SDF + tm), tpar);
        if (r == 0) K8_TRACE(n, 2);  // S/dP landed
        // next own item's loads go out now, ahead of this item's dq stores (a
        // load issued behind 32 KB of stores waits for the LSU queue to drain)
        stats_of(pos + 2 * p.tpi, ent_b, lse_a, dl_a);
        ent_a = ent_b;
        ent_b = kt < p.tpi ? entry_at<SL>(p, tr, pos + 4 * p.tpi) : 0;
        tc_fence_after();
        unsigned char* prow = smem + kOffP + s * 16384u;
        unsigned char* drw = smem + kOffDS + s * 16384u;
        if (SL == 0) {  // the previous own item's dq scatters have read these buffers
          if (lane < 16) bulk_wait_read();
          __syncwarp();
        }
        // P / dS in chunks of CW key columns: 16 in the selected mode (13 warps,
        // 128 registers), 32 in the window / compressed modes (10 warps)
        constexpr int CW = SL == 0 ? 16 : 32;
#pragma unroll
        for (int hf = 0; hf < 64 / CW; ++hf) {
          float sv[CW], dp[CW];
          if constexpr (CW == 16) {
            tmem_ld16(tmem + lb + 128u * tm + hf * 16, sv);
            tmem_ld16(tmem + lb + 128u * tm + 64 + hf * 16, dp);
          } else {
            tmem_ld32(tmem + lb + 128u * tm + hf * 32, sv);
            tmem_ld32(tmem + lb + 128u * tm + 64 + hf * 32, dp);
          }
          tmem_wait_ld();
          uint32_t pp[CW / 2], dd[CW / 2];
#pragma unroll
          for (int c2 = 0; c2 < CW; c2 += 2) {
            const int key = hf * CW + c2;
            float p0 = ex2(fmaf(sv[c2], sl2, -lse_r));
            float p1 = ex2(fmaf(sv[c2 + 1], sl2, -lse_r));
            if (!full) {
              p0 = (key >= klo && key <= khi) ? p0 : 0.f;
              p1 = (key + 1 >= klo && key + 1 <= khi) ? p1 : 0.f;
            }
            if (!ok) p0 = p1 = 0.f;
            pp[c2 >> 1] = pack_f16(p0 * kP16, p1 * kP16);
            dd[c2 >> 1] = pack_f16(p0 * ((dp[c2] - dl16) * kDS16), p1 * ((dp[c2 + 1] - dl16) * kDS16));
          }
#pragma unroll
          for (int c4 = 0; c4 < CW / 8; ++c4) {
            *reinterpret_cast<uint4*>(prow + sw128_off(r, hf * (CW / 8) + c4)) =
                make_uint4(pp[4 * c4], pp[4 * c4 + 1], pp[4 * c4 + 2], pp[4 * c4 + 3]);
            *reinterpret_cast<uint4*>(drw + sw128_off(r, hf * (CW / 8) + c4)) =
                make_uint4(dd[4 * c4], dd[4 * c4 + 1], dd[4 * c4 + 2], dd[4 * c4 + 3]);
          }
        }
        if (SL != 0) {  // S/dP consumed: the TMEM stage is free right away
          tc_fence_before();
          mbar_arrive(bar(B_SDE + tm));
        }
        fence_proxy_async();
        mbar_arrive(bar(B_PDF + s));
        if (lane == 0 && (warp & 3) < 3) K8_TRACE(n, 9 + (warp & 3));  // P/dS written by this warp
        if (r == 0) K8_TRACE(n, 3);  // P/dS written
        // products of this item landed -> dQ partial out of TMEM; stage the
        // bf16 rows in this wg's (now consumed) P buffer for coalesced stores
        mbar_spin_warp(bar(B_DQF + tm), tpar);
        if (r == 0) K8_TRACE(n, 5);  // products landed
        tc_fence_after();
        if constexpr (SL != 0) {
          if (c + 1 == tr.nitems) kv_epilogue(tr, kseq);
          continue;
        }
        // rows -> SW128 staging tile [2 halves][128 rows][128 B] in this wg's
        // consumed P (half 0) and dS (half 1) buffers, then 4-row
        // tile::scatter4 stores to the rows' dq partial slots (TMA: no LSU
        // queue, so the next item's loads are not stuck behind 32 KB of
        // stores).  fp16 with a
        // power-of-two scale per 32 columns (chunk max -> [2^14, 2^15)):
        // 11-bit rows at the bf16 rows' traffic, one pass over TMEM.
        uint32_t ex4 = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float v[32];
          tmem_ld32(tmem + lb + 128u * tm + q * 32, v);
          tmem_wait_ld();
          float amax = 0.f;
#pragma unroll
          for (int c = 0; c < 32; ++c) amax = fmaxf(amax, fabsf(v[c]));
          const int ex = f16_row_exp(amax * mul_q);
          const float mul = ldexpf(mul_q, ex);
          ex4 |= (uint32_t)(ex & 0xff) << (8 * q);
          unsigned char* half = q < 2 ? prow : drw;
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const uint4 u = make_uint4(pack_f16(v[8 * c4] * mul, v[8 * c4 + 1] * mul),
                                       pack_f16(v[8 * c4 + 2] * mul, v[8 * c4 + 3] * mul),
                                       pack_f16(v[8 * c4 + 4] * mul, v[8 * c4 + 5] * mul),
                                       pack_f16(v[8 * c4 + 6] * mul, v[8 * c4 + 7] * mul));
            *reinterpret_cast<uint4*>(half + sw128_off(r, (q & 1) * 4 + c4)) = u;
          }
        }
        if (drow >= 0) __stcs(p.dqe + drow, (int32_t)ex4);
        tc_fence_before();
        mbar_arrive(bar(B_SDE + tm));  // TMEM stage free for S/dP of item n+3
        if (r == 0) K8_TRACE(n, 6);  // dQ read out of TMEM
        fence_proxy_async();
        __syncwarp();
        {
          const int grp = lane & 7, hf = lane >> 3;  // lanes 0-15: 8 row groups x 2 halves
          int32_t rows[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int64_t d = __shfl_sync(0xffffffffu, drow, 4 * grp + i);
            rows[i] = d >= 0 ? (int32_t)d : INT32_MAX;  // out of the map: dropped
          }
          if (lane < 16) {
            tma_scatter4_hint(&p.tmDQ, hf * 64, rows,
                              smem_u32(hf ? drw : prow) + (uint32_t)(32 * (warp & 3) + 4 * grp) * 128u,
                              l2_evict_first());
            bulk_commit();
          }
        }
        if (r == 0) K8_TRACE(n, 7);  // dQ rows stored
        if (c + 1 == tr.nitems) kv_epilogue(tr, kseq);
      }
      ++kseq;
    }
  }

  if (warp < 8 && lane < 16) bulk_wait_all();  // dq scatters complete before exit
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

bool tc_bwd_supported(const fsa_shape& s, int dtype) { return tc_fwd_supported(s, dtype); }

namespace {
#ifdef FSA_TRACE
long long* g_trace = nullptr;
#else
constexpr long long* g_trace = nullptr;
#endif
Params make_params(const fsa_shape* s, const void* Q, const void* K, const void* V,
                   const void* dOut, const void* lse, const void* delta, void* dq_buf, void* dK,
                   void* dV, F16Scales sc) {
  Params p{};
  p.sc = sc;
  p.trace = g_trace;
  p.Q = (const __half*)Q;
  p.K = (const __half*)K;
  p.V = (const __half*)V;
  p.dO = (const __half*)dOut;
  p.lse = (const float*)lse;
  p.delta = (const float*)delta;
  p.dq = (__half*)dq_buf;
  p.dqe = dq_buf ? reinterpret_cast<int32_t*>(p.dq + s->h * s->N * s->T * kD) : nullptr;
  p.dK = (float*)dK;
  p.dV = (float*)dV;
  p.N = s->N;
  p.h = s->h;
  p.h_K = s->h_K;
  p.T = s->T;
  p.b = s->N / s->B_K;
  p.g = s->h / s->h_K;
  p.ntask = p.h_K * p.b;
  p.tpi = (int)(kRows / p.g);
  p.scale = (float)s->scale;
  p.scale_log2 = (float)(s->scale * 1.4426950408889634);
  p.fdT.init((uint32_t)s->T);
  return p;
}

int launch_bwd(Params& p, cudaStream_t st) {
  cudaMemsetAsync(p.counter, 0, sizeof(int32_t), st);
  static unsigned long long done[3] = {0, 0, 0};
  ensure_smem_attr(tc_sel_bwd_kernel<0>, (int)kSmemBytes, done[0]);
  ensure_smem_attr(tc_sel_bwd_kernel<1>, (int)kSmemBytes, done[1]);
  ensure_smem_attr(tc_sel_bwd_kernel<2>, (int)kSmemBytes, done[2]);
  if (p.slide == 1)
    tc_sel_bwd_kernel<1><<<num_sms(), threads_of<1>(), kSmemBytes, st>>>(p);
  else if (p.slide == 2)
    tc_sel_bwd_kernel<2><<<num_sms(), threads_of<2>(), kSmemBytes, st>>>(p);
  else
    tc_sel_bwd_kernel<0><<<num_sms(), threads_of<0>(), kSmemBytes, st>>>(p);
  FSA_LAUNCH_CHECK("tc_sel_bwd");
  return FSA_OK;
}

}  // namespace

int tc_sel_bwd(const fsa_shape* s, const void* Q, const void* K, const void* V, const void* dOut,
               const void* lse, const void* delta, const int32_t* offsets, const int32_t* qlist,
               const int32_t* work, void* dq_buf, int dqbuf_dtype, void* dK, void* dV,
               F16Scales sc, cudaStream_t st) {
  FSA_REQUIRE(work != nullptr, "tensor-core backward needs the inverse work buffer");
  FSA_REQUIRE(dqbuf_dtype == FSA_DT_F16R,
              "tensor-core backward writes fp16 dq partials with row exponents (FSA_DT_F16R)");
  Params p = make_params(s, Q, K, V, dOut, lse, delta, dq_buf, dK, dV, sc);
  p.offsets = offsets;
  p.qlist = qlist;
  p.counter = plan_view(*s, work).counter;
  int rc = make_tmap_rows(&p.tmDQ, dq_buf, s->h * s->N * s->T, 1);  // scatter4 dq rows
  if (!rc) rc = make_tmap_tokens(&p.tmK, K, s->N, s->h_K, 1, 64);  // K_i / V_i boxes
  if (!rc) rc = make_tmap_tokens(&p.tmV, V, s->N, s->h_K, 1, 64);
  if (rc) return rc;
  return launch_bwd(p, st);
}

size_t tc_slide_bwd_workspace_bytes(const fsa_shape* s) { return 256; }  // scheduler counter

// K11: dK/dV on the KV-block-outer FSA backward kernel over each block's
// window of tokens (no dQ there), then dQ query-outer (tc_slide_dq.cu).
int tc_slide_bwd(const fsa_shape* s, const void* Q, const void* K, const void* V,
                 const void* dOut, const void* lse, const void* delta, void* dQ, void* dK,
                 void* dV, void* workspace, int accumulate, F16Scales sc, cudaStream_t st) {
  const int64_t S = (s->W - 1) / kBK + 2;  // window slots of a token (for the row bookkeeping)
  Params p = make_params(s, Q, K, V, dOut, lse, delta, nullptr, dK, dV, sc);
  p.slide = 1;
  p.no_dq = 1;
  p.accumulate = accumulate != 0;  // dK/dV += (modes 1 and 2)
  p.W = s->W;
  p.T = S;
  p.fdT.init((uint32_t)S);
  p.counter = (int32_t*)workspace;
  int rc = make_tmap_tokens(&p.tmQ, Q, s->N, s->h, (int)p.g, p.tpi);
  if (!rc) rc = make_tmap_tokens(&p.tmO, dOut, s->N, s->h, (int)p.g, p.tpi);
  if (!rc) rc = make_tmap_tokens(&p.tmK, K, s->N, s->h_K, 1, 64);
  if (!rc) rc = make_tmap_tokens(&p.tmV, V, s->N, s->h_K, 1, 64);
  if (rc) return rc;
  rc = launch_bwd(p, st);
  if (rc) return rc;
  // mode 1: dQ +=; mode 2: dQ written (fp32)
  return tc_slide_dq(s, Q, K, V, dOut, lse, delta, dQ, accumulate == 1, sc, st);
}

// Compressed-branch dK_cmp / dV_cmp: the same kernel with
// 64 pooled rows as a task's keys and a chunk of CH tokens as its rows; each
// (kv head, pooled tile, chunk) task writes its own partial slab.  Kb / Vb are
// bf16 [b][h_K][128]; dKp / dVp hold nch slabs of nct * 64 * h_K * 128 floats.
int64_t cmp_chunk_tokens(const fsa_shape* s) {
  int64_t ch = 2048;
  while (s->N > 32 * ch) ch *= 2;  // at most 32 slabs
  return ch;
}

int tc_cmp_bwd_kv(const fsa_shape* s, const void* Q, const void* Kb, const void* Vb,
                  const void* dOut, const void* lse, const void* delta, void* dKp, void* dVp,
                  int32_t* counter, F16Scales sc, cudaStream_t st) {
  Params p = make_params(s, Q, Kb, Vb, dOut, lse, delta, nullptr, dKp, dVp, sc);
  p.slide = 2;
  p.no_dq = 1;
  p.accumulate = 0;
  p.cmpBK = s->B_K;
  p.CH = cmp_chunk_tokens(s);
  p.nct = (p.b + kBK - 1) / kBK;
  p.nch = (p.N + p.CH - 1) / p.CH;
  p.cstride = p.nct * kBK * p.h_K * kD;
  p.ntask = p.h_K * p.nct * p.nch;
  p.T = 1;
  p.fdT.init(1u);
  p.counter = counter;
  int rc = make_tmap_tokens(&p.tmQ, Q, s->N, s->h, (int)p.g, p.tpi);
  if (!rc) rc = make_tmap_tokens(&p.tmO, dOut, s->N, s->h, (int)p.g, p.tpi);
  if (!rc) rc = make_tmap_tokens(&p.tmK, Kb, p.b, s->h_K, 1, 64);
  if (!rc) rc = make_tmap_tokens(&p.tmV, Vb, p.b, s->h_K, 1, 64);
  if (rc) return rc;
  return launch_bwd(p, st);
}

}  // namespace fsa

#ifdef FSA_TRACE
// debug: record a per-item timeline of CTA 0 of the next tc_sel_bwd launches
extern "C" void fsa_debug_bwd_trace(void* device_buf) { fsa::g_trace = (long long*)device_buf; }
#endif
