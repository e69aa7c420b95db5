// FSA selected-attention forward on tcgen05 tensor cores (K5), bf16, d = 128,
// B_K = 64.  Replaces kv_major.py:152-204 / _core.pyx:49-94 for the
// BASELINE.json shapes, in the fused LOCAL mode: per gathered
// (token, head) row it writes O_i / l_i (fp16, in the V16 scale) and (m_i, l_i)
// for block i into the slot-indexed partial buffer that the merge kernel (K6)
// combines.  S = Q K^T runs in bf16; O = P V in fp16 against the scaled fp16
// copy of V (f16_stage.cu), so P is rounded to 11 bits instead of 8.
// Partial rows are item-major (common.cuh, work plan): item n of the plan owns
// rows [128 n, 128 n + 128), so each warp's 32 rows leave as two TMA tile
// stores of 32 x 128 B instead of 16 four-row scatters.
//
// Persistent, warp-specialised, one CTA per SM:
//   warps 0-7  two softmax + epilogue warpgroups ping-ponging over items, one
//              TMEM lane (= MMA row) per thread; P goes back to TMEM (the PV A
//              operand) and the partial rows leave by TMA tile::scatter4
//   warps 8-11 loaders: cp.async gather of an item's 128 query rows (TPI
//              tokens x g group heads); one item's gather stays in flight while
//              the next is issued (4 Q stages); K_i/V_i per task by 3-D TMA
//              boxes from one lane (2 stages)
//   warp  12   MMA issuer (one elected lane): S = Q K^T (M128 N64 K128, bf16)
//              and O = P V (M128 N128 K64, fp16) into TMEM, tcgen05.commit;
//              S of item n+1 is issued before PV of item n
// Tasks (kv head, block) are claimed dynamically in head-major order
// (tc_sched.cuh), so the gathered Q rows of the current kv group stay in L2.
#include "tc_plan.cuh"
#include "tc_sched.cuh"

namespace fsa {
namespace {

using namespace tc;

constexpr int kD = 128, kBK = 64, kRows = 128;
constexpr int kThreads = 13 * 32;  // 2 softmax warpgroups, 4 loader warps, 1 MMA warp
constexpr int kQStages = 4;

constexpr uint32_t kQBytes = kRows * kD * 2;     // 32768: [2 halves][128 rows][128 B]
constexpr uint32_t kKVBytes = 2 * kBK * kD * 2;  // 32768: K [2][64][128 B], V [2][64][128 B]
constexpr uint32_t kOffQ = 0;
constexpr uint32_t kOffKV = kOffQ + kQStages * kQBytes;
constexpr uint32_t kOffSt = kOffKV + 2 * kKVBytes;  // P lives in TMEM (A operand of PV)
// epilogue staging: per softmax warp one SW128 half tile (32 rows x 128 B), the
// source of its tile::scatter4 stores
constexpr uint32_t kOffBar = kOffSt + 8 * 4096;
enum { B_QF = 0, B_QE = 4, B_KVF = 8, B_KVE = 10, B_SF = 12, B_PF = 14, B_PE = 16,
       B_OF = 18, B_OE = 21, B_RF = 24, B_RE = 28, kNumBars = 32 };
constexpr uint32_t kOffRing = kOffBar + kNumBars * 8;
constexpr uint32_t kOffTmem = kOffRing + kRingBytes;
constexpr uint32_t kSmemBytes = kOffTmem + 16 + 1024;

// TMEM: S/P stages [2] at 0 / 64 (P, fp16 pairs, overwrites its S: the stage is
// free again once PV has read P), O stages [3] at 128 + 128 o.  Three O stages:
// PV of item n waits for the epilogue of item n - 3 (the other warpgroup's),
// not for the same warpgroup's n - 2 epilogue, which runs after softmax(n).
constexpr int kOStages = 3;
constexpr uint32_t kIdescS = idesc_bf16(128, 64, false, false);
constexpr uint32_t kIdescPV = idesc_f16(128, 128, false, true);  // P, V16 in fp16

#ifdef FSA_TRACE
#define K5_TRACE(item, slot)                                                          \
  do {                                                                                \
    if (p.trace && blockIdx.x == 0 && (item) < 256) p.trace[(item) * 8 + (slot)] = clock64(); \
  } while (0)
#else
#define K5_TRACE(item, slot) \
  do {                       \
  } while (0)
#endif

struct Params {
  CUtensorMap tmO;
  CUtensorMap tmK, tmV;  // the task's 64 key rows of K / V16 (3-D TMA boxes)
  long long* trace;  // debug timeline (CTA 0, trace build only)  // obuf rows [h N T][128] fp16 (tile::scatter4 stores)
  const __nv_bfloat16 *Q, *K;
  const __half* V;  // the scaled fp16 copy (fsa_v_to_f16)
  const int32_t *offsets, *qlist;
  PlanView plan;  // token-chunked tasks (common.cuh): item prefix, sub-lists
  int32_t* counter;
  __half* obuf;
  float* ml;
  // phase API (kv_major.py:105-204): STATS writes slot-indexed (m_i, l_i)
  // [h][N][T] into ml; GLOBAL writes exp(z - m_global) V_i rows, fp32
  // slot-indexed [h][N][T][128], into gbuf
  const float* mg;
  float* gbuf;
  const float* vscale;
  int N, h, h_K, T, b, g, ntask, tpi;
  FastDiv fdT;  // entry -> token (entries are t * T + slot)
  float scale_log2, scale;
};

// chunked task `task` of the work plan: its sub-list of block i's query list
__device__ __forceinline__ void plan_slot(const Params& p, int32_t task, TaskSlot& ts) {
  const int32_t ki = __ldg(p.plan.tki + task);
  ts.kh = ki / p.b;
  ts.i = ki - ts.kh * p.b;
  ts.beg = __ldg(p.plan.tbeg + task);
  ts.ntok = __ldg(p.plan.tn + task);
  ts.ibase = __ldg(p.plan.item + task);
}

// non-empty tasks handed from the MMA thread's S stream to its PV stream
struct TaskFifo {
  TaskRows task[4];
  int head = 0, tail = 0;
  __device__ void push(const TaskRows& t) { task[tail++ & 3] = t; }
  __device__ TaskRows pop() { return task[head++ & 3]; }
};

// MODE: FSA_FWD_LOCAL (the fused fast path), FSA_FWD_STATS (softmax statistics
// only: no PV), FSA_FWD_GLOBAL (rows against the given global row max)
template <int MODE>
__global__ void __launch_bounds__(kThreads, 1) tc_sel_fwd_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int k) { return sb + kOffBar + 8u * (uint32_t)k; };
  Ring ring{bar(B_RF), bar(B_RE), reinterpret_cast<volatile TaskSlot*>(smem + kOffRing)};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kQStages; ++s) {
      mbar_init(bar(B_QF + s), 128);
      mbar_init(bar(B_QE + s), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(B_KVF + s), 128);
      mbar_init(bar(B_KVE + s), 1);
      mbar_init(bar(B_SF + s), 1);
      mbar_init(bar(B_PF + s), 128);
      mbar_init(bar(B_PE + s), 1);
    }
    for (int s = 0; s < kOStages; ++s) {
      mbar_init(bar(B_OF + s), 1);
      mbar_init(bar(B_OE + s), 128);
    }
    for (int k = 0; k < kRingDepth; ++k) {
      mbar_init(bar(B_RF + k), 1);
      mbar_init(bar(B_RE + k), 385);  // 256 softmax + 128 loader + 1 MMA
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8 && warp < 12) {
    // ------------------------------------------------------------ loaders
    const int lr = threadIdx.x - 256;
    const int kt_row = lr / p.g, hh = lr % p.g;
    int n = 0, kseq = 0;
    int prev_stage = -1;
    for (int k = 0;; ++k) {
      if (lr == 0) ring.produce(k, p.counter, p.ntask, [&](int32_t t, TaskSlot& ts) { plan_slot(p, t, ts); });
      const TaskSlot ts = ring.consume(k);
      if (ts.task < 0) break;
      const TaskRows tr = rows_of_slot(ts, p.tpi);
      if (tr.nitems == 0) continue;
      const int kvs = kseq & 1;
      mbar_wait(bar(B_KVE + kvs), (uint32_t)(((kseq >> 1) & 1) ^ 1));
      // K_i / V_i: the block's 64 contiguous key rows of this kv head, one 3-D
      // TMA box per 64-column half (loaded once per task, FSA's amortisation)
      if (lr == 0) {
        const uint32_t kv = sb + kOffKV + kvs * kKVBytes;
        mbar_arrive_expect_tx(bar(B_KVF + kvs), MODE == FSA_FWD_STATS ? 16384u : 32768u);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          tma_load_3d(kv + hf * 8192u, &p.tmK, hf * 64, (int)tr.kh, (int)(tr.i * kBK), bar(B_KVF + kvs));
          if (MODE != FSA_FWD_STATS)  // STATS: no values
            tma_load_3d(kv + 16384u + hf * 8192u, &p.tmV, hf * 64, (int)tr.kh, (int)(tr.i * kBK), bar(B_KVF + kvs));
        }
      } else {
        mbar_arrive(bar(B_KVF + kvs));
      }
      const int32_t* ql = p.qlist + (int64_t)tr.kh * p.N * p.T + tr.beg;
      // the query-list entry of the next item is loaded one item ahead, so its
      // latency hides behind the current item's stage wait and gather
      int ent_next = (kt_row < p.tpi && kt_row < tr.ntok) ? __ldg(ql + kt_row) : 0;
      for (int c = 0; c < tr.nitems; ++c, ++n) {
        const int s = n % kQStages;
        const int pos = c * p.tpi + kt_row;
        const bool ok = kt_row < p.tpi && pos < tr.ntok;
        const int ent = ent_next;
        const int pos1 = pos + p.tpi;
        ent_next = (kt_row < p.tpi && pos1 < tr.ntok) ? __ldg(ql + pos1) : 0;
        mbar_wait(bar(B_QE + s), (uint32_t)(((n / kQStages) & 1) ^ 1));
        const int t = ok ? (int)p.fdT.div((uint32_t)ent) : 0;
        warp_gather_rows32(sb + kOffQ + s * kQBytes, 16384u, lr & ~31,
                           p.Q + (t * p.h + (int)tr.kh * p.g + hh) * kD, ok, lane);
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (lr == 0) K5_TRACE(n, 0);  // gather issued
        // everything but this item's gather has landed: publish it
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        fence_proxy_async();
        if (prev_stage >= 0) mbar_arrive(bar(B_QF + prev_stage));
        prev_stage = s;
      }
      // publish the in-flight item before any wait that depends on consumers
      // (next task's K/V stage, task ring): the MMA's look-ahead needs it
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      fence_proxy_async();
      mbar_arrive(bar(B_QF + prev_stage));
      prev_stage = -1;
      ++kseq;
    }
  } else if (warp == 12) {
    // ------------------------------------------------------------ MMA issuer
    // Two in-order streams polled without blocking (as in tc_sel_bwd.cu):
    // S = Q K^T of item m needs its gather, the task's K/V stage and a free S
    // TMEM stage; O = P V of item m needs the softmax's P.  PV never waits for
    // the next item's gather.
    {  // whole warp: uniform state; one elected lane issues
      const uint32_t tS = tmem, tO = tmem + 128;
      TaskFifo fifo;
      int ka = 0, a_c = 0, a_n = 0, a_kseq = -1, ns = 0;
      bool a_done = false;
      TaskRows b_tr{};
      int b_c = 0, b_kseq = -1, np = 0;
      long long idle_since = 0;
      for (;;) {
        bool progressed = false;
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
            const int s = ns % kQStages, v = ns & 1, kvs = a_kseq & 1;
            if (mbar_test_warp(bar(B_KVF + kvs), (uint32_t)((a_kseq >> 1) & 1)) &&
                mbar_test_warp(bar(B_QF + s), (uint32_t)((ns / kQStages) & 1)) &&
                mbar_test_warp(bar(B_PE + v), (uint32_t)(((ns >> 1) & 1) ^ 1))) {
              tc_fence_after();
              const uint32_t qa = sb + kOffQ + s * kQBytes;
              const uint32_t ka_ = sb + kOffKV + kvs * kKVBytes;
              if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                  mma_bf16(tS + v * 64, desc_kmajor(qa + (k >> 2) * 16384u + (k & 3) * 32u),
                           desc_kmajor(ka_ + (k >> 2) * 8192u + (k & 3) * 32u), kIdescS, k > 0);
                mma_commit(bar(B_SF + v));
                mma_commit(bar(B_QE + s));
                K5_TRACE(ns, 1);  // S issued
              }
              __syncwarp();
              ++a_c;
              ++ns;
              progressed = true;
            }
          }
        }
        if (np < ns) {
          const int v = np & 1;
          const int o = np % kOStages;
          if (mbar_test_warp(bar(B_PF + v), (uint32_t)((np >> 1) & 1)) &&
              (MODE == FSA_FWD_STATS ||
               mbar_test_warp(bar(B_OE + o), (uint32_t)(((np / kOStages) & 1) ^ 1)))) {
            if (np == 0 || b_c + 1 >= b_tr.nitems) {
              b_tr = fifo.pop();
              b_c = 0;
              ++b_kseq;
            } else {
              ++b_c;
            }
            const bool last = b_c + 1 == b_tr.nitems;
            const int kvs = b_kseq & 1;
            tc_fence_after();
            const uint32_t va = sb + kOffKV + kvs * kKVBytes + 16384u;
            if (elect_one()) {
              if constexpr (MODE != FSA_FWD_STATS) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_bf16_ts(tO + o * 128, tS + v * 64 + k * 8,
                              desc_mnmajor(va + k * 2048u, 8192u), kIdescPV, k > 0);
                mma_commit(bar(B_OF + o));
              }
              mma_commit(bar(B_PE + v));  // (STATS: the S stage, read by the softmax)
              K5_TRACE(np, 4);  // PV issued
              if (last) mma_commit(bar(B_KVE + kvs));
            }
            __syncwarp();
            ++np;
            progressed = true;
          }
        }
        if (a_done && np == ns) break;
        if (progressed) {
          idle_since = 0;
        } else if (idle_since == 0) {
          __nanosleep(64);  // yield issue slots to the softmax warps sharing this SMSP
          idle_since = clock64();
        } else if (__nanosleep(64), clock64() - idle_since > (1ll << 34)) {
          mbar_stuck(bar(B_SF), 0);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    // Two warpgroups ping-pong over items (wg handles items n with n % 2 == wg):
    // each SM sub-partition runs two softmax warps, so one's TMEM loads,
    // exponentials and stores overlap the other's.
    const int wg = warp >> 2;
    const int r = threadIdx.x & 127;  // MMA row == TMEM lane
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    unsigned char* st = smem + kOffSt + warp * 4096u;
    const int kt_row = r / p.g, hh = r % p.g;
    int64_t prow = -1;  // obuf row of this thread's row in the pending item
    int pitem = 0;      // the pending item's index in the plan
    float pm = 0.f, pl = 1.f;
    bool pend = false;
    int pend_n = 0;
    int n = 0;
    auto epilogue = [&](int m1) {
      const int o1 = m1 % kOStages;
      mbar_wait(bar(B_OF + o1), (uint32_t)((m1 / kOStages) & 1));
      if (r == 0) K5_TRACE(m1, 5);  // O landed (epilogue)
      tc_fence_after();
      if constexpr (MODE == FSA_FWD_GLOBAL) {
        // unnormalised rows exp(z - m) V_i (kv_major.py:194-196), fp32, slot-indexed
        float* dst = prow >= 0 ? p.gbuf + prow * kD : nullptr;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float ov[32];
          tmem_ld32(tmem + lane_base + 128 + o1 * 128 + q * 32, ov);
          tmem_wait_ld();
          if (dst) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
              reinterpret_cast<float4*>(dst + q * 32)[c] =
                  make_float4(ov[4 * c] * pl, ov[4 * c + 1] * pl, ov[4 * c + 2] * pl, ov[4 * c + 3] * pl);
          }
        }
        tc_fence_before();
        mbar_arrive(bar(B_OE + o1));
        return;
      }
      const float inv = 1.f / pl;
      // The item's rows are contiguous: each warp's 32 rows leave by one TMA
      // tile store per 64-column half from its SW128 staging tile -- off the
      // LSU, which the loaders' gathers and the next item's entry loads share.
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        if (lane == 0) bulk_wait_read();  // the previous half's store has read the staging
        __syncwarp();
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const int q = 2 * hf + qq;
          float ov[32];
          tmem_ld32(tmem + lane_base + 128 + o1 * 128 + q * 32, ov);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 v4 = make_uint4(pack_f16(ov[8 * c] * inv, ov[8 * c + 1] * inv),
                                        pack_f16(ov[8 * c + 2] * inv, ov[8 * c + 3] * inv),
                                        pack_f16(ov[8 * c + 4] * inv, ov[8 * c + 5] * inv),
                                        pack_f16(ov[8 * c + 6] * inv, ov[8 * c + 7] * inv));
            *reinterpret_cast<uint4*>(st + sw128_off(lane, qq * 4 + c)) = v4;
          }
        }
        if (hf == 1) {
          tc_fence_before();
          mbar_arrive(bar(B_OE + o1));
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d_hint(&p.tmO, hf * 64, pitem * kRows + (warp & 3) * 32, smem_u32(st),
                            l2_evict_first());
          bulk_commit();
        }
      }
      __stcs(reinterpret_cast<float2*>(p.ml) + (int64_t)pitem * kRows + r, make_float2(pm, pl));
      if (r == 0) K5_TRACE(m1, 6);  // rows stored
    };
    for (int k = 0;; ++k) {
      const TaskSlot ts = ring.consume(k);
      if (ts.task < 0) break;
      const TaskRows tr = rows_of_slot(ts, p.tpi);
      const int32_t* ql = p.qlist + (int64_t)tr.kh * p.N * p.T + tr.beg;
      const int32_t ibase = ts.ibase;
      // entries of this warpgroup's items (every other item) are loaded one
      // own item ahead
      const int c0 = (int)((wg - n) & 1);
      int ent_next = (c0 < tr.nitems && kt_row < p.tpi && c0 * p.tpi + kt_row < tr.ntok)
                         ? __ldg(ql + c0 * p.tpi + kt_row) : 0;
      for (int c = 0; c < tr.nitems; ++c, ++n) {
        if ((n & 1) != wg) continue;
        const int s = n & 1;
        const int pos = c * p.tpi + kt_row;
        const int ent = ent_next;
        {
          const int pos2 = pos + 2 * p.tpi;
          ent_next = (kt_row < p.tpi && pos2 < tr.ntok) ? __ldg(ql + pos2) : 0;
        }
        int64_t orow = -1, grow = -1;  // item-major row; slot-indexed row (phase modes)
        float mgl = 0.f;                // GLOBAL: the row's global max (log2 units)
        int vis = kBK;
        if (kt_row < p.tpi && pos < tr.ntok) {
          const int t = (int)p.fdT.div((uint32_t)ent);
          orow = (int64_t)(ibase + c) * kRows + r;
          const int v = t - (int)tr.i * kBK + 1;
          vis = v < kBK ? v : kBK;
          if (MODE != FSA_FWD_LOCAL) {
            const int64_t j = (int64_t)tr.kh * p.g + hh;
            grow = (j * p.N + t) * p.T + (ent - t * p.T);
            if (MODE == FSA_FWD_GLOBAL) mgl = __ldg(p.mg + j * p.N + t) * 1.4426950408889634f;
          }
        }
        mbar_wait(bar(B_SF + s), (uint32_t)((n >> 1) & 1));
        if (r == 0) K5_TRACE(n, 2);  // S landed
        tc_fence_after();
        float sv[64];
        tmem_ld32(tmem + lane_base + s * 64, sv);
        tmem_ld32(tmem + lane_base + s * 64 + 32, sv + 32);
        tmem_wait_ld();
        // only rows whose token lies in block i see a causal prefix (vis < 64);
        // warps without such rows take the unmasked path
        const bool masked = __any_sync(0xffffffffu, vis < kBK);
        float mx = -INFINITY;
        float sum = 0.f, s2 = 0.f;
        uint32_t pk[32];
        if (MODE == FSA_FWD_GLOBAL) {  // P = exp(z - m_global) <= 1
#pragma unroll
          for (int c2 = 0; c2 < 64; c2 += 2) {
            const float e0 = c2 < vis && orow >= 0 ? ex2(fmaf(sv[c2], p.scale_log2, -mgl)) : 0.f;
            const float e1 = c2 + 1 < vis && orow >= 0 ? ex2(fmaf(sv[c2 + 1], p.scale_log2, -mgl)) : 0.f;
            pk[c2 >> 1] = pack_f16(e0, e1);
          }
        } else if (!masked) {
#pragma unroll
          for (int c2 = 0; c2 < 64; ++c2) mx = fmaxf(mx, sv[c2]);
          if (orow < 0) mx = 0.f;
          const float mb = mx * p.scale_log2;
#pragma unroll
          for (int c2 = 0; c2 < 64; c2 += 2) {
            const float e0 = ex2(fmaf(sv[c2], p.scale_log2, -mb));
            const float e1 = ex2(fmaf(sv[c2 + 1], p.scale_log2, -mb));
            sum += e0;
            s2 += e1;
            pk[c2 >> 1] = pack_f16(e0, e1);
          }
        } else {
#pragma unroll
          for (int c2 = 0; c2 < 64; ++c2) mx = fmaxf(mx, c2 < vis ? sv[c2] : -INFINITY);
          if (orow < 0) mx = 0.f;
          const float mb = mx * p.scale_log2;
#pragma unroll
          for (int c2 = 0; c2 < 64; c2 += 2) {
            const float e0 = c2 < vis ? ex2(fmaf(sv[c2], p.scale_log2, -mb)) : 0.f;
            const float e1 = c2 + 1 < vis ? ex2(fmaf(sv[c2 + 1], p.scale_log2, -mb)) : 0.f;
            sum += e0;
            s2 += e1;
            pk[c2 >> 1] = pack_f16(e0, e1);
          }
        }
        sum += s2;
        if constexpr (MODE == FSA_FWD_STATS) {  // local (m_i, l_i) only (kv_major.py:131-140)
          if (grow >= 0) reinterpret_cast<float2*>(p.ml)[grow] = make_float2(mx * p.scale, sum);
          tc_fence_before();
          mbar_arrive(bar(B_PF + s));
          continue;
        }
        tmem_st32u(tmem + lane_base + s * 64, pk);  // fp16 pairs, K-packed, over S
        tmem_wait_st_();
        tc_fence_before();
        mbar_arrive(bar(B_PF + s));
        if (r == 0) K5_TRACE(n, 3);  // P written
        if (pend) epilogue(pend_n);
        pend = true;
        pend_n = n;
        prow = MODE == FSA_FWD_GLOBAL ? grow : orow;
        pitem = ibase + c;
        pm = mx * p.scale;
        pl = MODE == FSA_FWD_GLOBAL ? 1.f / __ldg(p.vscale + tr.kh) : sum;
      }
    }
    if (pend) epilogue(pend_n);
  }

  if (warp < 8 && lane < 8) bulk_wait_all();  // partial-row scatters complete before exit
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

#ifdef FSA_TRACE
long long* g_k5_trace = nullptr;
#else
constexpr long long* g_k5_trace = nullptr;
#endif

int num_sms() {  // of the current device (a process may drive several)
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

bool tc_fwd_supported(const fsa_shape& s, int dtype) {
  return dtype == FSA_DT_BF16 && s.d_K == kD && s.d_V == kD && s.B_K == kBK && s.h_K > 0 &&
         s.h % s.h_K == 0 && s.h / s.h_K <= kRows && (int64_t)s.N * s.h < (1ll << 23);
}

int tc_sel_fwd(const fsa_shape* s, const void* Q, const void* K, const void* V,
               const int32_t* offsets, const int32_t* qlist, const int32_t* work, void* obuf,
               void* ml, cudaStream_t st, int mode, const float* m_global, const float* vscale) {
  FSA_REQUIRE(work != nullptr, "tensor-core forward needs the inverse work buffer");
  Params p{};
  p.Q = (const __nv_bfloat16*)Q;
  p.K = (const __nv_bfloat16*)K;
  p.V = (const __half*)V;
  p.offsets = offsets;
  p.qlist = qlist;
  p.plan = plan_view(*s, work);
  p.trace = g_k5_trace;
  p.obuf = mode == FSA_FWD_LOCAL ? (__half*)obuf : nullptr;
  p.gbuf = mode == FSA_FWD_GLOBAL ? (float*)obuf : nullptr;
  p.ml = (float*)ml;
  p.mg = m_global;
  p.vscale = vscale;
  p.N = (int)s->N;
  p.h = (int)s->h;
  p.h_K = (int)s->h_K;
  p.T = (int)s->T;
  p.b = (int)(s->N / s->B_K);
  p.g = (int)(s->h / s->h_K);
  p.ntask = (int)plan_ntask(*s);
  p.tpi = kRows / p.g;
  p.fdT.init((uint32_t)p.T);
  p.scale = (float)s->scale;
  p.scale_log2 = (float)(s->scale * 1.4426950408889634);
  p.counter = p.plan.counter;
  if (mode == FSA_FWD_LOCAL)
    if (int rc = make_tmap_rows(&p.tmO, obuf, plan_max_items(*s) * kRows, 32)) return rc;
  if (int rc = make_tmap_tokens(&p.tmK, K, s->N, s->h_K, 1, kBK)) return rc;  // K_i / V_i boxes
  if (mode != FSA_FWD_STATS)
    if (int rc = make_tmap_tokens(&p.tmV, V, s->N, s->h_K, 1, kBK)) return rc;
  cudaMemsetAsync(p.counter, 0, sizeof(int32_t), st);
  static unsigned long long done[3] = {0, 0, 0};
  if (mode == FSA_FWD_STATS) {
    ensure_smem_attr(tc_sel_fwd_kernel<FSA_FWD_STATS>, (int)kSmemBytes, done[1]);
    tc_sel_fwd_kernel<FSA_FWD_STATS><<<num_sms(), kThreads, kSmemBytes, st>>>(p);
  } else if (mode == FSA_FWD_GLOBAL) {
    FSA_REQUIRE(m_global && vscale, "sel_fwd GLOBAL: needs the global row max and the V scales");
    ensure_smem_attr(tc_sel_fwd_kernel<FSA_FWD_GLOBAL>, (int)kSmemBytes, done[2]);
    tc_sel_fwd_kernel<FSA_FWD_GLOBAL><<<num_sms(), kThreads, kSmemBytes, st>>>(p);
  } else {
    ensure_smem_attr(tc_sel_fwd_kernel<FSA_FWD_LOCAL>, (int)kSmemBytes, done[0]);
    tc_sel_fwd_kernel<FSA_FWD_LOCAL><<<num_sms(), kThreads, kSmemBytes, st>>>(p);
  }
  FSA_LAUNCH_CHECK("tc_sel_fwd");
  return FSA_OK;
}

}  // namespace fsa

#ifdef FSA_TRACE
// debug: record a per-item timeline of CTA 0 of the next tc_sel_fwd launches
extern "C" void fsa_debug_sel_fwd_trace(void* device_buf) { fsa::g_k5_trace = (long long*)device_buf; }
#endif
