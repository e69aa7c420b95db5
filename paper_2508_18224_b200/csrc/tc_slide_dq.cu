// Sliding-window dQ on tcgen05 tensor cores (part of K11), bf16, d = 128.
// The band-mask dense_backward of oracle.py:102-131 restricted to dQ:
//   P  = exp(S scale - lse),  dS = P * (dO V^T - delta),  dQ = scale * dS K
// computed query-outer, so every dQ row is produced by exactly one CTA and
// accumulated in TMEM over its window's key tiles: no per-slot partials, no
// reduction pass, deterministic.  (dK / dV come from the KV-block-outer FSA
// backward kernel in its sliding mode, tc_sel_bwd.cu, without its dQ.)
//
// Structure as the window forward (tc_qo_fwd.cu): a super item = 2 sub-items
// of TPI = 128/g tokens x g heads of one kv head sharing one stream of 64-key
// K/V tiles; softmax warpgroup w owns sub-item w.  Per tile:
//   S_w = Q_w K^T, dP_w = dO_w V^T      (2 x M128 N64 K128) -> TMEM of wg w
//   softmax: dS (fp16) written back over S in TMEM
//   dQ_w += dS K                        (M128 N128 K64, A = dS from TMEM)
// TMEM per wg (256 columns at 256 w): S +0, dP +64, dQ accumulator +128.
// Roles: warps 0-3 / 4-7 softmax + epilogue, warp 8 the TMA loader (one lane;
// 9-10 idle), 11 MMA issuer.
// fp16 operands (fsa_stage_f16_ops copies, as tc_sel_bwd.cu): S16 = S s_Q s_K,
// dP16 = dP s_V s_dO, dS16 = P (dP16 - delta s_V s_dO) 2^-23 (|dS16| <= 2^15),
// dQ = scale acc / (2^-23 s_K s_V s_dO).
#include "tc_plan.cuh"
#include "tc_sched.cuh"

namespace fsa {
namespace {

using namespace tc;

constexpr int kD = 128, kRows = 128;
constexpr int kThreads = 12 * 32;
constexpr uint32_t kT = 32768;                          // one 128-row tile [2 halves][128][128 B]
constexpr uint32_t kKV = 32768;                         // K | V tile of 64 keys
constexpr int kKVStages = 3;
constexpr uint32_t kOffQ = 0;                           // Q sub 0, Q sub 1, dO sub 0, dO sub 1
constexpr uint32_t kOffKV = 4 * kT;
constexpr uint32_t kOffBar = kOffKV + kKVStages * kKV;
enum { B_QF = 0, B_QE = 1, B_KF = 2, B_KE = 5, B_SF = 8, B_PF = 10, B_OF = 12, B_OE = 14,
       kNumBars = 16 };
constexpr uint32_t kOffTmem = kOffBar + kNumBars * 8;
constexpr uint32_t kSmemBytes = kOffTmem + 16 + 1024;
static_assert(kSmemBytes <= 232448, "shared memory budget");
constexpr uint32_t kIdS = idesc_f16(128, 64, false, false);
constexpr uint32_t kIdQ = idesc_f16(128, 128, false, true);
constexpr float kDS16 = 1.f / 8388608.f;  // dS16 = P (dP16 - delta16) 2^-23

struct Params {
  CUtensorMap tmQ, tmO, tmK, tmV;  // TMA descriptors (tma_host.cu): Q/dO boxes (64, g, tpi), K/V (64, 1, 64)
  CUtensorMap tmDQ;                 // dQ fp32 boxes (32, g, tpi): the epilogue's store / reduce-add
  long long* trace;  // debug timeline (CTA 0), null in production
  const __half *Q, *K, *V, *dO;  // fp16 staged copies
  F16Scales sc;
  const float *lse, *delta;
  float* dQ;  // [N][h][128]
  int64_t N, h, h_K, g, W, n_super;
  int tpi, accumulate;
  int cmp;         // compressed mode: keys = pooled rows of K_cmp / V_cmp (bf16), row j
  int64_t cmpBK;   // visible to token t iff j < (t + 1) / B_K (branches.py:47-78)
  float scale, scale_log2;
};

#ifdef FSA_TRACE
#define DQ_TRACE(w, item, slot)                                                          \
  do {                                                                                   \
    if (p.trace && blockIdx.x == 0 && (item) < 128)                                      \
      p.trace[((w) * 128 + (item)) * 8 + (slot)] = clock64();                            \
  } while (0)
#else
#define DQ_TRACE(w, item, slot) \
  do {                         \
  } while (0)
#endif

struct Sub {
  int t0, tlast;  // tokens [t0, tlast]
  int k0, k1;     // key tiles [k0, k1)
};
struct Super {
  int kh;
  Sub s[2];
  int u0, u1;
};

template <int CM>
__device__ __forceinline__ bool super_of(const Params& p, int id, Super& it) {
  if (id >= p.h_K * p.n_super) return false;
  it.kh = id % (int)p.h_K;
  const int st = CM ? (int)p.n_super - 1 - id / (int)p.h_K : id / (int)p.h_K;  // cmp: late (heavy) tokens first
  it.u0 = INT32_MAX;
  it.u1 = 0;
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    Sub& s = it.s[w];
    s.t0 = (2 * st + w) * p.tpi;
    s.tlast = min(s.t0 + p.tpi, (int)p.N) - 1;
    s.k0 = s.k1 = 0;
    if (s.tlast >= s.t0 && CM) {
      s.k1 = (int)(((s.tlast + 1) / p.cmpBK + 63) / 64);  // tiles of the formed pooled rows
      if (s.k1 > 0) {
        it.u0 = 0;
        it.u1 = max(it.u1, s.k1);
      }
    } else if (s.tlast >= s.t0) {
      s.k0 = (s.t0 - (int)p.W + 1 > 0 ? s.t0 - (int)p.W + 1 : 0) / 64;
      s.k1 = s.tlast / 64 + 1;
      it.u0 = min(it.u0, s.k0);
      it.u1 = max(it.u1, s.k1);
    }
  }
  if (it.u0 >= it.u1) it.u0 = it.u1 = 0;
  return true;
}

template <int CM>
struct Cursor {
  int n = -1, seq = -1, rbase = 0, rnext = 0;
  Super it;
  __device__ bool advance(const Params& p, int G) {
    for (;;) {
      ++n;
      if (!super_of<CM>(p, (int)blockIdx.x + n * G, it)) return false;
      if (it.u0 == it.u1) continue;
      ++seq;
      rbase = rnext;
      rnext += it.u1 - it.u0;
      return true;
    }
  }
};

// CM: compressed mode at compile time (per-mode code only)
template <int CM>
__global__ void __launch_bounds__(kThreads, 1) tc_slide_dq_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int k) { return sb + kOffBar + 8u * (uint32_t)k; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar(B_QF), 1);  // TMA: one arrive.expect_tx + the transaction bytes
    mbar_init(bar(B_QE), 2);  // one arrival per softmax warpgroup (epilogue staging read)
    for (int w = 0; w < 2; ++w) {
      mbar_init(bar(B_SF + w), 1);
      mbar_init(bar(B_PF + w), 128);
      mbar_init(bar(B_OF + w), 1);
      mbar_init(bar(B_OE + w), 128);
    }
    for (int s = 0; s < kKVStages; ++s) {
      mbar_init(bar(B_KF + s), 1);
      mbar_init(bar(B_KE + s), 1);  // one commit per union tile, after both streams
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int G = (int)gridDim.x;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA loader (one lane)
    // Q and dO of a sub-item are TPI consecutive tokens x the g heads of one kv
    // head: one 3-D box per 64-feature half lands as the SW128 K-major tile.
    if (lane == 0) {
      const uint32_t qbox = 64u * (uint32_t)(p.g * p.tpi) * 2u;  // bytes per half tile
      Cursor<CM> c;
      int r = 0;
      while (c.advance(p, G)) {
        mbar_spin(bar(B_QE), (uint32_t)((c.seq & 1) ^ 1));
        DQ_TRACE(0, c.seq, 4);  // loader: Q/dO stage free
        mbar_arrive_expect_tx(bar(B_QF), 8u * qbox);
#pragma unroll
        for (int w = 0; w < 2; ++w)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            tma_load_3d(sb + kOffQ + w * kT + hf * 16384u, &p.tmQ, hf * 64, c.it.kh * (int)p.g,
                        c.it.s[w].t0, bar(B_QF));
            tma_load_3d(sb + kOffQ + (2 + w) * kT + hf * 16384u, &p.tmO, hf * 64,
                        c.it.kh * (int)p.g, c.it.s[w].t0, bar(B_QF));
          }
        DQ_TRACE(0, c.seq, 5);  // loader: Q/dO loads issued
        for (int u = c.it.u0; u < c.it.u1; ++u, ++r) {
          const int v = r % kKVStages;
          mbar_spin(bar(B_KE + v), (uint32_t)(((r / kKVStages) & 1) ^ 1));
          mbar_arrive_expect_tx(bar(B_KF + v), kKV);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            tma_load_3d(sb + kOffKV + v * kKV + hf * 8192u, &p.tmK, hf * 64, c.it.kh, u * 64,
                        bar(B_KF + v));
            tma_load_3d(sb + kOffKV + v * kKV + 16384u + hf * 8192u, &p.tmV, hf * 64, c.it.kh,
                        u * 64, bar(B_KF + v));
          }
        }
      }
    }
  } else if (warp == 11) {
    // ------------------------------------------------------------ MMA issuer
    // Static order with blocking waits (one lane waits; one elected lane
    // issues).  Per union tile u of a super item and per sub-item w: first
    // dQ_w += dS K of tile u-1 (it frees wg w's single S/dP TMEM stage), then
    // S/dP_w of tile u.  KE: one commit per union tile after both streams;
    // QE: two arrivals per super item (the softmax warpgroups).
    {
      Cursor<CM> c;
      int ns[2] = {0, 0}, nd[2] = {0, 0}, nsub[2] = {0, 0};
      while (c.advance(p, G)) {
        const Super& it = c.it;
        bool q_ready = false;
        for (int u = it.u0; u <= it.u1; ++u) {
          const bool s_step = u < it.u1;
          const int rr = c.rbase + (u - it.u0), kv = rr % kKVStages;
          if (s_step) mbar_wait_warp(bar(B_KF + kv), (uint32_t)((rr / kKVStages) & 1));
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            const Sub& sw = it.s[w];
            if (u > it.u0) {  // ---- dQ of tile u-1
              const int up = u - 1, rp = rr - 1, kvp = rp % kKVStages;
              if (up >= sw.k0 && up < sw.k1) {
                const bool first = up == sw.k0, last = up + 1 == sw.k1;
                mbar_wait_warp(bar(B_PF + w), (uint32_t)(nd[w] & 1));
                if (first) mbar_wait_warp(bar(B_OE + w), (uint32_t)((nsub[w] & 1) ^ 1));
                tc_fence_after();
                const uint32_t k = sb + kOffKV + kvp * kKV;
                const uint32_t tS = tmem + 256u * w, tQ = tmem + 256u * w + 128u;
                if (elect_one()) {
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk)
                    mma_bf16_ts(tQ, tS + kk * 8, desc_mnmajor(k + kk * 2048u, 8192u), kIdQ,
                                (first && kk == 0) ? 0u : 1u);
                  DQ_TRACE(w, nd[w], 3);  // dQ issued
                  if (last) mma_commit(bar(B_OF + w));
                }
                __syncwarp();
                if (last) ++nsub[w];
                ++nd[w];
              }
              if (w == 1) {  // both streams' dQ of tile u-1 issued: free its K/V stage
                if (elect_one()) mma_commit(bar(B_KE + kvp));
                __syncwarp();
              }
            }
            if (s_step && u >= sw.k0 && u < sw.k1) {  // ---- S/dP of tile u
              if (!q_ready) {
                mbar_wait_warp(bar(B_QF), (uint32_t)(c.seq & 1));
                q_ready = true;
              }
              tc_fence_after();
              const uint32_t q = sb + kOffQ + w * kT, o = sb + kOffQ + (2 + w) * kT;
              const uint32_t k = sb + kOffKV + kv * kKV, vv = k + 16384u;
              const uint32_t tS = tmem + 256u * w;
              if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                  mma_bf16(tS, desc_kmajor(q + (kk >> 2) * 16384u + (kk & 3) * 32u),
                           desc_kmajor(k + (kk >> 2) * 8192u + (kk & 3) * 32u), kIdS, kk > 0);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                  mma_bf16(tS + 64, desc_kmajor(o + (kk >> 2) * 16384u + (kk & 3) * 32u),
                           desc_kmajor(vv + (kk >> 2) * 8192u + (kk & 3) * 32u), kIdS, kk > 0);
                mma_commit(bar(B_SF + w));
                DQ_TRACE(w, ns[w], 0);  // S/dP issued
              }
              __syncwarp();
              ++ns[w];
            }
          }
        }
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ softmax / epilogue
    const int w = warp >> 2;
    const int r = threadIdx.x & 127;
    const uint32_t lb = ((uint32_t)((warp & 3) * 32) << 16) + 256u * w;
    const int kt_row = r / (int)p.g, hh = r % (int)p.g;
    int u = 0, n_out = 0;
    Cursor<CM> c;
    while (c.advance(p, G)) {
      const Sub& s = c.it.s[w];
      if (s.k0 >= s.k1) {  // empty sub-item: nothing staged in this Q/dO stage
        if (r == 0) mbar_arrive(bar(B_QE));
        continue;
      }
      const int t = s.t0 + kt_row;
      const bool ok = kt_row < p.tpi && t <= s.tlast;
      const int64_t j = (int64_t)c.it.kh * p.g + hh;
      const int klo = CM ? 0 : (t - (int)p.W + 1 > 0 ? t - (int)p.W + 1 : 0);
      const int khi = !ok ? -1 : CM ? (int)((t + 1) / p.cmpBK) - 1 : t;
      const float lse_r = ok ? p.lse[j * p.N + t] * 1.4426950408889634f : 0.f;
      const float d16 = p.sc.v[c.it.kh] * p.sc.o[c.it.kh];
      const float sl2 = p.scale_log2 / (p.sc.q[c.it.kh] * p.sc.k[c.it.kh]);
      const float mul_q = p.scale / (kDS16 * p.sc.k[c.it.kh] * d16);
      const float dl = ok ? p.delta[j * p.N + t] * d16 : 0.f;
      for (int kt = s.k0; kt < s.k1; ++kt, ++u) {
        mbar_wait_warp(bar(B_SF + w), (uint32_t)(u & 1));
        if (r == 0) DQ_TRACE(w, u, 1);  // S/dP landed
        tc_fence_after();
        const int kbase = kt * 64;
        const bool full = __all_sync(0xffffffffu, klo <= kbase && kbase + 63 <= khi);
        uint32_t dd[32];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          float sv[32], dp[32];
          tmem_ld32(tmem + lb + hf * 32, sv);
          tmem_ld32(tmem + lb + 64 + hf * 32, dp);
          tmem_wait_ld();
#pragma unroll
          for (int cc = 0; cc < 32; cc += 2) {
            const int key = kbase + hf * 32 + cc;
            float p0 = ex2(fmaf(sv[cc], sl2, -lse_r));
            float p1 = ex2(fmaf(sv[cc + 1], sl2, -lse_r));
            if (!full) {
              p0 = (key >= klo && key <= khi) ? p0 : 0.f;
              p1 = (key + 1 >= klo && key + 1 <= khi) ? p1 : 0.f;
            }
            dd[hf * 16 + (cc >> 1)] =
                pack_f16(p0 * ((dp[cc] - dl) * kDS16), p1 * ((dp[cc + 1] - dl) * kDS16));
          }
        }
        tmem_st32u(tmem + lb, dd);  // dS over S: fp16 pairs, K-packed
        tmem_wait_st_();
        tc_fence_before();
        mbar_arrive(bar(B_PF + w));
        if (r == 0) DQ_TRACE(w, u, 2);  // dS written
      }
      // epilogue: dQ (+)= scale * accumulator.  The rows are staged in this
      // warpgroup's (consumed) Q / dO sub-tiles as four SW128 boxes of 32
      // fp32 columns x (g heads x tpi tokens) and leave by TMA store -- or
      // TMA reduce-add when accumulating -- instead of 16-byte scattered
      // per-thread stores; then the Q / dO stage is released to the loader.
      mbar_wait_warp(bar(B_OF + w), (uint32_t)(n_out & 1));
      tc_fence_after();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float ov[32];
        tmem_ld32(tmem + lb + 128u + q * 32, ov);
        tmem_wait_ld();
        unsigned char* box = smem + kOffQ + (q < 2 ? w : 2 + w) * kT + (q & 1) * 16384u;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<float4*>(box + sw128_off(r, cc)) =
              make_float4(ov[4 * cc] * mul_q, ov[4 * cc + 1] * mul_q, ov[4 * cc + 2] * mul_q,
                          ov[4 * cc + 3] * mul_q);
      }
      fence_proxy_async();
      named_bar(1 + w, 128);
      if (r == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t box = sb + kOffQ + (q < 2 ? w : 2 + w) * kT + (q & 1) * 16384u;
          if (p.accumulate)
            tma_reduce_add_3d(&p.tmDQ, q * 32, c.it.kh * (int)p.g, s.t0, box);
          else
            tma_store_3d(&p.tmDQ, q * 32, c.it.kh * (int)p.g, s.t0, box);
        }
        bulk_commit();
        bulk_wait_read();
        mbar_arrive(bar(B_QE));
      }
      tc_fence_before();
      mbar_arrive(bar(B_OE + w));
      ++n_out;
    }
  }

  if (threadIdx.x == 0 || threadIdx.x == 128) bulk_wait_all();  // dQ stores complete before exit
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

#ifdef FSA_TRACE
long long* g_dq_trace = nullptr;
#else
constexpr long long* g_dq_trace = nullptr;
#endif
int tc_slide_dq(const fsa_shape* s, const void* Q, const void* K, const void* V, const void* dOut,
                const void* lse, const void* delta, void* dQ, int accumulate, F16Scales sc,
                cudaStream_t st) {
  Params p{};
  p.sc = sc;
  p.trace = g_dq_trace;
  p.Q = (const __half*)Q;
  p.K = (const __half*)K;
  p.V = (const __half*)V;
  p.dO = (const __half*)dOut;
  p.lse = (const float*)lse;
  p.delta = (const float*)delta;
  p.dQ = (float*)dQ;
  p.N = s->N;
  p.h = s->h;
  p.h_K = s->h_K;
  p.g = s->h / s->h_K;
  p.W = s->W;
  p.tpi = (int)(kRows / p.g);
  p.n_super = (p.N + 2 * p.tpi - 1) / (2 * p.tpi);
  p.accumulate = accumulate;
  p.scale = (float)s->scale;
  p.scale_log2 = (float)(s->scale * 1.4426950408889634);
  int rc = make_tmap_tokens(&p.tmQ, Q, p.N, p.h, (int)p.g, p.tpi);
  if (!rc) rc = make_tmap_tokens(&p.tmO, dOut, p.N, p.h, (int)p.g, p.tpi);
  if (!rc) rc = make_tmap_tokens(&p.tmK, K, p.N, p.h_K, 1, 64);
  if (!rc) rc = make_tmap_tokens(&p.tmV, V, p.N, p.h_K, 1, 64);
  if (!rc) rc = make_tmap_tokens_f32(&p.tmDQ, dQ, p.N, p.h, (int)p.g, p.tpi);
  if (rc) return rc;
  static unsigned long long done = 0;
  ensure_smem_attr(tc_slide_dq_kernel<0>, (int)kSmemBytes, done);
  int64_t items = p.h_K * p.n_super;
  int grid = num_sms();
  if (items < grid) grid = (int)items;
  if (grid < 1) return FSA_OK;
  tc_slide_dq_kernel<0><<<grid, kThreads, kSmemBytes, st>>>(p);
  FSA_LAUNCH_CHECK("tc_slide_dq");
  return FSA_OK;
}

// Compressed-branch dQ += scale * dS K_cmp: the same
// query-outer kernel over the formed pooled rows (Kb / Vb bf16 [b][h_K][128]).
int tc_cmp_dq(const fsa_shape* s, const void* Q, const void* Kb, const void* Vb, const void* dOut,
              const void* lse, const void* delta, void* dQ, F16Scales sc, cudaStream_t st) {
  Params p{};
  p.sc = sc;
  p.Q = (const __half*)Q;
  p.K = (const __half*)Kb;
  p.V = (const __half*)Vb;
  p.dO = (const __half*)dOut;
  p.lse = (const float*)lse;
  p.delta = (const float*)delta;
  p.dQ = (float*)dQ;
  p.N = s->N;
  p.h = s->h;
  p.h_K = s->h_K;
  p.g = s->h / s->h_K;
  p.W = s->W;
  p.cmp = 1;
  p.cmpBK = s->B_K;
  p.tpi = (int)(kRows / p.g);
  p.n_super = (p.N + 2 * p.tpi - 1) / (2 * p.tpi);
  p.accumulate = 1;
  p.scale = (float)s->scale;
  p.scale_log2 = (float)(s->scale * 1.4426950408889634);
  const int64_t b = s->N / s->B_K;
  int rc = make_tmap_tokens(&p.tmQ, Q, p.N, p.h, (int)p.g, p.tpi);
  if (!rc) rc = make_tmap_tokens(&p.tmO, dOut, p.N, p.h, (int)p.g, p.tpi);
  if (!rc) rc = make_tmap_tokens(&p.tmK, Kb, b, p.h_K, 1, 64);
  if (!rc) rc = make_tmap_tokens(&p.tmV, Vb, b, p.h_K, 1, 64);
  if (!rc) rc = make_tmap_tokens_f32(&p.tmDQ, dQ, p.N, p.h, (int)p.g, p.tpi);
  if (rc) return rc;
  static unsigned long long done = 0;
  ensure_smem_attr(tc_slide_dq_kernel<1>, (int)kSmemBytes, done);
  int64_t items = p.h_K * p.n_super;
  int grid = num_sms();
  if (items < grid) grid = (int)items;
  if (grid < 1) return FSA_OK;
  tc_slide_dq_kernel<1><<<grid, kThreads, kSmemBytes, st>>>(p);
  FSA_LAUNCH_CHECK("tc_cmp_dq");
  return FSA_OK;
}

}  // namespace fsa

#ifdef FSA_TRACE
extern "C" void fsa_debug_dq_trace(void* device_buf) { fsa::g_dq_trace = (long long*)device_buf; }
#endif
