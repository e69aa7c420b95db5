// Query-outer tcgen05 attention forward for the two dense-window NSA branches
// (bf16, d = 128):
//   mode SLIDE: sliding_attention_forward (branches.py:81-83): token t sees
//               keys s in [t - W + 1, t]                        (K10)
//   mode CMP  : compressed_attention_forward (branches.py:47-78): token t sees
//               the (t+1) // B_K formed pooled rows, with the importance
//               scores of selection.py:105-120 as a fused epilogue   (K2)
//
// Work unit = a *super item*: 2 sub-items of TPI = 128/g consecutive tokens x
// the g query heads of one kv head (128 MMA rows each).  The two sub-items
// share one stream of 64-key K/V tiles (the union of their key ranges), so
// every K/V tile is loaded once for 256 rows.  Softmax warpgroup w owns
// sub-item w:
//   S_w = Q_w K^T  (M128 N64 K128) -> TMEM stage v of wg w
//   softmax: mask, lazy running max (moved only on a > 2^8 increase, so the
//            O accumulator is rescaled almost never), P = exp2(...) <= 2^8
//            packed fp16 written back over S in TMEM (tcgen05.st)
//   O_w += P V     (M128 N128 K64, fp16: A operand = P read from TMEM, V the
//                   power-of-two scaled fp16 copy of f16_stage.cu; the
//                   epilogue divides by the head's scale)
// The MMA thread runs four in-order streams (S_0, S_1, PV_0, PV_1) polled
// without blocking, so neither warpgroup waits for the other.
//
// Roles: warps 0-3 / 4-7 softmax + epilogue of sub-item 0 / 1 (thread = TMEM
// lane = MMA row), warp 8 the TMA loader (one lane; 9-10 idle), warp 11 the MMA issuer.
// TMEM: wg w owns columns [256 w, 256 w + 256): S/P stages at +0 / +64, O at +128.
#include "tc_plan.cuh"
#include "tc_sched.cuh"

namespace fsa {
namespace {

using namespace tc;

constexpr int kD = 128, kRows = 128;
constexpr int kThreads = 12 * 32;  // 2 softmax warpgroups, 3 loader warps, 1 MMA warp
constexpr uint32_t kQ = 32768, kKV = 32768;
constexpr int kKVStages = 3;
constexpr uint32_t kOffQ = 0;                           // [2 stages][2 subs] x kQ
constexpr uint32_t kOffKV = 4 * kQ;                     // [3 stages] x (K | V)
constexpr uint32_t kOffBar = kOffKV + kKVStages * kKV;  // 229376
enum { B_QF = 0, B_QE = 2, B_KF = 4, B_KE = 7, B_SF = 10, B_PF = 14, B_OF = 18, B_OE = 20,
       B_PV = 22, kNumBars = 24 };
constexpr uint32_t kOffTmem = kOffBar + kNumBars * 8;
constexpr uint32_t kSmemBytes = kOffTmem + 16 + 1024;
static_assert(kSmemBytes <= 232448, "shared memory budget");
// S operands: bf16 Q / K (SLIDE; SCORES: the hi/lo pairs), fp16 in CMP mode --
// the fsa_stage_f16_ops copy of Q against the fp16 staged pooled K, exactly
// the operands the compressed backward recomputes S from (tc_sel_bwd.cu /
// tc_slide_dq.cu compressed modes), so its P = exp(S - lse) is consistent
template <int M>
__host__ __device__ constexpr uint32_t ids_of() {
  return M == 1 ? idesc_f16(128, 64, false, false) : idesc_bf16(128, 64, false, false);
}
constexpr uint32_t kIdPV = idesc_f16(128, 128, false, true);  // P, V16 in fp16
constexpr float kRescale = 8.f;  // exp2 units

// SCORES: importance scores only (no softmax / PV), on the group-summed
// queries as bf16 hi/lo pairs (a g = 2 problem: the epilogue adds a token's
// two rows) against K_cmp hi (K slot) + lo (V slot): scores = Qsum . K_cmp *
// score_mul at ~fp32 accuracy.
enum Mode { SLIDE = 0, CMP = 1, SCORES = 2 };

#ifdef FSA_TRACE
#define QO_TRACE(w, item, slot)                                                          \
  do {                                                                                   \
    if (p.trace && blockIdx.x == 0 && (item) < 128)                                      \
      p.trace[((w) * 128 + (item)) * 8 + (slot)] = clock64();                            \
  } while (0)
#else
#define QO_TRACE(w, item, slot) \
  do {                         \
  } while (0)
#endif

struct Params {
  CUtensorMap tmOut;  // out boxes (fp32, 32 columns x g x tpi): the epilogue TMA store
  CUtensorMap tmQ, tmK, tmV;  // TMA: Q box (64, g, tpi), key/value boxes (64, 1, 64)
  long long* trace;  // debug timeline (CTA 0), null in production
  // keys bf16, values the fp16 staged copy (SCORES: the V slot holds K_cmp's
  // bf16 low part): K,V [N][h_K][128] or pooled [b][h_K][128]
  const void *Q, *Kx;      // 16-bit: bf16, or fp16 (CMP: Q16, pooled K16)
  const float *qscale, *kscale;  // CMP: the fp16 operands' per-kv-head scales
  const void* Vx;
  const float* vscale;  // [h_K] power-of-two scale of the fp16 values
  float *out, *lse, *scores;
  int64_t N, h, h_K, g, W, B_K, b, n_keys, n_super;
  int tpi, mode;
  float scale, scale_log2;
  float score_mul;  // scale / g of the real head group
};

struct Sub {
  int t0, tlast;  // tokens [t0, tlast] (tlast < t0: none)
  int k0, k1;     // key tiles [k0, k1)
};
struct Super {
  int kh;
  Sub s[2];
  int u0, u1;  // union of the key-tile ranges
};

template <int M>
__device__ __forceinline__ bool super_of(const Params& p, int id, Super& it) {
  if (id >= p.h_K * p.n_super) return false;
  it.kh = id % (int)p.h_K;
  int st = id / (int)p.h_K;
  if (M != SLIDE) st = (int)p.n_super - 1 - st;  // heavy (late) tokens first
  it.u0 = INT32_MAX;
  it.u1 = 0;
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    Sub& s = it.s[w];
    s.t0 = (2 * st + w) * p.tpi;
    s.tlast = min(s.t0 + p.tpi, (int)p.N) - 1;
    s.k0 = s.k1 = 0;
    if (s.tlast >= s.t0) {
      if (M == SLIDE) {
        s.k0 = (s.t0 - (int)p.W + 1 > 0 ? s.t0 - (int)p.W + 1 : 0) / 64;
        s.k1 = s.tlast / 64 + 1;
      } else {
        s.k1 = ((s.tlast + 1) / (int)p.B_K + 63) / 64;
      }
    }
    if (s.k0 < s.k1) {
      it.u0 = min(it.u0, s.k0);
      it.u1 = max(it.u1, s.k1);
    }
  }
  if (it.u0 >= it.u1) it.u0 = it.u1 = 0;
  return true;
}

// Position of one stream in the CTA's sequence of non-empty super items.
template <int M>
struct Cursor {
  int n = -1;    // enumeration index
  int seq = -1;  // index among non-empty super items (Q stage sequence)
  int rbase = 0, rnext = 0;  // ring index of it.u0 / of the next item's u0
  Super it;
  __device__ bool advance(const Params& p, int G) {
    for (;;) {
      ++n;
      if (!super_of<M>(p, (int)blockIdx.x + n * G, it)) return false;
      if (it.u0 == it.u1) continue;
      ++seq;
      rbase = rnext;
      rnext += it.u1 - it.u0;
      return true;
    }
  }
};

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  tmem_st32u(taddr, reinterpret_cast<const uint32_t*>(v));
}

// M: SLIDE / CMP / SCORES at compile time (per-mode code only: instruction-cache footprint)
template <int M>
__global__ void __launch_bounds__(kThreads, 1) tc_qo_fwd_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int k) { return sb + kOffBar + 8u * (uint32_t)k; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(B_QF + s), 1);  // TMA: arrive.expect_tx + bytes
      mbar_init(bar(B_QE + s), M == SCORES ? 1 : 2);  // SCORES: one MMA commit; else both epilogues
      mbar_init(bar(B_OF + s), 1);
      mbar_init(bar(B_OE + s), 128);
      mbar_init(bar(B_PV + s), 1);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(bar(B_SF + s), 1);
      mbar_init(bar(B_PF + s), 128);
    }
    for (int s = 0; s < kKVStages; ++s) {
      mbar_init(bar(B_KF + s), 1);
      mbar_init(bar(B_KE + s), 1);  // one commit per union tile, after both PV streams
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
    // A sub-item's Q is TPI consecutive tokens x the g heads of one kv head:
    // one 3-D box per 64-feature half lands as the SW128 K-major tile; key /
    // value tiles are 64 consecutive rows of one kv head.
    if (lane == 0) {
      const uint32_t qbox = 64u * (uint32_t)(p.g * p.tpi) * 2u;
      Cursor<M> c;
      int r = 0;
      while (c.advance(p, G)) {
        const int qs = (int)(c.seq & 1);
        mbar_spin(bar(B_QE + qs), (uint32_t)(((c.seq >> 1) & 1) ^ 1));
        mbar_arrive_expect_tx(bar(B_QF + qs), 4u * qbox);
#pragma unroll
        for (int w = 0; w < 2; ++w)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
            tma_load_3d(sb + kOffQ + (qs * 2 + w) * kQ + hf * 16384u, &p.tmQ, hf * 64,
                        c.it.kh * (int)p.g, c.it.s[w].t0, bar(B_QF + qs));
        const bool with_v = true;  // SCORES: the V slot carries K_cmp's low part
        for (int u = c.it.u0; u < c.it.u1; ++u, ++r) {
          const int v = (int)(r % kKVStages);
          mbar_spin(bar(B_KE + v), (uint32_t)(((r / kKVStages) & 1) ^ 1));
          mbar_arrive_expect_tx(bar(B_KF + v), with_v ? kKV : kKV / 2);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            tma_load_3d(sb + kOffKV + v * kKV + hf * 8192u, &p.tmK, hf * 64, c.it.kh, u * 64,
                        bar(B_KF + v));
            if (with_v)
              tma_load_3d(sb + kOffKV + v * kKV + 16384u + hf * 8192u, &p.tmV, hf * 64, c.it.kh,
                          u * 64, bar(B_KF + v));
          }
        }
      }
    }
  } else if (warp == 11) {
    // ------------------------------------------------------------ MMA issuer
    // Static order with blocking waits (one lane waits, the warp follows; one
    // elected lane issues): per union tile u of a super item, S of both
    // sub-items for tile u, then PV of both for tile u-1 (S runs one tile
    // ahead so the softmax of u-1 overlaps the S MMAs of u).  One KE commit per
    // union tile after both PV streams frees its K/V stage (a single arrival
    // per phase: synccheck-clean); SCORES: one QE commit per super item (the
    // other modes' QE arrivals come from the two epilogues).
    {
      Cursor<M> c;
      int ns[2] = {0, 0}, np[2] = {0, 0}, nsub[2] = {0, 0};
      while (c.advance(p, G)) {
        const Super& it = c.it;
        const int qs = (int)(c.seq & 1);
        bool q_ready = false;
        for (int u = it.u0; u <= it.u1; ++u) {
          if (u < it.u1) {  // ---- S of tile u
            const int rr = c.rbase + (u - it.u0), kv = rr % kKVStages;
            mbar_wait_warp(bar(B_KF + kv), (uint32_t)((rr / kKVStages) & 1));
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              if (u < it.s[w].k0 || u >= it.s[w].k1) continue;
              if (!q_ready) {
                mbar_wait_warp(bar(B_QF + qs), (uint32_t)((c.seq >> 1) & 1));
                q_ready = true;
              }
              tc_fence_after();
              const int v = ns[w] & 1;
              const uint32_t q = sb + kOffQ + (qs * 2 + w) * kQ, k = sb + kOffKV + kv * kKV;
              const uint32_t tS = tmem + 256u * w + 64u * v;
              if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                  mma_bf16(tS, desc_kmajor(q + (kk >> 2) * 16384u + (kk & 3) * 32u),
                           desc_kmajor(k + (kk >> 2) * 8192u + (kk & 3) * 32u), ids_of<M>(), kk > 0);
                if constexpr (M == SCORES) {  // + Q . K_lo^T (the V slot holds K_cmp's low part)
#pragma unroll
                  for (int kk = 0; kk < 8; ++kk)
                    mma_bf16(tS, desc_kmajor(q + (kk >> 2) * 16384u + (kk & 3) * 32u),
                             desc_kmajor(k + 16384u + (kk >> 2) * 8192u + (kk & 3) * 32u), ids_of<M>(), 1u);
                }
                mma_commit(bar(B_SF + 2 * w + v));
                QO_TRACE(w, ns[w], 0);  // S issued
              }
              __syncwarp();
              ++ns[w];
            }
          }
          if (u > it.u0) {  // ---- PV of tile u-1, then the K/V stage release
            const int up = u - 1;
            const int rr = c.rbase + (up - it.u0), kv = rr % kKVStages;
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              const Sub& sw = it.s[w];
              if (up < sw.k0 || up >= sw.k1) continue;  // tile outside this sub-item
              const int v = np[w] & 1;
              const bool first = up == sw.k0, last = up + 1 == sw.k1;
              mbar_wait_warp(bar(B_PF + 2 * w + v), (uint32_t)((np[w] >> 1) & 1));
              if (M == SCORES) {  // no PV: the K tile is released once S is consumed
                ++np[w];
                continue;
              }
              if (first) mbar_wait_warp(bar(B_OE + w), (uint32_t)((nsub[w] & 1) ^ 1));
              tc_fence_after();
              const uint32_t vv = sb + kOffKV + kv * kKV + 16384u;
              const uint32_t tS = tmem + 256u * w + 64u * v, tO = tmem + 256u * w + 128u;
              if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_bf16_ts(tO, tS + kk * 8, desc_mnmajor(vv + kk * 2048u, 8192u), kIdPV,
                              (first && kk == 0) ? 0u : 1u);
                mma_commit(bar(B_PV + w));
                if (last) mma_commit(bar(B_OF + w));
                QO_TRACE(w, np[w], 3);  // PV issued
              }
              __syncwarp();
              if (last) ++nsub[w];
              ++np[w];
            }
            // one commit per union tile frees its K/V stage once every MMA
            // reading it (both sub-items' S and PV) has completed
            if (elect_one()) mma_commit(bar(B_KE + kv));
            __syncwarp();
          }
        }
        // SCORES: both S streams are done with this Q stage.  (SLIDE / CMP: the
        // softmax warpgroups release it after their epilogue has staged the
        // output rows in it and the TMA store has read them.)
        if constexpr (M == SCORES) {
          if (elect_one()) mma_commit(bar(B_QE + qs));
          __syncwarp();
        }
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ softmax / epilogue
    const int w = warp >> 2;
    const int r = threadIdx.x & 127;
    const uint32_t lb = ((uint32_t)((warp & 3) * 32) << 16) + 256u * w;
    const int kt_row = r / (int)p.g, hh = r % (int)p.g;
    int u = 0, n_out = 0;  // tiles processed / sub-items finished by this wg
    Cursor<M> c;
    while (c.advance(p, G)) {
      const Sub& s = c.it.s[w];
      if (s.k0 >= s.k1) {  // empty sub-item: nothing staged in this Q stage
        if (M != SCORES && r == 0) mbar_arrive(bar(B_QE + (c.seq & 1)));
        continue;
      }
      const int t = s.t0 + kt_row;
      const bool ok = kt_row < p.tpi && t <= s.tlast;
      const int64_t j = (int64_t)c.it.kh * p.g + hh;
      int klo, khi;  // visible keys [klo, khi]
      if (M == SLIDE) {
        klo = t - (int)p.W + 1 > 0 ? t - (int)p.W + 1 : 0;
        khi = t;
      } else {
        klo = 0;
        khi = (t + 1) / (int)p.B_K - 1;
      }
      if (!ok) khi = -1;
      float m_used = -INFINITY, l = 0.f;
      float sl2 = p.scale_log2, scl = p.scale;  // per unit of S as computed
      if (M == CMP) {  // S16 = S s_Q s_Kc
        const float f = 1.f / (__ldg(p.qscale + c.it.kh) * __ldg(p.kscale + c.it.kh));
        sl2 *= f;
        scl *= f;
      }
      for (int kt = s.k0; kt < s.k1; ++kt, ++u) {
        const int v = (int)(u & 1);
        const uint32_t tS = tmem + lb + 64u * v;
        mbar_wait_warp(bar(B_SF + 2 * w + v), (uint32_t)((u >> 1) & 1));
        if (r == 0) QO_TRACE(w, u, 1);  // S landed
        tc_fence_after();
        float sv[64];
        tmem_ld32(tS, sv);
        tmem_ld32(tS + 32, sv + 32);
        tmem_wait_ld();
        const int kbase = kt * 64;
        if (M == SCORES) {
          // the token's rows (hi, lo) are adjacent lanes (g = 2): each lane of
          // the pair sends the half the other one stores -- lane hh sums and
          // writes columns [32 hh, 32 hh + 32) (hi + lo, lo + hi: the same
          // float sum), so one shuffle and half a row of stores per column pair
          const float gm = p.score_mul;
          const int c0 = 32 * hh;
          float* dst = p.scores + ((int64_t)c.it.kh * p.N + t) * p.b + kbase + c0;
          const bool wr = ok;
#pragma unroll
          for (int cc = 0; cc < 32; cc += 8) {
            float x[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float mine = hh ? sv[32 + cc + e] : sv[cc + e];
              const float give = hh ? sv[cc + e] : sv[32 + cc + e];
              x[e] = (mine + __shfl_xor_sync(0xffffffffu, give, 1)) * gm;
            }
            if (wr) {
              if (kbase + c0 + cc + 7 < p.b && (p.b & 7) == 0) {  // one full 32 B sector per store
                asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + cc),
                             "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]),
                             "f"(x[7])
                             : "memory");
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                  if (kbase + c0 + cc + e < p.b) dst[cc + e] = x[e];
              }
            }
          }
        }
        if (M == SCORES) {  // S consumed: hand the stage back
          tc_fence_before();
          mbar_arrive(bar(B_PF + 2 * w + v));
          continue;
        }
        // rows whose visible range covers the whole tile skip the masking
        const bool full = __all_sync(0xffffffffu, klo <= kbase && kbase + 63 <= khi);
        float mx = -INFINITY;
        if (full) {
#pragma unroll
          for (int cc = 0; cc < 64; ++cc) mx = fmaxf(mx, sv[cc]);
        } else {
#pragma unroll
          for (int cc = 0; cc < 64; ++cc) {
            const bool vis = kbase + cc >= klo && kbase + cc <= khi;
            sv[cc] = vis ? sv[cc] : -INFINITY;
            mx = fmaxf(mx, sv[cc]);
          }
        }
        // move the reference max only on a large increase (or the first finite max)
        float f = 1.f;
        bool resc = false;
        if (mx > -INFINITY && (m_used == -INFINITY || (mx - m_used) * sl2 > kRescale)) {
          if (m_used != -INFINITY) {
            f = ex2((m_used - mx) * sl2);
            l *= f;
            resc = true;
          }
          m_used = mx;
        }
        // rescale O in TMEM once PV(u-1) has landed (warp-collective)
        if (__any_sync(0xffffffffu, resc)) {
          mbar_wait_warp(bar(B_PV + w), (uint32_t)((u - 1) & 1));
          tc_fence_after();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float ov[32];
            tmem_ld32(tmem + lb + 128u + q * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) ov[cc] *= f;
            tmem_st32(tmem + lb + 128u + q * 32, ov);
          }
          tmem_wait_st_();
        }
        const float mb = m_used == -INFINITY ? 0.f : m_used * sl2;
        uint32_t pk[32];
        float l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int cc = 0; cc < 64; cc += 2) {
          const float e0 = ex2(fmaf(sv[cc], sl2, -mb));  // -inf -> 0
          const float e1 = ex2(fmaf(sv[cc + 1], sl2, -mb));
          l0 += e0;
          l1 += e1;
          pk[cc >> 1] = pack_f16(e0, e1);
        }
        l += l0 + l1;
        tmem_st32u(tS, pk);  // P over S: fp16 pairs, K-packed
        tmem_wait_st_();
        // observe PV(u-1)'s completion every tile (the rescale above waits for
        // it only when the reference max moves), so every commit-driven phase
        // of B_PV gets a waiter.  Before P(u) is published: PV(u) cannot have
        // completed yet, so the parity test cannot alias a later phase; PV(u-1)
        // was issued a whole softmax ago and rarely blocks.
        if (u > 0) mbar_wait_warp(bar(B_PV + w), (uint32_t)((u - 1) & 1));
        tc_fence_before();
        mbar_arrive(bar(B_PF + 2 * w + v));
        if (r == 0) QO_TRACE(w, u, 2);  // P written
        if (lane == 0) QO_TRACE(w + 2, u, 2 + (warp & 3));  // per-warp P arrival
      }
      if (M == SCORES) continue;
      // epilogue: out = O / l, lse = m + ln l
      if (r == 0) QO_TRACE(w, u - 1, 4);  // epilogue: waiting for O
      mbar_wait_warp(bar(B_OF + w), (uint32_t)(n_out & 1));
      if (r == 0) QO_TRACE(w, u - 1, 5);  // O complete
      tc_fence_after();
      const bool write = ok && l > 0.f;
      const float inv = write ? 1.f / (l * __ldg(p.vscale + c.it.kh)) : 0.f;
      // Rows leave by TMA store: staged in this warpgroup's consumed Q
      // sub-tile (32 KB) as two SW128 boxes of 32 fp32 columns x (g heads x
      // tpi tokens) at a time -- instead of 16-byte scattered per-thread
      // stores.  Rows without a visible key are stored as 0 (the compressed
      // branch's pending tokens are written after this kernel).
      unsigned char* qsub = smem + kOffQ + ((c.seq & 1) * 2 + w) * kQ;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
          if (r == 0) bulk_wait_read();
          named_bar(1 + w, 128);
        }
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const int q = 2 * pass + qq;
          float ov[32];
          tmem_ld32(tmem + lb + 128u + q * 32, ov);
          tmem_wait_ld();
          unsigned char* box = qsub + qq * 16384u;
#pragma unroll
          for (int cc = 0; cc < 8; ++cc)
            *reinterpret_cast<float4*>(box + sw128_off(r, cc)) =
                make_float4(ov[4 * cc] * inv, ov[4 * cc + 1] * inv, ov[4 * cc + 2] * inv,
                            ov[4 * cc + 3] * inv);
        }
        fence_proxy_async();
        named_bar(1 + w, 128);
        if (r == 0) {
#pragma unroll
          for (int qq = 0; qq < 2; ++qq)
            tma_store_3d(&p.tmOut, (2 * pass + qq) * 32, c.it.kh * (int)p.g, s.t0,
                         smem_u32(qsub) + qq * 16384u);
          bulk_commit();
        }
      }
      if (r == 0) {
        bulk_wait_read();
        mbar_arrive(bar(B_QE + (c.seq & 1)));
      }
      tc_fence_before();
      mbar_arrive(bar(B_OE + w));
      if (r == 0) QO_TRACE(w, u - 1, 6);  // epilogue done
      if (write) p.lse[j * p.N + t] = m_used * scl + __logf(l);
      ++n_out;
    }
  }

  if (threadIdx.x == 0 || threadIdx.x == 128) bulk_wait_all();  // out stores complete before exit
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

__global__ void to_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = __float2bfloat16_rn(x[e]);
}

#ifdef FSA_TRACE
long long* g_qo_trace = nullptr;
#else
constexpr long long* g_qo_trace = nullptr;
#endif
int launch(Params& p, cudaStream_t st) {
  p.trace = (p.mode == SLIDE) ? g_qo_trace : nullptr;
  int rc = make_tmap_tokens(&p.tmQ, p.Q, p.N, p.h, (int)p.g, p.tpi);
  if (!rc) rc = make_tmap_tokens(&p.tmK, p.Kx, p.n_keys, p.h_K, 1, 64);
  if (!rc) rc = make_tmap_tokens(&p.tmV, p.Vx, p.n_keys, p.h_K, 1, 64);
  if (!rc && p.out) rc = make_tmap_tokens_f32(&p.tmOut, p.out, p.N, p.h, (int)p.g, p.tpi);
  if (rc) return rc;
  static unsigned long long done[3] = {0, 0, 0};
  ensure_smem_attr(tc_qo_fwd_kernel<SLIDE>, (int)kSmemBytes, done[0]);
  ensure_smem_attr(tc_qo_fwd_kernel<CMP>, (int)kSmemBytes, done[1]);
  ensure_smem_attr(tc_qo_fwd_kernel<SCORES>, (int)kSmemBytes, done[2]);
  int64_t items = p.h_K * p.n_super;
  int grid = num_sms();
  if (items < grid) grid = (int)items;
  if (grid < 1) return FSA_OK;
  if (p.mode == SLIDE)
    tc_qo_fwd_kernel<SLIDE><<<grid, kThreads, kSmemBytes, st>>>(p);
  else if (p.mode == CMP)
    tc_qo_fwd_kernel<CMP><<<grid, kThreads, kSmemBytes, st>>>(p);
  else
    tc_qo_fwd_kernel<SCORES><<<grid, kThreads, kSmemBytes, st>>>(p);
  return FSA_OK;
}

Params base_params(const fsa_shape* s) {
  Params p{};
  p.N = s->N;
  p.h = s->h;
  p.h_K = s->h_K;
  p.g = s->h / s->h_K;
  p.W = s->W;
  p.B_K = s->B_K;
  p.b = s->N / s->B_K;
  p.tpi = (int)(kRows / p.g);
  p.n_super = (p.N + 2 * p.tpi - 1) / (2 * p.tpi);
  p.scale = (float)s->scale;
  p.scale_log2 = (float)(s->scale * 1.4426950408889634);
  p.score_mul = (float)(s->scale / (double)p.g);
  return p;
}

// Qsum[t][kh] = sum of the g query rows of kv head kh, as a bf16 hi/lo pair
// Qs[t][kh][0] = bf16(sum), Qs[t][kh][1] = bf16(sum - hi): the scores pass runs
// it as a g = 2 problem whose two rows per token are added in the epilogue, so
// (hi + lo) . (K_hi + K_lo) keeps the scores at ~fp32 accuracy -- bf16 operands
// alone flip ~2 % of the top-k selections against the float64 reference.
__global__ void qsum_kernel(const __nv_bfloat16* __restrict__ Q, __nv_bfloat16* __restrict__ Qs,
                            int64_t N, int64_t h_K, int64_t g) {
  const int64_t row = blockIdx.x * 8ll + (threadIdx.x >> 5);  // (t, kh)
  if (row >= N * h_K) return;
  const int lane = threadIdx.x & 31;
  const __nv_bfloat16* src = Q + row * g * kD + lane * 4;
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t j = 0; j < g; ++j) {
    const uint2 u = *reinterpret_cast<const uint2*>(src + j * kD);
    const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    a[0] += x.x; a[1] += x.y; a[2] += y.x; a[3] += y.y;
  }
  __nv_bfloat16 hi[4], lo[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    hi[e] = __float2bfloat16_rn(a[e]);
    lo[e] = __float2bfloat16_rn(a[e] - __bfloat162float(hi[e]));
  }
  *reinterpret_cast<uint2*>(Qs + (row * 2) * kD + lane * 4) = *reinterpret_cast<const uint2*>(hi);
  *reinterpret_cast<uint2*>(Qs + (row * 2 + 1) * kD + lane * 4) = *reinterpret_cast<const uint2*>(lo);
}

// K_lo = bf16(K_cmp - bf16(K_cmp))
__global__ void lo_part_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ hi,
                               __nv_bfloat16* __restrict__ lo, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    lo[e] = __float2bfloat16_rn(x[e] - __bfloat162float(hi[e]));
}

}  // namespace

bool tc_qo_supported(const fsa_shape& s, int dtype) {
  return dtype == FSA_DT_BF16 && s.d_K == kD && s.d_V == kD && s.h_K > 0 && s.h % s.h_K == 0 &&
         s.h / s.h_K <= kRows && s.N < (1ll << 30);
}

int tc_slide_fwd(const fsa_shape* s, const void* Q, const void* K, const void* V16,
                 const float* vscale, void* out, void* lse, cudaStream_t st) {
  FSA_REQUIRE(vscale != nullptr, "slide_fwd: the tensor-core path takes the fp16 V copy and its "
              "scales (fsa_v_to_f16)");
  Params p = base_params(s);
  p.mode = SLIDE;
  p.Q = Q;
  p.Kx = K;
  p.Vx = V16;
  p.vscale = vscale;
  p.n_keys = s->N;
  p.out = (float*)out;
  p.lse = (float*)lse;
  p.scores = nullptr;
  if (int rc = launch(p, st)) return rc;
  FSA_LAUNCH_CHECK("tc_slide_fwd");
  return FSA_OK;
}

size_t tc_cmp_workspace_bytes(const fsa_shape* s) {
  // bf16 pooled K, fp16 (scaled) pooled V, the group-summed queries as bf16
  // hi/lo pairs, the pooled V's per-head scales (+ scratch), the fp16 (scaled)
  // pooled K and its scales (+ scratch)
  const size_t n = (size_t)(s->N / s->B_K) * s->h_K * kD;
  return 2 * n * 2 + (size_t)2 * s->N * s->h_K * kD * 2 + 2 * s->h_K * sizeof(float) + 256 +
         n * 2 + 256 + 2 * s->h_K * sizeof(float);
}

int tc_cmp_fwd(const fsa_shape* s, const void* Q, const void* Q16, const float* qscale,
               const void* Kc, const void* Vc, void* out, void* lse, void* scores, void* workspace,
               cudaStream_t st) {
  FSA_REQUIRE(Q16 != nullptr && qscale != nullptr,
              "cmp_attn_fwd: the tensor-core path reads the fsa_stage_f16_ops copy of Q and its scales");
  Params p = base_params(s);
  p.mode = CMP;
  const int64_t n = p.b * p.h_K * kD;
  __nv_bfloat16* kb = (__nv_bfloat16*)workspace;
  __nv_bfloat16* vb = kb + n;
  float* vsc = reinterpret_cast<float*>(vb + n + 2 * p.N * p.h_K * kD);
  // 256-byte aligned (TMA base addresses need 16)
  auto align = [](void* x) { return (void*)(((uintptr_t)x + 255) & ~(uintptr_t)255); };
  __half* k16 = (__half*)align(vsc + 2 * p.h_K);
  float* ksc = (float*)align(k16 + n);
  if (int rc = stage_f16(FSA_DT_F32, Kc, p.b, p.h_K, kD, k16, ksc, st)) return rc;
  if (int rc = stage_f16(FSA_DT_F32, Vc, p.b, p.h_K, kD, vb, vsc, st)) return rc;
  p.Q = Q16;
  p.qscale = qscale;
  p.Kx = k16;
  p.kscale = ksc;
  p.Vx = vb;
  p.vscale = vsc;
  p.n_keys = p.b;
  p.out = (float*)out;
  p.lse = (float*)lse;
  p.scores = nullptr;  // the scores come from their own hi/lo pass below
  if (int rc = launch(p, st)) return rc;
  FSA_LAUNCH_CHECK("tc_cmp_fwd");
  if (scores != nullptr) {
    // scores on the tensor cores for any g: the g query rows of a kv head are
    // summed first (hi/lo), then a g = 2 problem over (Qsum_hi, Qsum_lo) against
    // K_cmp hi (the K slot) + lo (the V slot, overwriting the pooled V copy the
    // compressed pass above has finished with) computes Qsum . K_cmp
    __nv_bfloat16* qs = vb + n;
    to_bf16_kernel<<<148, 256, 0, st>>>((const float*)Kc, kb, n);
    lo_part_kernel<<<148, 256, 0, st>>>((const float*)Kc, kb, vb, n);
    qsum_kernel<<<(unsigned)((p.N * p.h_K + 7) / 8), 256, 0, st>>>((const __nv_bfloat16*)Q, qs,
                                                                    p.N, p.h_K, p.g);
    Params q = p;
    q.mode = SCORES;
    q.Q = qs;
    q.Kx = kb;  // K_cmp hi; lo in the V slot (vb)
    q.h = 2 * p.h_K;
    q.g = 2;
    q.tpi = kRows / 2;
    q.n_super = (q.N + 2 * q.tpi - 1) / (2 * q.tpi);
    q.scores = (float*)scores;
    q.out = nullptr;
    q.lse = nullptr;
    if (int rc = launch(q, st)) return rc;
    FSA_LAUNCH_CHECK("tc_cmp_scores");
  }
  return FSA_OK;
}

}  // namespace fsa

#ifdef FSA_TRACE
extern "C" void fsa_debug_qo_trace(void* device_buf) { fsa::g_qo_trace = (long long*)device_buf; }
#endif
