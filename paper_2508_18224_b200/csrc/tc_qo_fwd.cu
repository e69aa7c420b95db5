// Query-outer tcgen05 attention forward for the two dense-window NSA branches
// (bf16, d = 128):
//   mode SLIDE: sliding_attention_forward (branches.py:81-83): token t sees
//               keys s in [t - W + 1, t]                        (K10)
//   mode CMP  : compressed_attention_forward (branches.py:47-78): token t sees
//               the (t+1) // B_K formed pooled rows, with the importance
//               scores of selection.py:105-120 as a fused epilogue   (K2)
// One item = TPI = 128/g consecutive tokens x the g query heads of one kv head
// (128 MMA rows sharing every key tile).  Per 64-key tile: S = Q K^T (TMEM),
// softmax warps mask + exponentiate into bf16 P (smem), O += P V accumulates
// in TMEM across the item's tiles.  The running max is only moved when it
// grows by more than 2^8 (exp2 units), so O is rescaled (TMEM ld/st) almost
// never; P <= 256 stays exact enough in bf16 and the fp32 sums cannot overflow.
//
// Roles as in tc_sel_fwd.cu: warps 0-3 softmax/epilogue (thread = TMEM lane),
// 4-7 cp.async loaders, 8 MMA issuer (S of tile u+1 issued ahead of PV of u).
#include "tc_plan.cuh"
#include "tc_sched.cuh"

namespace fsa {
namespace {

using namespace tc;

constexpr int kD = 128, kRows = 128;
constexpr int kThreads = 9 * 32;
constexpr uint32_t kQ = 32768, kKV = 32768, kP = 16384;
constexpr int kKVStages = 3;
constexpr uint32_t kOffQ = 0, kOffKV = 2 * kQ, kOffP = kOffKV + kKVStages * kKV,
                   kOffBar = kOffP + 2 * kP;
enum { B_QF = 0, B_QE = 2, B_KF = 4, B_KE = 7, B_SF = 10, B_SE = 12, B_PF = 14, B_PE = 16,
       B_OF = 18, B_OE = 20, B_PV = 22, kNumBars = 23 };
constexpr uint32_t kOffTmem = kOffBar + kNumBars * 8;
constexpr uint32_t kSmemBytes = kOffTmem + 16 + 1024;
constexpr uint32_t kColS = 0, kColO = 128;  // S[2] 0..127, O[2] 128..383
constexpr uint32_t kIdS = idesc_bf16(128, 64, false, false);
constexpr uint32_t kIdPV = idesc_bf16(128, 128, false, true);
constexpr float kRescale = 8.f;  // exp2 units

enum Mode { SLIDE = 0, CMP = 1 };

struct Params {
  const __nv_bfloat16 *Q, *Kx, *Vx;  // keys/values: K,V [N][h_K][128] or pooled [b][h_K][128]
  float *out, *lse, *scores;
  int64_t N, h, h_K, g, W, B_K, b, n_keys, n_tiles_tok;
  int tpi, mode;
  float scale, scale_log2;
};

struct ItemInfo {
  int64_t kh, t0, tlast;
  int64_t k0, k1;  // key tiles [k0, k1)
};

__device__ __forceinline__ bool item_of(const Params& p, int64_t id, ItemInfo& it) {
  const int64_t total = p.h_K * p.n_tiles_tok;
  if (id >= total) return false;
  it.kh = id % p.h_K;
  int64_t tile = id / p.h_K;
  if (p.mode == CMP) tile = p.n_tiles_tok - 1 - tile;  // heavy (late) tokens first
  it.t0 = tile * p.tpi;
  it.tlast = min(it.t0 + p.tpi, p.N) - 1;
  if (p.mode == SLIDE) {
    const int64_t lo = it.t0 - p.W + 1 > 0 ? it.t0 - p.W + 1 : 0;
    it.k0 = lo / 64;
    it.k1 = it.tlast / 64 + 1;
  } else {
    const int64_t nf = (it.tlast + 1) / p.B_K;
    it.k0 = 0;
    it.k1 = (nf + 63) / 64;
  }
  return true;
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]),
      "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]),
      "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads, 1) tc_qo_fwd_kernel(const Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int k) { return sb + kOffBar + 8u * (uint32_t)k; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(B_QF + s), 128);
      mbar_init(bar(B_QE + s), 1);
      mbar_init(bar(B_SF + s), 1);
      mbar_init(bar(B_SE + s), 128);
      mbar_init(bar(B_PF + s), 128);
      mbar_init(bar(B_PE + s), 1);
      mbar_init(bar(B_OF + s), 1);
      mbar_init(bar(B_OE + s), 128);
    }
    for (int s = 0; s < kKVStages; ++s) {
      mbar_init(bar(B_KF + s), 128);
      mbar_init(bar(B_KE + s), 1);
    }
    mbar_init(bar(B_PV), 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t G = gridDim.x;

  if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ loaders
    // Each gather is its own cp.async group; the newest one stays in flight
    // while the previous one is published (one-group-deep software pipeline).
    // Blocking waits (Q stage, K/V stage) only depend on work the MMA can
    // finish without the in-flight group (3 K/V stages, look-ahead of one).
    const int lr = threadIdx.x - 128;
    int64_t u = 0, nq = 0;  // tile counter, counter of items with at least one tile
    uint32_t pend = 0;      // barrier of the in-flight group (0: none)
    auto push_group = [&](uint32_t b) {
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      fence_proxy_async();
      if (pend) mbar_arrive(pend);
      pend = b;
    };
    ItemInfo it;
    for (int64_t n = 0; item_of(p, blockIdx.x + n * G, it); ++n) {
      if (it.k0 == it.k1) continue;
      const int s = (int)(nq & 1);
      mbar_wait(bar(B_QE + s), (uint32_t)(((nq >> 1) & 1) ^ 1));
      ++nq;
      {
        const int64_t kt = lr / p.g, hh = lr % p.g, t = it.t0 + kt;
        const bool ok = kt < p.tpi && t < p.N;
        const __nv_bfloat16* src = p.Q + ((ok ? t : 0) * p.h + it.kh * p.g + hh) * kD;
        warp_gather_rows32(sb + kOffQ + s * kQ, 16384u, lr & ~31, src, ok, lane);
      }
      push_group(bar(B_QF + s));
      for (int64_t kt = it.k0; kt < it.k1; ++kt, ++u) {
        const int v = (int)(u % kKVStages);
        mbar_wait(bar(B_KE + v), (uint32_t)(((u / kKVStages) & 1) ^ 1));
        const int lw = warp - 4, row0 = (lw & 1) * 32;  // warps 4,5: K; 6,7: V
        const int64_t key = kt * 64 + row0 + lane;
        const bool ok = key < p.n_keys;
        const __nv_bfloat16* src = (lw < 2 ? p.Kx : p.Vx) + ((ok ? key : 0) * p.h_K + it.kh) * kD;
        warp_gather_rows32(sb + kOffKV + v * kKV + (lw < 2 ? 0u : 16384u), 8192u, row0, src, ok,
                           lane);
        push_group(bar(B_KF + v));
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    fence_proxy_async();
    if (pend) mbar_arrive(pend);
  } else if (warp == 8) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // flat walk over (item, tile) of the items that have tiles; S runs one
      // tile ahead of PV.  na/nb index items, qa/qb count non-empty items
      // (the Q and O stage sequence).
      ItemInfo ia, ib;
      int64_t na = 0, nb = 0, ka = 0, kb = 0, ua = 0, qa = 0, qb = 0;
      bool ha = item_of(p, blockIdx.x, ia);
      while (ha && ia.k0 == ia.k1) ha = item_of(p, blockIdx.x + (++na) * G, ia);
      bool hb = ha;
      ib = ia;
      nb = na;
      if (ha) ka = ia.k0;
      if (hb) kb = ib.k0;
      auto issue_s = [&]() {
        const int s = (int)(qa & 1), v = (int)(ua & 1), kv = (int)(ua % kKVStages);
        if (ka == ia.k0) mbar_wait(bar(B_QF + s), (uint32_t)((qa >> 1) & 1));
        mbar_wait(bar(B_KF + kv), (uint32_t)((ua / kKVStages) & 1));
        mbar_wait(bar(B_SE + v), (uint32_t)(((ua >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t q = sb + kOffQ + s * kQ, k = sb + kOffKV + kv * kKV;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_bf16(tmem + kColS + v * 64,
                   desc_kmajor(q + (kk >> 2) * 16384u + (kk & 3) * 32u),
                   desc_kmajor(k + (kk >> 2) * 8192u + (kk & 3) * 32u), kIdS, kk > 0);
        mma_commit(bar(B_SF + v));
        if (ka + 1 == ia.k1) mma_commit(bar(B_QE + s));
        ++ua;
        if (++ka == ia.k1) {  // next item with at least one tile
          ++qa;
          do {
            ha = item_of(p, blockIdx.x + (++na) * G, ia);
          } while (ha && ia.k0 == ia.k1);
          if (ha) ka = ia.k0;
        }
      };
      if (ha) issue_s();
      for (int64_t u = 0; hb; ++u) {
        if (ha) issue_s();
        const int v = (int)(u & 1), so = (int)(qb & 1), kv = (int)(u % kKVStages);
        const bool first = kb == ib.k0, last = kb + 1 == ib.k1;
        mbar_wait(bar(B_PF + v), (uint32_t)((u >> 1) & 1));
        if (first) mbar_wait(bar(B_OE + so), (uint32_t)(((qb >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t pp = sb + kOffP + v * kP, vv = sb + kOffKV + kv * kKV + 16384u;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(tmem + kColO + so * 128, desc_kmajor(pp + kk * 32u),
                   desc_mnmajor(vv + kk * 2048u, 8192u), kIdPV, (first && kk == 0) ? 0u : 1u);
        mma_commit(bar(B_PE + v));
        mma_commit(bar(B_KE + kv));
        mma_commit(bar(B_PV));
        if (last) mma_commit(bar(B_OF + so));
        if (++kb == ib.k1) {
          ++qb;
          do {
            hb = item_of(p, blockIdx.x + (++nb) * G, ib);
          } while (hb && ib.k0 == ib.k1);
          if (hb) kb = ib.k0;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax / epilogue
    const int r = threadIdx.x;
    const uint32_t lb = (uint32_t)(warp * 32) << 16;
    const int64_t kt_row = r / p.g, hh = r % p.g;
    int64_t u = 0, n_out = 0;
    ItemInfo it;
    for (int64_t n = 0; item_of(p, blockIdx.x + n * G, it); ++n) {
      if (it.k0 == it.k1) continue;  // only pending tokens: handled by the SIMT kernel
      const int64_t t = it.t0 + kt_row;
      const bool ok = kt_row < p.tpi && t < p.N;
      const int64_t j = it.kh * p.g + hh;
      // visible key range [klo, khi]
      int64_t klo, khi;
      if (p.mode == SLIDE) {
        klo = t - p.W + 1 > 0 ? t - p.W + 1 : 0;
        khi = t;
      } else {
        klo = 0;
        khi = (t + 1) / p.B_K - 1;
      }
      if (!ok) khi = -1;
      float m_used = -INFINITY, l = 0.f;
      for (int64_t kt = it.k0; kt < it.k1; ++kt, ++u) {
        const int v = (int)(u & 1);
        mbar_wait(bar(B_SF + v), (uint32_t)((u >> 1) & 1));
        tc_fence_after();
        float sv[64];
        tmem_ld32(tmem + lb + kColS + v * 64, sv);
        tmem_ld32(tmem + lb + kColS + v * 64 + 32, sv + 32);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(bar(B_SE + v));
        const int64_t kbase = kt * 64;
        if (p.mode == CMP && p.scores != nullptr) {
          // group mean over the g heads of this token (rows of a token are
          // adjacent lanes; g divides 32), written by the token's first row
          const float gm = p.scale / (float)p.g;
          float* dst = p.scores + (it.kh * p.N + t) * p.b + kbase;
          const bool wr = ok && hh == 0;
#pragma unroll
          for (int c = 0; c < 64; c += 4) {
            float x0 = sv[c], x1 = sv[c + 1], x2 = sv[c + 2], x3 = sv[c + 3];
            for (int o = 1; o < p.g; o <<= 1) {
              x0 += __shfl_xor_sync(0xffffffffu, x0, o);
              x1 += __shfl_xor_sync(0xffffffffu, x1, o);
              x2 += __shfl_xor_sync(0xffffffffu, x2, o);
              x3 += __shfl_xor_sync(0xffffffffu, x3, o);
            }
            if (wr) {
              if (kbase + c + 3 < p.b) {
                *reinterpret_cast<float4*>(dst + c) = make_float4(x0 * gm, x1 * gm, x2 * gm, x3 * gm);
              } else {
                if (kbase + c < p.b) dst[c] = x0 * gm;
                if (kbase + c + 1 < p.b) dst[c + 1] = x1 * gm;
                if (kbase + c + 2 < p.b) dst[c + 2] = x2 * gm;
              }
            }
          }
        }
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const int64_t key = kbase + c;
          if (key >= klo && key <= khi) mx = fmaxf(mx, sv[c]);
        }
        // P(u-2) consumed => PV(u-2) done, so the PV barrier parity below is unambiguous
        mbar_wait(bar(B_PE + v), (uint32_t)(((u >> 1) & 1) ^ 1));
        // move the reference max only on a large increase (or the first finite max)
        float f = 1.f;
        bool resc = false;
        if (mx > -INFINITY && (m_used == -INFINITY || (mx - m_used) * p.scale_log2 > kRescale)) {
          if (m_used != -INFINITY) {
            f = ex2((m_used - mx) * p.scale_log2);
            l *= f;
            resc = true;
          }
          m_used = mx;
        }
        // rescale the O accumulator in TMEM (warp-collective: every lane joins,
        // lanes without a new max scale by 1) once PV(u-1) has landed
        if (__any_sync(0xffffffffu, resc)) {
          mbar_wait(bar(B_PV), (uint32_t)((u - 1) & 1));
          tc_fence_after();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float ov[32];
            tmem_ld32(tmem + lb + kColO + (n_out & 1) * 128 + q * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) ov[c] *= f;
            tmem_st32(tmem + lb + kColO + (n_out & 1) * 128 + q * 32, ov);
          }
          tmem_wait_st();
          tc_fence_before();
        }
        const float mb = m_used == -INFINITY ? 0.f : m_used * p.scale_log2;
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const int64_t key = kbase + c;
          const float e0 = (key >= klo && key <= khi) ? ex2(fmaf(sv[c], p.scale_log2, -mb)) : 0.f;
          const float e1 = (key + 1 >= klo && key + 1 <= khi) ? ex2(fmaf(sv[c + 1], p.scale_log2, -mb)) : 0.f;
          l += e0 + e1;
          pk[c >> 1] = pack_bf16(e0, e1);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(smem + kOffP + v * kP + sw128_off(r, c)) =
              make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        fence_proxy_async();
        mbar_arrive(bar(B_PF + v));
      }
      // epilogue: out = O / l, lse = m + ln l
      const int so = (int)(n_out & 1);
      mbar_wait(bar(B_OF + so), (uint32_t)((n_out >> 1) & 1));
      tc_fence_after();
      const bool write = ok && l > 0.f;
      const float inv = write ? 1.f / l : 0.f;
      float* orow = p.out + (t * p.h + j) * kD;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float ov[32];
        tmem_ld32(tmem + lb + kColO + so * 128 + q * 32, ov);
        tmem_wait_ld();
        if (write) {
#pragma unroll
          for (int c = 0; c < 32; c += 4)
            *reinterpret_cast<float4*>(orow + q * 32 + c) =
                make_float4(ov[c] * inv, ov[c + 1] * inv, ov[c + 2] * inv, ov[c + 3] * inv);
        }
      }
      tc_fence_before();
      mbar_arrive(bar(B_OE + so));
      if (write) p.lse[j * p.N + t] = m_used * p.scale + __logf(l);
      ++n_out;
    }
  }

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

int launch(const Params& p, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_qo_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemBytes);
    attr = true;
  }
  int64_t items = p.h_K * p.n_tiles_tok;
  int grid = num_sms();
  if (items < grid) grid = (int)items;
  if (grid < 1) return FSA_OK;
  tc_qo_fwd_kernel<<<grid, kThreads, kSmemBytes, st>>>(p);
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
  p.n_tiles_tok = (p.N + p.tpi - 1) / p.tpi;
  p.scale = (float)s->scale;
  p.scale_log2 = (float)(s->scale * 1.4426950408889634);
  return p;
}

}  // namespace

bool tc_qo_supported(const fsa_shape& s, int dtype) {
  return dtype == FSA_DT_BF16 && s.d_K == kD && s.d_V == kD && s.h_K > 0 && s.h % s.h_K == 0 &&
         s.h / s.h_K <= kRows;
}
bool tc_cmp_scores_fused(const fsa_shape& s) {
  const int64_t g = s.h / s.h_K;
  return g <= 32 && (32 % g) == 0;
}

int tc_slide_fwd(const fsa_shape* s, const void* Q, const void* K, const void* V, void* out,
                 void* lse, cudaStream_t st) {
  Params p = base_params(s);
  p.mode = SLIDE;
  p.Q = (const __nv_bfloat16*)Q;
  p.Kx = (const __nv_bfloat16*)K;
  p.Vx = (const __nv_bfloat16*)V;
  p.n_keys = s->N;
  p.out = (float*)out;
  p.lse = (float*)lse;
  p.scores = nullptr;
  launch(p, st);
  FSA_LAUNCH_CHECK("tc_slide_fwd");
  return FSA_OK;
}

size_t tc_cmp_workspace_bytes(const fsa_shape* s) {
  return (size_t)2 * (s->N / s->B_K) * s->h_K * kD * sizeof(__nv_bfloat16);
}

int tc_cmp_fwd(const fsa_shape* s, const void* Q, const void* Kc, const void* Vc, void* out,
               void* lse, void* scores, void* workspace, cudaStream_t st) {
  Params p = base_params(s);
  p.mode = CMP;
  const int64_t n = p.b * p.h_K * kD;
  __nv_bfloat16* kb = (__nv_bfloat16*)workspace;
  __nv_bfloat16* vb = kb + n;
  to_bf16_kernel<<<148, 256, 0, st>>>((const float*)Kc, kb, n);
  to_bf16_kernel<<<148, 256, 0, st>>>((const float*)Vc, vb, n);
  p.Q = (const __nv_bfloat16*)Q;
  p.Kx = kb;
  p.Vx = vb;
  p.n_keys = p.b;
  p.out = (float*)out;
  p.lse = (float*)lse;
  p.scores = (float*)scores;
  launch(p, st);
  FSA_LAUNCH_CHECK("tc_cmp_fwd");
  return FSA_OK;
}

}  // namespace fsa
