// NSA query-major selected-attention forward on tcgen05 (the paper's
// baseline schedule, query_major.py:45-69, _core.pyx:134-181), bf16, d = 128,
// B_K = 64: one task per (kv head, token) batches the group's g query heads,
// padded to NP = max(g, min_tile) rounded up to 8 (the reference meter's
// min_tile padding, query_major.py:32-42), and walks the token's selected
// blocks; the own (partially causal) block is loaded in full and masked by
// position.
//
// On the tensor cores the g rows sit on the MMA's N side, the keys on M:
//   S^T  = K_pair Q_t^T   M128 (two 64-key blocks) x N NP x K128   (bf16)
//   O^T += V16_pair^T P^T M128 (features) x N NP x K128 (keys)     (fp16)
// so a (token, pair of blocks) costs two MMA groups of 8 K-steps whatever g
// is, and every pair reloads its 32 KB K/V tile from L2 -- the per-token
// K/V traffic FSA's KV-block-major order amortises over all attending tokens.
// The softmax is exact in two passes over the token's S^T tiles (all held in
// TMEM): per-head max, then P = exp(S - m) and the per-head sums, reduced
// across the 128 key lanes through shared memory.
//
// Roles: warps 0-3 softmax + epilogue (thread = TMEM lane = key within the
// pair, then = feature in the epilogue), warp 4 TMA producer, warp 5 MMA
// issuer.  Units u = (kh, t) kv-head-major, round-robin over the CTAs; the
// producer and the MMA thread run the tile stream K(0), then per unit
// [K(u+1), V(u)], so S of the next token overlaps the softmax of this one.
#include "tc_plan.cuh"
#include "tc_sched.cuh"

namespace fsa {
namespace {

using namespace tc;

constexpr int kD = 128, kBK = 64;
constexpr int kThreads = 6 * 32;
constexpr int kStages = 4;
constexpr int kMaxPairs = 8;                  // T <= 16 (P^T tiles of a unit in smem)
constexpr uint32_t kTile = 32768;             // [2 halves][128 keys][128 B]
constexpr uint32_t kOffKV = 0;
constexpr uint32_t kOffQ = kStages * kTile;   // [2 units][2 halves][16 rows][128 B]
constexpr uint32_t kQBytes = 4096;
constexpr uint32_t kOffP = kOffQ + 2 * kQBytes;  // P^T [2 units][pairs][2 halves][16 rows][128 B]
constexpr uint32_t kPBytes = 4096;               // one pair, NP <= 16 rows
constexpr uint32_t kOffRed = kOffP + 2 * kMaxPairs * kPBytes;  // [4 warps][16] floats
constexpr uint32_t kOffBar = kOffRed + 2 * 4 * 16 * 4;
enum { B_F = 0, B_E = 4, B_QF = 8, B_QE = 10, B_SF = 12, B_SE = 14, B_PF = 16, B_PE = 18,
       B_OF = 20, B_OE = 22, kNumBars = 24 };
constexpr uint32_t kOffTmem = kOffBar + kNumBars * 8;
constexpr uint32_t kSmemBytes = kOffTmem + 16 + 1024;
static_assert(kSmemBytes <= 232448, "shared memory budget");
// TMEM: S^T of unit parity v at 256 v + NP p (p < pairs), O^T at 256 v + 240
constexpr uint32_t kColO = 240;

struct Params {
  CUtensorMap tmQ, tmK, tmV;
  const int32_t* idx;
  const float* vscale;
  float *out, *lse;
  int N, h, h_K, g, T, NP, units;
  float scale, scale_log2;
};

// the unit's selected blocks (ascending, -1 padded) and their count
__device__ __forceinline__ int unit_blocks(const Params& p, int u, int kh, int t, int* blk) {
  const int32_t* row = p.idx + ((int64_t)kh * p.N + t) * p.T;
  int n = 0;
  for (int s = 0; s < p.T; ++s) {
    const int b = __ldg(row + s);
    if (b < 0) break;
    blk[n++] = b;
  }
  return n;
}

template <int NP>
__device__ __forceinline__ void tmem_ldn(uint32_t taddr, float* v) {
  if constexpr (NP == 16) {
    tmem_ld16(taddr, v);
  } else {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
  }
}

template <int NP>
__global__ void __launch_bounds__(kThreads, 1) tc_qm_fwd_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sb = smem_u32(smem);
  auto bar = [&](int k) { return sb + kOffBar + 8u * (uint32_t)k; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = (int)gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(bar(B_F + s), 1);
      mbar_init(bar(B_E + s), 1);
    }
    for (int v = 0; v < 2; ++v) {
      mbar_init(bar(B_QF + v), 1);
      mbar_init(bar(B_QE + v), 1);
      mbar_init(bar(B_SF + v), 1);
      mbar_init(bar(B_SE + v), 128);
      mbar_init(bar(B_PF + v), 128);
      mbar_init(bar(B_PE + v), 1);
      mbar_init(bar(B_OF + v), 1);
      mbar_init(bar(B_OE + v), 128);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t kIdS = idesc_bf16(128, NP, false, false);
  constexpr uint32_t kIdPV = idesc_f16(128, NP, true, false);

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int r = 0;  // tile-stream position (stage ring)
      auto load_pairs = [&](int kh, const int* blk, int n, const CUtensorMap* map) {
        for (int q = 0; q < (n + 1) / 2; ++q, ++r) {
          const int s = r % kStages;
          mbar_wait(bar(B_E + s), (uint32_t)(((r / kStages) & 1) ^ 1));
          mbar_arrive_expect_tx(bar(B_F + s), kTile);
          const int b0 = blk[2 * q], b1 = 2 * q + 1 < n ? blk[2 * q + 1] : b0;  // odd: repeat, masked
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            tma_load_3d(sb + kOffKV + s * kTile + hf * 16384u, map, hf * 64, kh, b0 * kBK, bar(B_F + s));
            tma_load_3d(sb + kOffKV + s * kTile + hf * 16384u + 8192u, map, hf * 64, kh, b1 * kBK,
                        bar(B_F + s));
          }
        }
      };
      int blk[2][32], nb[2] = {0, 0};
      int j = 0;
      for (int u = blockIdx.x; u < p.units; u += G, ++j) {
        const int kh = u / p.N, t = u % p.N;
        const int v = j & 1;
        nb[v] = unit_blocks(p, u, kh, t, blk[v]);
        // q rows of the unit (B operand of S^T): g rows x 128 features
        mbar_wait(bar(B_QE + v), (uint32_t)(((j >> 1) & 1) ^ 1));
        mbar_arrive_expect_tx(bar(B_QF + v), 2u * (uint32_t)p.g * 128u);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf)
          tma_load_3d(sb + kOffQ + v * kQBytes + hf * 2048u, &p.tmQ, hf * 64, kh * p.g, t, bar(B_QF + v));
        load_pairs(kh, blk[v], nb[v], &p.tmK);  // K(j)
        if (j > 0) {                             // V(j - 1)
          const int up = u - G;
          load_pairs(up / p.N, blk[v ^ 1], nb[v ^ 1], &p.tmV);
        }
      }
      if (j > 0) {
        const int up = (int)blockIdx.x + (j - 1) * G;
        load_pairs(up / p.N, blk[(j - 1) & 1], nb[(j - 1) & 1], &p.tmV);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    int r = 0;
    int nb[2] = {0, 0};
    auto s_mma = [&](int j, int n) {
      const int v = j & 1;
      mbar_wait_warp(bar(B_QF + v), (uint32_t)((j >> 1) & 1));
      mbar_wait_warp(bar(B_SE + v), (uint32_t)(((j >> 1) & 1) ^ 1));
      const uint32_t q = sb + kOffQ + v * kQBytes;
      for (int pr = 0; pr < (n + 1) / 2; ++pr, ++r) {
        const int s = r % kStages;
        mbar_wait_warp(bar(B_F + s), (uint32_t)((r / kStages) & 1));
        tc_fence_after();
        const uint32_t k = sb + kOffKV + s * kTile;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_bf16(tmem + 256u * v + (uint32_t)(NP * pr), desc_kmajor(k + (kk >> 2) * 16384u + (kk & 3) * 32u),
                     desc_kmajor(q + (kk >> 2) * 2048u + (kk & 3) * 32u), kIdS, kk > 0);
          mma_commit(bar(B_E + s));
        }
        __syncwarp();
      }
      if (elect_one()) {
        mma_commit(bar(B_SF + v));
        mma_commit(bar(B_QE + v));
      }
      __syncwarp();
    };
    auto pv_mma = [&](int j, int n) {
      const int v = j & 1;
      mbar_wait_warp(bar(B_PF + v), (uint32_t)((j >> 1) & 1));
      mbar_wait_warp(bar(B_OE + v), (uint32_t)(((j >> 1) & 1) ^ 1));
      for (int pr = 0; pr < (n + 1) / 2; ++pr, ++r) {
        const int s = r % kStages;
        mbar_wait_warp(bar(B_F + s), (uint32_t)((r / kStages) & 1));
        tc_fence_after();
        const uint32_t vt = sb + kOffKV + s * kTile;
        const uint32_t pt = sb + kOffP + (uint32_t)(v * kMaxPairs + pr) * kPBytes;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_bf16(tmem + 256u * v + kColO, desc_mnmajor(vt + kk * 2048u, 16384u),
                     desc_kmajor(pt + (kk >> 2) * 2048u + (kk & 3) * 32u), kIdPV,
                     (pr > 0 || kk > 0) ? 1u : 0u);
          mma_commit(bar(B_E + s));
        }
        __syncwarp();
      }
      if (elect_one()) {
        mma_commit(bar(B_OF + v));
        mma_commit(bar(B_PE + v));
      }
      __syncwarp();
    };
    int j = 0;
    for (int u = blockIdx.x; u < p.units; u += G, ++j) {
      int blk[32];
      nb[j & 1] = unit_blocks(p, u, u / p.N, u % p.N, blk);
      s_mma(j, nb[j & 1]);
      if (j > 0) pv_mma(j - 1, nb[(j - 1) & 1]);
    }
    if (j > 0) pv_mma(j - 1, nb[(j - 1) & 1]);
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    const int r = threadIdx.x;  // TMEM lane: key within the pair; feature in the epilogue
    const uint32_t lb = (uint32_t)(warp * 32) << 16;
    float* red = reinterpret_cast<float*>(smem + kOffRed);  // [2][4 warps][16]
    int pend_u = -1, pend_j = 0;
    float pm[NP], pl[NP];
    auto epilogue = [&](int u, int j) {
      const int v = j & 1, kh = u / p.N, t = u % p.N;
      mbar_wait(bar(B_OF + v), (uint32_t)((j >> 1) & 1));
      tc_fence_after();
      float o[NP];
      tmem_ldn<NP>(tmem + lb + 256u * v + kColO, o);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(bar(B_OE + v));
      const float vs = 1.f / __ldg(p.vscale + kh);
#pragma unroll
      for (int hh = 0; hh < NP; ++hh) {
        if (hh < p.g) {
          const int64_t j2 = (int64_t)kh * p.g + hh;
          p.out[(((int64_t)t * p.h) + j2) * kD + r] = o[hh] * vs / pl[hh];
          if (r == 0) p.lse[j2 * p.N + t] = pm[hh] * p.scale + __logf(pl[hh]);
        }
      }
    };
    int j = 0;
    for (int u = blockIdx.x; u < p.units; u += G, ++j) {
      const int v = j & 1, kh = u / p.N, t = u % p.N;
      int blk[32];
      const int n = unit_blocks(p, u, kh, t, blk);
      const int npair = (n + 1) / 2;
      mbar_wait(bar(B_SF + v), (uint32_t)((j >> 1) & 1));
      tc_fence_after();
      // pass 1: per-head max over the visible keys
      float m[NP];
#pragma unroll
      for (int hh = 0; hh < NP; ++hh) m[hh] = -INFINITY;
      for (int pr = 0; pr < npair; ++pr) {
        const int b = (r < 64) ? blk[2 * pr] : (2 * pr + 1 < n ? blk[2 * pr + 1] : -1);
        const bool vis = b >= 0 && b * kBK + (r & 63) <= t;
        float sv[NP];
        tmem_ldn<NP>(tmem + lb + 256u * v + (uint32_t)(NP * pr), sv);
        tmem_wait_ld();
#pragma unroll
        for (int hh = 0; hh < NP; ++hh) m[hh] = vis ? fmaxf(m[hh], sv[hh]) : m[hh];
      }
#pragma unroll
      for (int hh = 0; hh < NP; ++hh) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m[hh] = fmaxf(m[hh], __shfl_xor_sync(0xffffffffu, m[hh], o));
      }
      float* rv = red + v * 64;
      if (lane == 0) {
#pragma unroll
        for (int hh = 0; hh < NP; ++hh) rv[warp * 16 + hh] = m[hh];
      }
      named_bar(1, 128);
#pragma unroll
      for (int hh = 0; hh < NP; ++hh)
        m[hh] = fmaxf(fmaxf(rv[hh], rv[16 + hh]), fmaxf(rv[32 + hh], rv[48 + hh]));
      // the P^T buffer of this parity: PV of unit j - 2 has read it
      mbar_wait(bar(B_PE + v), (uint32_t)(((j >> 1) & 1) ^ 1));
      // pass 2: P = exp(S - m) (fp16, K-major rows = heads), per-head sums
      float l[NP];
#pragma unroll
      for (int hh = 0; hh < NP; ++hh) l[hh] = 0.f;
      for (int pr = 0; pr < npair; ++pr) {
        const int b = (r < 64) ? blk[2 * pr] : (2 * pr + 1 < n ? blk[2 * pr + 1] : -1);
        const bool vis = b >= 0 && b * kBK + (r & 63) <= t;
        float sv[NP];
        tmem_ldn<NP>(tmem + lb + 256u * v + (uint32_t)(NP * pr), sv);
        tmem_wait_ld();
        unsigned char* pt = smem + kOffP + (uint32_t)(v * kMaxPairs + pr) * kPBytes;
        const uint32_t half = (uint32_t)(r >> 6) * 2048u, ch = (uint32_t)((r & 63) >> 3);
#pragma unroll
        for (int hh = 0; hh < NP; ++hh) {
          const float e = (vis && hh < p.g) ? ex2((sv[hh] - m[hh]) * p.scale_log2) : 0.f;
          l[hh] += e;
          *reinterpret_cast<__half*>(pt + half + sw128_off((uint32_t)hh, ch) + (uint32_t)(r & 7) * 2u) =
              __float2half_rn(e);
        }
      }
      tc_fence_before();
      mbar_arrive(bar(B_SE + v));  // S^T read: the MMA may write the next unit of this parity
#pragma unroll
      for (int hh = 0; hh < NP; ++hh) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], o);
      }
      named_bar(1, 128);  // everyone has read the maxima
      if (lane == 0) {
#pragma unroll
        for (int hh = 0; hh < NP; ++hh) rv[warp * 16 + hh] = l[hh];
      }
      fence_proxy_async();
      mbar_arrive(bar(B_PF + v));
      named_bar(1, 128);
      float lt[NP];
#pragma unroll
      for (int hh = 0; hh < NP; ++hh) lt[hh] = (rv[hh] + rv[16 + hh]) + (rv[32 + hh] + rv[48 + hh]);
      // the previous unit's epilogue overlaps this unit's P.V
      if (pend_u >= 0) epilogue(pend_u, pend_j);
#pragma unroll
      for (int hh = 0; hh < NP; ++hh) {
        pm[hh] = m[hh];
        pl[hh] = lt[hh];
      }
      pend_u = u;
      pend_j = j;
      named_bar(1, 128);  // the reduction buffer of this parity is free again
    }
    if (pend_u >= 0) epilogue(pend_u, pend_j);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

bool tc_qm_supported(const fsa_shape& s, int dtype) {
  const int64_t g = s.h_K > 0 ? s.h / s.h_K : 0;
  return dtype == FSA_DT_BF16 && s.d_K == kD && s.d_V == kD && s.B_K == kBK && s.h_K > 0 &&
         s.h % s.h_K == 0 && g >= 1 && g <= 16 && s.T <= 2 * kMaxPairs &&
         (s.T + 1) / 2 * (g <= 8 ? 8 : 16) <= (int64_t)kColO && s.N * s.h_K < (1ll << 31);
}

int tc_qm_fwd(const fsa_shape* s, const void* Q, const void* K, const void* V16,
              const float* vscale, const int32_t* idx, void* out, void* lse, int min_tile,
              cudaStream_t st) {
  FSA_REQUIRE(tc_qm_supported(*s, FSA_DT_BF16), "qm_fwd_tc: bf16, d = 128, B_K = 64, g <= 16, T <= 16");
  Params p{};
  p.idx = idx;
  p.vscale = vscale;
  p.out = (float*)out;
  p.lse = (float*)lse;
  p.N = (int)s->N;
  p.h = (int)s->h;
  p.h_K = (int)s->h_K;
  p.g = (int)(s->h / s->h_K);
  p.T = (int)s->T;
  const int pad = p.g > min_tile ? p.g : min_tile;
  FSA_REQUIRE(pad <= 16, "qm_fwd_tc: max(g, min_tile) = %d > 16", pad);
  p.NP = pad <= 8 ? 8 : 16;
  FSA_REQUIRE((s->T + 1) / 2 * p.NP <= (int64_t)kColO, "qm_fwd_tc: T = %lld too large for the TMEM tiles",
              (long long)s->T);
  p.units = (int)(s->h_K * s->N);
  p.scale = (float)s->scale;
  p.scale_log2 = (float)(s->scale * 1.4426950408889634);
  int rc = make_tmap_tokens(&p.tmQ, Q, s->N, s->h, p.g, 1);
  if (!rc) rc = make_tmap_tokens(&p.tmK, K, s->N, s->h_K, 1, 64);
  if (!rc) rc = make_tmap_tokens(&p.tmV, V16, s->N, s->h_K, 1, 64);
  if (rc) return rc;
  if (p.units == 0) return FSA_OK;
  int grid = num_sms();
  if (grid > p.units) grid = p.units;
  static unsigned long long done[2] = {0, 0};
  if (p.NP == 8) {
    ensure_smem_attr(tc_qm_fwd_kernel<8>, (int)kSmemBytes, done[0]);
    tc_qm_fwd_kernel<8><<<grid, kThreads, kSmemBytes, st>>>(p);
  } else {
    ensure_smem_attr(tc_qm_fwd_kernel<16>, (int)kSmemBytes, done[1]);
    tc_qm_fwd_kernel<16><<<grid, kThreads, kSmemBytes, st>>>(p);
  }
  FSA_LAUNCH_CHECK("tc_qm_fwd");
  return FSA_OK;
}

}  // namespace fsa

extern "C" int fsa_qm_fwd_tc(const fsa_shape* s, const void* Q, const void* K, const void* V16,
                             const float* vscale, const int32_t* idx, void* out, void* lse,
                             int min_tile, void* stream) {
  return fsa::tc_qm_fwd(s, Q, K, V16, vscale, idx, out, lse, min_tile, (cudaStream_t)stream);
}
