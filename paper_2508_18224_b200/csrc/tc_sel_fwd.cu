// FSA selected-attention forward on tcgen05 tensor cores (K5), bf16, d = 128,
// B_K = 64.  Replaces kv_major.py:152-204 / _core.pyx:49-94 for the
// BASELINE.json shapes, in the fused LOCAL mode: per gathered
// (token, head) row it writes O_i / l_i (bf16) and (m_i, l_i) for block i into
// the slot-indexed partial buffer that the merge kernel (K6) combines.
//
// Persistent, warp-specialised, one CTA per SM:
//   warps 0-3  softmax + epilogue, one TMEM lane (= MMA row) per thread
//   warps 4-7  loaders: cp.async gather of the 128 query rows of an item
//              (tokens x group heads) and, on a task change, the K_i / V_i block
//   warp  8    MMA issuer (one thread): S = Q K^T (M128 N64 K128) and
//              O = P V (M128 N128 K64) into TMEM, tcgen05.commit -> mbarriers
// Stages: Q, P, S, O double-buffered; K/V double-buffered per task.  The
// epilogue of item n-1 overlaps the PV MMA of item n and the S MMA of n+1.
//
// Work: the inverse build's plan (include/fsa_b200.h, fsa_build_inverse) lists
// items of <= 128 rows, heavy blocks first; CTA c owns the contiguous item
// range [c W / G, (c+1) W / G), so consecutive items share K_i / V_i.
#include "tc_common.cuh"
#include "tc_plan.cuh"

namespace fsa {
namespace {

using namespace tc;

constexpr int kD = 128, kBK = 64, kRows = 128;
constexpr int kComputeWarps = 4, kLoadWarps = 4;
constexpr int kThreads = (kComputeWarps + kLoadWarps + 1) * 32;  // 288

// shared-memory map (bytes from a 1024-aligned base)
constexpr uint32_t kQBytes = kRows * kD * 2;         // 32768: [2 halves][128 rows][128 B]
constexpr uint32_t kKVBytes = 2 * kBK * kD * 2;      // 32768: K [2][64][128 B], V [2][64][128 B]
constexpr uint32_t kPBytes = kRows * kBK * 2;        // 16384: [128 rows][128 B]
constexpr uint32_t kOStride = 272;                   // padded staging row (bank-conflict free)
constexpr uint32_t kOStageBytes = kComputeWarps * 32 * kOStride;
constexpr uint32_t kOffQ = 0;
constexpr uint32_t kOffKV = kOffQ + 2 * kQBytes;
constexpr uint32_t kOffP = kOffKV + 2 * kKVBytes;
constexpr uint32_t kOffO = kOffP + 2 * kPBytes;
constexpr uint32_t kOffBar = kOffO + kOStageBytes;
constexpr uint32_t kNumBars = 20;
constexpr uint32_t kOffTmem = kOffBar + kNumBars * 8;
constexpr uint32_t kSmemBytes = kOffTmem + 16 + 1024;  // + alignment slack

// barrier indices (x2 stages each)
enum { B_QF = 0, B_QE = 2, B_KVF = 4, B_KVE = 6, B_SF = 8, B_SE = 10, B_PF = 12, B_PE = 14,
       B_OF = 16, B_OE = 18 };

constexpr uint32_t kIdescS = idesc_bf16(128, 64, false, false);
constexpr uint32_t kIdescPV = idesc_bf16(128, 128, false, true);

struct Params {
  const __nv_bfloat16* Q;
  const __nv_bfloat16* K;
  const __nv_bfloat16* V;
  const int32_t* offsets;
  const int32_t* qlist;
  const int32_t* work;
  __nv_bfloat16* obuf;
  float* ml;
  int64_t N, h, h_K, T, b, g;
  int tpi;
  float scale_log2, scale;
};

// Walks the contiguous item range of this CTA; tracks task changes (kseq).
struct Walker {
  const int32_t* work;
  int64_t ntask, task, w, w_end;
  int64_t kseq;
  bool first;
  __device__ void init(const Params& p) {
    work = p.work;
    ntask = p.h_K * p.b;
    const int64_t W = work[ntask];
    const int64_t G = gridDim.x, c = blockIdx.x;
    w = W * c / G;
    w_end = W * (c + 1) / G;
    int64_t lo = 0, hi = ntask - 1;
    while (lo < hi) {  // largest task with work[task] <= w
      const int64_t mid = (lo + hi + 1) >> 1;
      if (work[mid] <= w) lo = mid; else hi = mid - 1;
    }
    task = lo;
    kseq = -1;
    first = true;
  }
  __device__ bool valid() const { return w < w_end; }
  // position on item w; returns true when the task changed (new K/V block)
  __device__ bool settle() {
    bool changed = first;
    while (work[task + 1] <= w) {
      ++task;
      changed = true;
    }
    first = false;
    if (changed) ++kseq;
    return changed;
  }
  __device__ bool last_of_task() const { return w + 1 >= w_end || work[task + 1] <= w + 1; }
  __device__ int64_t chunk() const { return w - work[task]; }
};

struct Item {
  int64_t i, kh, beg, ntok, p0, nrows_tok;
};
__device__ __forceinline__ Item item_of(const Params& p, const Walker& wk) {
  Item it;
  it.i = wk.task / p.h_K;
  it.kh = wk.task % p.h_K;
  const int32_t* off = p.offsets + it.kh * (p.b + 1) + it.i;
  it.beg = off[0];
  it.ntok = off[1] - off[0];
  it.p0 = wk.chunk() * p.tpi;
  it.nrows_tok = min((int64_t)p.tpi, it.ntok - it.p0);
  return it;
}

__global__ void __launch_bounds__(kThreads, 1) tc_sel_fwd_kernel(const Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + kOffBar;
  auto bar = [&](int k) { return bar0 + 8u * (uint32_t)k; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(bar(B_QF + s), 128);
      mbar_init(bar(B_QE + s), 1);
      mbar_init(bar(B_KVF + s), 128);
      mbar_init(bar(B_KVE + s), 1);
      mbar_init(bar(B_SF + s), 1);
      mbar_init(bar(B_SE + s), 128);
      mbar_init(bar(B_PF + s), 128);
      mbar_init(bar(B_PE + s), 1);
      mbar_init(bar(B_OF + s), 1);
      mbar_init(bar(B_OE + s), 128);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(smem_u32(tmem_slot));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= kComputeWarps && warp < kComputeWarps + kLoadWarps) {
    // ------------------------------------------------------------ loaders
    const int r = threadIdx.x - kComputeWarps * 32;  // 0..127
    Walker wk;
    wk.init(p);
    for (int64_t n = 0; wk.valid(); ++n, ++wk.w) {
      const bool newkv = wk.settle();
      const Item it = item_of(p, wk);
      const int s = (int)(n & 1);
      const int kvs = (int)(wk.kseq & 1);
      if (newkv) {
        mbar_wait(bar(B_KVE + kvs), (uint32_t)(((wk.kseq >> 1) & 1) ^ 1));
        const int rr = r & 63;
        const __nv_bfloat16* src = (r < 64 ? p.K : p.V) + ((it.i * kBK + rr) * p.h_K + it.kh) * kD;
        const uint32_t dst = sbase + kOffKV + kvs * kKVBytes + (r < 64 ? 0u : 16384u);
#pragma unroll
        for (int c = 0; c < 16; ++c)
          cp_async16(dst + (c >> 3) * 8192u + sw128_off(rr, c & 7), src + c * 8);
      }
      mbar_wait(bar(B_QE + s), (uint32_t)(((n >> 1) & 1) ^ 1));
      const int64_t k = r / p.g, hh = r % p.g;
      if (k < it.nrows_tok) {
        const int32_t ent = p.qlist[it.kh * p.N * p.T + it.beg + it.p0 + k];
        const int64_t t = ent / p.T;
        const __nv_bfloat16* src = p.Q + (t * p.h + it.kh * p.g + hh) * kD;
        const uint32_t dst = sbase + kOffQ + s * kQBytes;
#pragma unroll
        for (int c = 0; c < 16; ++c)
          cp_async16(dst + (c >> 3) * 16384u + sw128_off(r, c & 7), src + c * 8);
      }
      cp_async_wait_all();
      fence_proxy_async();
      if (newkv) mbar_arrive(bar(B_KVF + kvs));
      mbar_arrive(bar(B_QF + s));
    }
  } else if (warp == kComputeWarps + kLoadWarps) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      Walker ws, wp;  // S runs one item ahead of PV
      ws.init(p);
      wp.init(p);
      const uint32_t tS = tmem, tO = tmem + 128;
      auto issue_S = [&](int64_t n) {
        ws.settle();
        const int s = (int)(n & 1);
        const int kvs = (int)(ws.kseq & 1);
        mbar_wait(bar(B_KVF + kvs), (uint32_t)((ws.kseq >> 1) & 1));
        mbar_wait(bar(B_QF + s), (uint32_t)((n >> 1) & 1));
        mbar_wait(bar(B_SE + s), (uint32_t)(((n >> 1) & 1) ^ 1));
        tc_fence_after();
        fence_proxy_async();
        const uint32_t qa = sbase + kOffQ + s * kQBytes;
        const uint32_t ka = sbase + kOffKV + kvs * kKVBytes;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = desc_kmajor(qa + (k >> 2) * 16384u + (k & 3) * 32u);
          const uint64_t bd = desc_kmajor(ka + (k >> 2) * 8192u + (k & 3) * 32u);
          mma_bf16(tS + s * 64, ad, bd, kIdescS, k > 0);
        }
        mma_commit(bar(B_SF + s));
        mma_commit(bar(B_QE + s));
        ++ws.w;
      };
      int64_t n = 0;
      if (ws.valid()) issue_S(0);
      for (; wp.valid(); ++n, ++wp.w) {
        wp.settle();
        if (ws.valid()) issue_S(n + 1);
        const int s = (int)(n & 1);
        const int kvs = (int)(wp.kseq & 1);
        mbar_wait(bar(B_PF + s), (uint32_t)((n >> 1) & 1));
        mbar_wait(bar(B_OE + s), (uint32_t)(((n >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t pa = sbase + kOffP + s * kPBytes;
        const uint32_t va = sbase + kOffKV + kvs * kKVBytes + 16384u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = desc_kmajor(pa + k * 32u);
          const uint64_t bd = desc_mnmajor(va + k * 2048u, 8192u);
          mma_bf16(tO + s * 128, ad, bd, kIdescPV, k > 0);
        }
        mma_commit(bar(B_OF + s));
        mma_commit(bar(B_PE + s));
        if (wp.last_of_task()) mma_commit(bar(B_KVE + kvs));
      }
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    const int r = threadIdx.x;  // MMA row == TMEM lane
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    unsigned char* ost = smem + kOffO + warp * 32 * kOStride;
    Walker wk;
    wk.init(p);
    // row state carried from item n-1 into its epilogue
    int64_t prow = -1;  // obuf row index of the previous item's row, or -1
    float pm = 0.f, pl = 1.f;
    int64_t n = 0;
    for (;; ++n) {
      const bool have = wk.valid();
      int64_t orow = -1;
      float mrow = 0.f, lrow = 1.f;
      if (have) {
        wk.settle();
        const Item it = item_of(p, wk);
        const int s = (int)(n & 1);
        const int64_t k = r / p.g, hh = r % p.g;
        int vis = kBK;
        if (k < it.nrows_tok) {
          const int32_t ent = p.qlist[it.kh * p.N * p.T + it.beg + it.p0 + k];
          const int64_t t = ent / p.T, slot = ent % p.T;
          const int64_t j = it.kh * p.g + hh;
          orow = (j * p.N + t) * p.T + slot;
          const int64_t v = t - it.i * kBK + 1;
          vis = v < kBK ? (int)v : kBK;
        }
        mbar_wait(bar(B_SF + s), (uint32_t)((n >> 1) & 1));
        tc_fence_after();
        float sv[64];
        tmem_ld32(tmem + lane_base + s * 64, sv);
        tmem_ld32(tmem + lane_base + s * 64 + 32, sv + 32);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(bar(B_SE + s));
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c < vis) mx = fmaxf(mx, sv[c]);
        if (orow < 0) mx = 0.f;
        const float mb = mx * p.scale_log2;
        float sum = 0.f;
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float e0 = (c < vis && orow >= 0) ? ex2(fmaf(sv[c], p.scale_log2, -mb)) : 0.f;
          const float e1 = (c + 1 < vis && orow >= 0) ? ex2(fmaf(sv[c + 1], p.scale_log2, -mb)) : 0.f;
          sum += e0 + e1;
          pk[c >> 1] = pack_bf16(e0, e1);
        }
        mrow = mx * p.scale;
        lrow = sum;
        mbar_wait(bar(B_PE + s), (uint32_t)(((n >> 1) & 1) ^ 1));
        unsigned char* prow_s = smem + kOffP + s * kPBytes;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 v4 = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          *reinterpret_cast<uint4*>(prow_s + sw128_off(r, c)) = v4;
        }
        fence_proxy_async();
        mbar_arrive(bar(B_PF + s));
      }
      if (n > 0) {
        // epilogue of item n-1: O / l -> bf16 staging -> coalesced global rows
        const int64_t m1 = n - 1;
        const int s1 = (int)(m1 & 1);
        mbar_wait(bar(B_OF + s1), (uint32_t)((m1 >> 1) & 1));
        tc_fence_after();
        const float inv = 1.f / pl;
        unsigned char* mine = ost + lane * kOStride;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float ov[32];
          tmem_ld32(tmem + lane_base + 128 + s1 * 128 + q * 32, ov);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint4 v4 = make_uint4(pack_bf16(ov[8 * c] * inv, ov[8 * c + 1] * inv),
                                  pack_bf16(ov[8 * c + 2] * inv, ov[8 * c + 3] * inv),
                                  pack_bf16(ov[8 * c + 4] * inv, ov[8 * c + 5] * inv),
                                  pack_bf16(ov[8 * c + 6] * inv, ov[8 * c + 7] * inv));
            *reinterpret_cast<uint4*>(mine + q * 64 + c * 16) = v4;
          }
        }
        tc_fence_before();
        mbar_arrive(bar(B_OE + s1));
        if (prow >= 0) *reinterpret_cast<float2*>(p.ml + 2 * prow) = make_float2(pm, pl);
        __syncwarp();
        // 32 rows x 256 B: two rows per warp instruction, 16 B per lane
#pragma unroll 4
        for (int it2 = 0; it2 < 16; ++it2) {
          const int rr = it2 * 2 + (lane >> 4), ch = lane & 15;
          const int64_t dst_row = __shfl_sync(0xffffffffu, prow, rr);
          const uint4 v4 = *reinterpret_cast<const uint4*>(ost + rr * kOStride + ch * 16);
          if (dst_row >= 0)
            *reinterpret_cast<uint4*>(p.obuf + dst_row * kD + ch * 8) = v4;
        }
        __syncwarp();
      }
      if (!have) break;
      prow = orow;
      pm = mrow;
      pl = lrow;
      ++wk.w;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

bool tc_fwd_supported(const fsa_shape& s, int dtype) {
  return dtype == FSA_DT_BF16 && s.d_K == kD && s.d_V == kD && s.B_K == kBK && s.h_K > 0 &&
         s.h % s.h_K == 0 && s.h / s.h_K <= kRows;
}

int tc_sel_fwd(const fsa_shape* s, const void* Q, const void* K, const void* V,
               const int32_t* offsets, const int32_t* qlist, const int32_t* work, void* obuf,
               void* ml, cudaStream_t st) {
  FSA_REQUIRE(work != nullptr, "tensor-core forward needs the inverse work plan");
  Params p;
  p.Q = (const __nv_bfloat16*)Q;
  p.K = (const __nv_bfloat16*)K;
  p.V = (const __nv_bfloat16*)V;
  p.offsets = offsets;
  p.qlist = qlist;
  p.work = work;
  p.obuf = (__nv_bfloat16*)obuf;
  p.ml = (float*)ml;
  p.N = s->N;
  p.h = s->h;
  p.h_K = s->h_K;
  p.T = s->T;
  p.b = s->N / s->B_K;
  p.g = s->h / s->h_K;
  p.tpi = (int)(kRows / p.g);
  p.scale = (float)s->scale;
  p.scale_log2 = (float)(s->scale * 1.4426950408889634);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc_sel_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemBytes);
    attr = true;
  }
  tc_sel_fwd_kernel<<<num_sms(), kThreads, kSmemBytes, st>>>(p);
  FSA_LAUNCH_CHECK("tc_sel_fwd");
  return FSA_OK;
}

}  // namespace fsa
