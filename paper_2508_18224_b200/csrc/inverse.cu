// K4 build_inverse_index (selection.py:146-169) as a deterministic, stable
// counting sort -- no atomics decide any order.
//
//   count   : per (kv head, 256-token tile) histogram over blocks, with the
//             selection validity flags (selection.py:49-75) fused in;
//   scan    : per (kv head, block) exclusive scan over tiles -> tile bases;
//   offsets : per kv head exclusive scan over blocks -> CSR offsets;
//   scatter : each (token, slot) entry lands at
//             offsets[e] + tile_base[tile][e] + rank-within-tile,
//             where the in-tile rank is computed in token order (warps take
//             turns; lanes of a warp rank through a shared-memory lane mask).
// Queries inside each block therefore come out in ascending token order, the
// reference's canonical order, independent of scheduling.
#include <cstdlib>

#include "common.cuh"

namespace fsa {

constexpr int kInvTile = 256;  // tokens per CTA (8 warps x 32)

__device__ __forceinline__ bool live_entry(int e, int64_t own) { return e >= 0 && e <= own; }

__device__ __forceinline__ int row_flags(const int32_t* r, int T, int64_t own, int64_t b) {
  int f = 0;
  int prev = r[0];
  bool prev_live = prev != -1;
  if (!prev_live) f |= FSA_SEL_EMPTY_ROW;
  if ((prev < 0 && prev != -1) || prev >= b) f |= FSA_SEL_OUT_OF_RANGE;
  if (prev_live && prev > own) f |= FSA_SEL_NON_CAUSAL;
  for (int k = 1; k < T; ++k) {
    const int v = r[k];
    const bool live = v != -1;
    if (live && !prev_live) f |= FSA_SEL_AFTER_SENTINEL;
    if ((v < 0 && v != -1) || v >= b) f |= FSA_SEL_OUT_OF_RANGE;
    if (live && v > own) f |= FSA_SEL_NON_CAUSAL;
    if (live && prev_live) {
      if (v == prev) f |= FSA_SEL_DUPLICATE;
      if (v < prev) f |= FSA_SEL_NOT_INCREASING;
    }
    prev = v;
    prev_live = live;
  }
  return f;
}

// kScatter = false: histogram + flags.  kScatter = true: write qlist.
template <bool kScatter>
__global__ void __launch_bounds__(kInvTile)
inverse_tile_kernel(const int32_t* __restrict__ idx, int64_t N, int64_t B_K, int64_t b, int T,
                    int32_t* __restrict__ hist, const int32_t* __restrict__ offsets,
                    int32_t* __restrict__ qlist, int32_t* flags, int32_t* __restrict__ pos,
                    int64_t ctiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem_raw);  // [b]
  int32_t* cnt = reinterpret_cast<int32_t*>(mask + b);     // [b]
  const int64_t kh = blockIdx.y, tile = blockIdx.x, n_tiles = gridDim.x;
  const int64_t t0 = tile * kInvTile;
  for (int64_t e = threadIdx.x; e < b; e += blockDim.x) {
    mask[e] = 0;
    cnt[e] = 0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t = t0 + threadIdx.x;
  const bool has_row = t < N;
  const int64_t own = has_row ? t / B_K : -1;
  const int32_t* row = idx + (kh * N + (has_row ? t : 0)) * T;
  if (!kScatter && flags) {
    int f = has_row ? row_flags(row, T, own, b) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f |= __shfl_xor_sync(0xffffffffu, f, o);
    if (lane == 0 && f) atomicOr(flags, f);
  }
  const unsigned lt = lanemask_lt();
  int32_t* ql = kScatter ? qlist + kh * N * T : nullptr;
  const int32_t* off = kScatter ? offsets + kh * (b + 1) : nullptr;
  const int32_t* base = kScatter ? hist + (kh * n_tiles + tile) * b : nullptr;
  // the work plan's positions are relative to the token chunk's sub-list
  const int32_t* cbase = kScatter ? hist + (kh * n_tiles + tile / ctiles * ctiles) * b : nullptr;
  __syncthreads();
  for (int w = 0; w < kInvTile / 32; ++w) {
    if (warp == w && has_row) {
      const unsigned me = 1u << lane;
      for (int s = 0; s < T; ++s) {
        const int e = row[s];
        if (live_entry(e, own)) atomicOr(&mask[e], me);
      }
    }
    __syncwarp();
    if (warp == w && has_row && kScatter) {
      for (int s = 0; s < T; ++s) {
        const int e = row[s];
        if (!live_entry(e, own)) continue;
        const int rank = cnt[e] + __popc(mask[e] & lt);
        ql[off[e] + base[e] + rank] = (int32_t)(t * T + s);
        if (pos) pos[(kh * N + t) * T + s] = base[e] + rank - cbase[e];
      }
    }
    __syncwarp();
    if (warp == w && has_row) {  // the lowest lane owning e publishes the warp's count
      for (int s = 0; s < T; ++s) {
        const int e = row[s];
        if (!live_entry(e, own)) continue;
        const uint32_t m = mask[e];
        if (lane == __ffs(m) - 1) cnt[e] += __popc(m);
      }
    }
    __syncwarp();
    if (warp == w && has_row) {
      for (int s = 0; s < T; ++s) {
        const int e = row[s];
        if (live_entry(e, own)) mask[e] = 0;
      }
    }
    __syncthreads();
  }
  if (!kScatter) {
    int32_t* h = hist + (kh * n_tiles + tile) * b;
    for (int64_t e = threadIdx.x; e < b; e += blockDim.x) h[e] = cnt[e];
  }
}

// Same contract, one pass instead of 8 warp turns: a 256-bit token mask per
// block in shared memory ([b][8] words, word w = warp w's lanes), set with one
// atomicOr per live entry; after one barrier the in-tile rank of (t, e) is the
// popcount of e's mask below t (token order) and a block's count is its total.
template <bool kScatter>
__global__ void __launch_bounds__(kInvTile)
inverse_tile_bits_kernel(const int32_t* __restrict__ idx, int64_t N, int64_t B_K, int64_t b, int T,
                         int32_t* __restrict__ hist, const int32_t* __restrict__ offsets,
                         int32_t* __restrict__ qlist, int32_t* flags, int32_t* __restrict__ pos,
                         int64_t ctiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem_raw);  // [b][8]
  const int kh = blockIdx.y, tile = blockIdx.x, n_tiles = gridDim.x;
  const int t0 = tile * kInvTile;
  for (int e = threadIdx.x; e < 8 * (int)b; e += blockDim.x) mask[e] = 0u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = t0 + threadIdx.x;
  const bool has_row = t < (int)N;
  const int own = has_row ? t / (int)B_K : -1;
  const int32_t* row = idx + ((int64_t)kh * N + (has_row ? t : 0)) * T;
  if (!kScatter && flags) {
    int f = has_row ? row_flags(row, T, own, b) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f |= __shfl_xor_sync(0xffffffffu, f, o);
    if (lane == 0 && f) atomicOr(flags, f);
  }
  __syncthreads();
  if (has_row) {
    for (int s = 0; s < T; ++s) {
      const int e = row[s];
      if (live_entry(e, own)) atomicOr(&mask[e * 8 + warp], 1u << lane);
    }
  }
  __syncthreads();
  if (!kScatter) {
    int32_t* h = hist + ((int64_t)kh * n_tiles + tile) * b;
    for (int e = threadIdx.x; e < (int)b; e += blockDim.x) {
      const uint4 a = reinterpret_cast<const uint4*>(mask)[2 * e];
      const uint4 c = reinterpret_cast<const uint4*>(mask)[2 * e + 1];
      h[e] = __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w) + __popc(c.x) + __popc(c.y) +
             __popc(c.z) + __popc(c.w);
    }
  } else if (has_row) {
    int32_t* ql = qlist + (int64_t)kh * N * T;
    const int32_t* off = offsets + (int64_t)kh * (b + 1);
    const int32_t* base = hist + ((int64_t)kh * n_tiles + tile) * b;
    const int32_t* cb = hist + ((int64_t)kh * n_tiles + tile / ctiles * ctiles) * b;
    const unsigned lt = lanemask_lt();
    for (int s = 0; s < T; ++s) {
      const int e = row[s];
      if (!live_entry(e, own)) continue;
      const uint32_t* m = mask + e * 8;
      int rank = __popc(m[warp] & lt);
      for (int w = 0; w < warp; ++w) rank += __popc(m[w]);
      ql[off[e] + base[e] + rank] = (int32_t)(t * T + s);
      if (pos) pos[((int64_t)kh * N + t) * T + s] = base[e] + rank - cb[e];
    }
  }
}

// per (kh, block): exclusive scan over tiles, totals into offsets[kh][e+1]
__global__ void inverse_scan_tiles_kernel(int32_t* __restrict__ hist, int32_t* __restrict__ offsets,
                                          int64_t h_K, int64_t n_tiles, int64_t b) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= h_K * b) return;
  const int64_t kh = id / b, e = id % b;
  int32_t* h = hist + kh * n_tiles * b + e;
  int32_t run = 0;
  int64_t tile = 0;
  for (; tile + 4 <= n_tiles; tile += 4) {
    int32_t v0 = h[(tile + 0) * b], v1 = h[(tile + 1) * b], v2 = h[(tile + 2) * b],
            v3 = h[(tile + 3) * b];
    h[(tile + 0) * b] = run; run += v0;
    h[(tile + 1) * b] = run; run += v1;
    h[(tile + 2) * b] = run; run += v2;
    h[(tile + 3) * b] = run; run += v3;
  }
  for (; tile < n_tiles; ++tile) {
    int32_t v = h[tile * b];
    h[tile * b] = run;
    run += v;
  }
  offsets[kh * (b + 1) + e + 1] = run;
}

// per kh: inclusive scan of offsets[kh][1..b]; offsets[kh][0] = 0
__global__ void inverse_scan_blocks_kernel(int32_t* __restrict__ offsets, int64_t b) {
  __shared__ int32_t warp_tot[32];
  __shared__ int32_t carry_s;
  int32_t* o = offsets + blockIdx.x * (b + 1);
  if (threadIdx.x == 0) {
    o[0] = 0;
    carry_s = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t c0 = 0; c0 < b; c0 += blockDim.x) {
    const int64_t e = c0 + threadIdx.x;
    int32_t v = (e < b) ? o[e + 1] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int32_t u = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += u;
    }
    if (lane == 31) warp_tot[warp] = v;
    __syncthreads();
    if (warp == 0) {
      int32_t w = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        int32_t u = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += u;
      }
      if (lane < nw) warp_tot[lane] = w;
    }
    __syncthreads();
    const int32_t carry = carry_s;
    const int32_t prefix = (warp > 0 ? warp_tot[warp - 1] : 0) + carry;
    if (e < b) o[e + 1] = v + prefix;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry_s = v + prefix;
    __syncthreads();
  }
}

// Work plan of the persistent tensor-core kernels (common.cuh): pass 1 (one
// thread per chunked task) derives the task's sub-list from the scanned tile
// histograms -- hist[kh][tile][i] is the list position of tile's first entry
// of block i, so a chunk's sub-list starts at its first tile's value -- and
// scans the item counts inside each CTA; pass 2 adds the CTA carries.
struct PlanArgs {
  const int32_t* offsets;
  const int32_t* hist;
  int32_t* work;
  int32_t *item, *tbeg, *tn, *tki;
  int32_t* carry;  // per pass-1 CTA item totals
  int64_t h_K, b, N, B_K, n_tiles, C, nc, nph, ntask;
  int tpi;
};

__device__ __forceinline__ int64_t bic_of(const PlanArgs& a, int64_t c) {
  const int64_t tend = (c + 1) * a.C < a.N ? (c + 1) * a.C : a.N;
  const int64_t n = (tend - 1) / a.B_K + 1;
  return n < a.b ? n : a.b;
}

__global__ void __launch_bounds__(1024) work_plan_tasks_kernel(PlanArgs a) {
  __shared__ int32_t cb[kPlanMaxChunks + 1];
  __shared__ int32_t warp_tot[32];
  if (threadIdx.x == 0) {
    int32_t run = 0;
    for (int64_t c = 0; c < a.nc; ++c) {
      cb[c] = run;
      run += (int32_t)bic_of(a, c);
    }
    cb[a.nc] = run;
    if (blockIdx.x == 0) {
      a.work[0] = (int32_t)a.C;
      a.work[1] = (int32_t)a.nc;
      a.work[2] = (int32_t)a.nph;
      for (int64_t c = 0; c <= a.nc; ++c) a.work[64 + c] = cb[c];
    }
  }
  __syncthreads();
  const int64_t task = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int32_t v = 0;
  if (task < a.ntask) {
    const int64_t kh = task / a.nph, r = task % a.nph;
    int64_t c = 0;
    while (c + 1 < a.nc && r >= cb[c + 1]) ++c;
    const int64_t i = r - cb[c];
    const int32_t* off = a.offsets + kh * (a.b + 1);
    const int32_t* h = a.hist + kh * a.n_tiles * a.b + i;
    const int64_t ct = a.C / 256;
    const int32_t lo = h[c * ct * a.b];
    const int32_t hi = c + 1 < a.nc ? h[(c + 1) * ct * a.b] : off[i + 1] - off[i];
    a.tbeg[task] = off[i] + lo;
    a.tn[task] = hi - lo;
    a.tki[task] = (int32_t)(kh * a.b + i);
    v = (hi - lo + a.tpi - 1) / a.tpi;
  }
  const int32_t own = v;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t u = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += u;
  }
  if (lane == 31) warp_tot[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int32_t u = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += u;
    }
    if (lane < nw) warp_tot[lane] = w;
  }
  __syncthreads();
  const int32_t incl = v + (warp > 0 ? warp_tot[warp - 1] : 0);
  if (task < a.ntask) a.item[task] = incl - own;
  if (threadIdx.x == blockDim.x - 1) a.carry[blockIdx.x] = incl;
}

__global__ void __launch_bounds__(1024) work_plan_carry_kernel(PlanArgs a) {
  __shared__ int32_t base;
  if (threadIdx.x == 0) {
    int32_t run = 0;
    for (unsigned k = 0; k < blockIdx.x; ++k) run += a.carry[k];
    base = run;
    if (blockIdx.x == gridDim.x - 1) a.item[a.ntask] = run + a.carry[blockIdx.x];
  }
  __syncthreads();
  const int64_t task = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (task < a.ntask) a.item[task] += base;
}

int64_t plan_chunk_tokens(const fsa_shape& s) {
  // Default: one chunk (C = N).  Measured on B200: chunks
  // sized for an L2-resident query working set (16K tokens at Qwen3-14B 128K)
  // cut K5's DRAM reads 11.9 -> 4.9 GB but not its time (HBM writes and the
  // item pipeline bound it), and made K8 slower (17.9 vs 16.5 ms: per-task K/V
  // reloads, short tasks).  FSA_CHUNK_TOKENS overrides it (tests, tuning).
  int64_t C = 0;
  if (const char* e = getenv("FSA_CHUNK_TOKENS")) C = atoll(e);
  const int64_t n = s.N > 0 ? s.N : 1;
  if (C <= 0 || C > n) C = n;
  const int64_t min_c = (n + kPlanMaxChunks - 1) / kPlanMaxChunks;
  if (C < min_c) C = min_c;
  return (C + 255) / 256 * 256;
}

}  // namespace fsa

static int64_t n_tiles_of(const fsa_shape* s) { return (s->N + fsa::kInvTile - 1) / fsa::kInvTile; }

extern "C" size_t fsa_work_plan_bytes(const fsa_shape* s) {
  return (size_t)(fsa::plan_pos_offset(*s) + s->h_K * s->N * s->T) * sizeof(int32_t);
}

static int64_t plan_ctas(const fsa_shape* s) { return (fsa::plan_ntask(*s) + 1023) / 1024; }

extern "C" size_t fsa_inverse_workspace_bytes(const fsa_shape* s) {
  const int64_t b = s->N / s->B_K;
  // tile histograms, then the work plan's per-CTA carries
  return (size_t)(s->h_K * n_tiles_of(s) * b + plan_ctas(s) + 32) * sizeof(int32_t);
}

extern "C" int fsa_build_inverse(const fsa_shape* s, const int32_t* idx, void* workspace,
                                 int32_t* offsets, int32_t* qlist, int32_t* work, int32_t* flags,
                                 void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t b = s->N / s->B_K, nt = n_tiles_of(s);
  if (s->N == 0) return FSA_OK;
  int32_t* hist = (int32_t*)workspace;
  const int64_t C = fsa::plan_chunk_tokens(*s), ctiles = C / fsa::kInvTile;
  dim3 grid((unsigned)nt, (unsigned)s->h_K);
  const size_t smem_bits = (size_t)b * 32;
  const bool bits = smem_bits <= 100 * 1024 && s->N * s->T < (1ll << 31);
  const size_t smem = bits ? smem_bits : (size_t)b * 8;
  FSA_REQUIRE(smem <= 200 * 1024, "build_inverse: b=%lld too large", (long long)b);
  if (bits) {
    cudaFuncSetAttribute(fsa::inverse_tile_bits_kernel<false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(fsa::inverse_tile_bits_kernel<true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    fsa::inverse_tile_bits_kernel<false><<<grid, fsa::kInvTile, smem, st>>>(
        idx, s->N, s->B_K, b, (int)s->T, hist, nullptr, nullptr, flags, nullptr, ctiles);
  } else {
    cudaFuncSetAttribute(fsa::inverse_tile_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(fsa::inverse_tile_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    fsa::inverse_tile_kernel<false><<<grid, fsa::kInvTile, smem, st>>>(
        idx, s->N, s->B_K, b, (int)s->T, hist, nullptr, nullptr, flags, nullptr, ctiles);
  }
  fsa::inverse_scan_tiles_kernel<<<(unsigned)((s->h_K * b + 255) / 256), 256, 0, st>>>(
      hist, offsets, s->h_K, nt, b);
  fsa::inverse_scan_blocks_kernel<<<(unsigned)s->h_K, 1024, 0, st>>>(offsets, b);
  int32_t* pos = work ? work + fsa::plan_pos_offset(*s) : nullptr;
  if (bits)
    fsa::inverse_tile_bits_kernel<true><<<grid, fsa::kInvTile, smem, st>>>(
        idx, s->N, s->B_K, b, (int)s->T, hist, offsets, qlist, nullptr, pos, ctiles);
  else
    fsa::inverse_tile_kernel<true><<<grid, fsa::kInvTile, smem, st>>>(
        idx, s->N, s->B_K, b, (int)s->T, hist, offsets, qlist, nullptr, pos, ctiles);
  if (work) {
    fsa::PlanArgs a{};
    a.offsets = offsets;
    a.hist = hist;
    a.work = work;
    a.item = work + fsa::plan_item_offset(*s);
    a.tbeg = work + fsa::plan_tbeg_offset(*s);
    a.tn = work + fsa::plan_tn_offset(*s);
    a.tki = work + fsa::plan_tki_offset(*s);
    a.carry = hist + s->h_K * nt * b;
    a.h_K = s->h_K;
    a.b = b;
    a.N = s->N;
    a.B_K = s->B_K;
    a.n_tiles = nt;
    a.C = C;
    a.nc = fsa::plan_nchunks(*s);
    a.nph = fsa::plan_tasks_per_head(*s);
    a.ntask = fsa::plan_ntask(*s);
    a.tpi = (int)fsa::plan_tpi(*s);
    const unsigned ctas = (unsigned)plan_ctas(s);
    fsa::work_plan_tasks_kernel<<<ctas, 1024, 0, st>>>(a);
    fsa::work_plan_carry_kernel<<<ctas, 1024, 0, st>>>(a);
  }
  FSA_LAUNCH_CHECK("build_inverse");
  return FSA_OK;
}
