// K3 top-k block selection (selection.py:78-102) and selection validation
// (selection.py:49-75).  Integer output, bit-exact with the reference:
//   * only causal blocks i <= t // B_K compete; the own block scores +inf;
//   * order = (score desc, block index asc); -inf and NaN are never selected;
//     -0.0 ties +0.0; a non-own +inf ties the own block and wins on index;
//   * output ascending, -1 padded.
// Scores are compared through a monotone integer key, so the comparison is
// exact for f32 and f64 inputs alike.
#include "common.cuh"

#include <cfloat>

namespace fsa {

struct SelKey {
  uint64_t sk;  // 0 = not selectable; larger = better
  uint32_t ix;  // block index; smaller wins ties
};

__device__ __forceinline__ uint64_t score_key(float f) {
  if (isnan(f) || f == -INFINITY) return 0;
  if (f == 0.0f) f = 0.0f;  // canonicalise -0.0
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? (uint64_t)(~u) : (uint64_t)(u | 0x80000000u);
}
__device__ __forceinline__ uint64_t score_key(double f) {
  if (isnan(f) || f == -(double)INFINITY) return 0;
  if (f == 0.0) f = 0.0;
  uint64_t u = (uint64_t)__double_as_longlong(f);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
template <typename S> __device__ __forceinline__ uint64_t own_key() {
  return score_key((S)INFINITY);
}

__device__ __forceinline__ bool better(uint64_t ask, uint32_t aix, uint64_t bsk, uint32_t bix) {
  return ask > bsk || (ask == bsk && aix < bix);
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// One warp per (kh, t) row, T <= 32.  Lane k holds the k-th best candidate;
// candidates stream in 32 at a time and only those beating the current T-th
// best are inserted (a handful per row after the first chunk).
template <typename S>
__global__ void topk_warp_kernel(const S* __restrict__ scores, int32_t* __restrict__ idx,
                                 int64_t rows, int64_t N, int64_t B_K, int64_t b, int T) {
  const int lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int64_t t = row % N;
  const int64_t own = t / B_K, ncand = own + 1;
  const S* sr = scores + row * b;
  uint64_t hsk = 0;
  uint32_t hix = 0xffffffffu;
  const uint64_t okey = own_key<S>();
  for (int64_t base = 0; base < ncand; base += 32) {
    const int64_t c = base + lane;
    uint64_t csk = 0;
    if (c < ncand) csk = (c == own) ? okey : score_key(sr[c]);
    const uint32_t cix = (uint32_t)c;
    uint64_t tsk = shfl64(hsk, T - 1);
    uint32_t tix = __shfl_sync(0xffffffffu, hix, T - 1);
    unsigned mask = __ballot_sync(0xffffffffu, csk != 0 && better(csk, cix, tsk, tix));
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const uint64_t isk = shfl64(csk, src);
      const uint32_t iix = __shfl_sync(0xffffffffu, cix, src);
      tsk = shfl64(hsk, T - 1);
      tix = __shfl_sync(0xffffffffu, hix, T - 1);
      if (!better(isk, iix, tsk, tix)) continue;  // warp-uniform
      const bool bt = lane < T && better(isk, iix, hsk, hix);
      const uint64_t psk = __shfl_up_sync(0xffffffffu, hsk, 1);
      const uint32_t pix = __shfl_up_sync(0xffffffffu, hix, 1);
      const bool pbt = __shfl_up_sync(0xffffffffu, (int)bt, 1) && lane > 0;
      if (bt) {
        hsk = pbt ? psk : isk;
        hix = pbt ? pix : iix;
      }
    }
  }
  // ascending block order, sentinels last: bitonic sort across the warp
  int v = (lane < T && hsk != 0) ? (int)hix : 0x7fffffff;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int p = __shfl_xor_sync(0xffffffffu, v, j);
      const bool up = (lane & k) == 0;
      const bool lo = (lane & j) == 0;
      v = (lo == up) ? min(v, p) : max(v, p);
    }
  }
  if (lane < T) idx[row * T + lane] = (v == 0x7fffffff) ? -1 : v;
}

// 32-bit monotone key of an f32 score (0 = not selectable: NaN / -inf).
__device__ __forceinline__ uint32_t score_key32(float f) {
  if (isnan(f) || f == -INFINITY) return 0u;
  if (f == 0.0f) f = 0.0f;  // canonicalise -0.0
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// f32 scores, T <= 32, any b: one warp per (kh, t) row, streaming over the
// row's causal candidates 32 at a time (few registers -> full occupancy):
//   pass 1: count the selectable keys and take each lane's maximum; with
//           <= T selectable the answer is all of them (index order);
//   theta = the T-th largest lane maximum, a lower bound of the T-th best
//           key (T lanes hold a key >= theta), so the answer lies among the
//           keys >= theta;
//   pass 2: collect those (typically ~T..2T) as (key, index) into shared
//           memory and sort them exactly (warp bitonic, key desc / index
//           asc): the first T are the selection -- exactly the first T of the
//           reference's stable (score desc, index asc) order;
//   fallback (> 64 candidates): an exact 4-pass 8-bit radix select of the
//           T-th key, then an index-order compaction.
// Output ascending, -1 padded (selection.py:78-102).
__global__ void __launch_bounds__(256) topk_stream_kernel(const float* __restrict__ scores,
                                                          int32_t* __restrict__ idx, int64_t rows,
                                                          int64_t N, int64_t B_K, int64_t b, int T) {
  __shared__ __align__(16) uint32_t smem_all[8][256];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t row = blockIdx.x * 8ll + wib;
  if (row >= rows) return;
  uint32_t* hist = smem_all[wib];
  // 32-bit index math (rows = h_K N < 2^31): a 64-bit divide is a long
  // emulated sequence, paid once per row
  const int64_t t = (int64_t)((uint32_t)row % (uint32_t)N);
  const int own = (int)((uint32_t)t / (uint32_t)B_K), ncand = own + 1;
  const float* sr = scores + row * b;
  int32_t* dst = idx + row * T;
  const unsigned lt = (1u << lane) - 1u;
  auto keyat = [&](int c) -> uint32_t {
    return c < ncand ? (c == own ? 0xFF800000u : score_key32(__ldg(sr + c))) : 0u;
  };
  // ---- pass 1
  int nsel = 0;
  uint32_t lm = 0u;
#pragma unroll 4
  for (int base = 0; base < ncand; base += 32) {
    const uint32_t k = keyat(base + lane);
    nsel += __popc(__ballot_sync(0xffffffffu, k != 0u));
    lm = max(lm, k);
  }
  if (nsel <= T) {
    int out = 0;
#pragma unroll 4
    for (int base = 0; base < ncand; base += 32) {
      const uint32_t k = keyat(base + lane);
      const unsigned m = __ballot_sync(0xffffffffu, k != 0u);
      if (k != 0u) dst[out + __popc(m & lt)] = base + lane;
      out += __popc(m);
    }
    if (lane >= out && lane < T) dst[lane] = -1;
    return;
  }
  // ---- theta: T-th largest lane maximum (warp bitonic, descending)
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, lm, j);
      const bool take_max = ((lane & j) == 0) == ((lane & kk) == 0);
      lm = take_max ? max(lm, y) : min(lm, y);
    }
  }
  const uint32_t theta = max(__shfl_sync(0xffffffffu, lm, T - 1), 1u);
  // ---- pass 2: candidates >= theta, packed so that larger = better
  unsigned long long* slots = reinterpret_cast<unsigned long long*>(hist);
  int cand = 0;
#pragma unroll 4
  for (int base = 0; base < ncand; base += 32) {
    const uint32_t k = keyat(base + lane);
    const bool c = k >= theta;
    const unsigned m = __ballot_sync(0xffffffffu, c);
    const int pos = cand + __popc(m & lt);
    if (c && pos < 64)
      slots[pos] = ((unsigned long long)k << 32) | (0xFFFFFFFFu - (uint32_t)(base + lane));
    cand += __popc(m);
  }
  __syncwarp();
  if (cand <= 64) {
    unsigned long long x0 = lane < cand ? slots[lane] : 0ull;
    unsigned long long x1 = lane + 32 < cand ? slots[lane + 32] : 0ull;
#pragma unroll
    for (int kk = 2; kk <= 64; kk <<= 1) {
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        if (j == 32) {  // partner in the same lane (only at kk = 64)
          const unsigned long long hi = max(x0, x1), lo = min(x0, x1);
          x0 = hi;
          x1 = lo;
        } else {
          const unsigned long long y0 = __shfl_xor_sync(0xffffffffu, x0, j);
          const unsigned long long y1 = __shfl_xor_sync(0xffffffffu, x1, j);
          const bool lower = (lane & j) == 0;
          const bool d0 = (lane & kk) == 0, d1 = ((lane + 32) & kk) == 0;
          x0 = (lower == d0) ? max(x0, y0) : min(x0, y0);
          x1 = (lower == d1) ? max(x1, y1) : min(x1, y1);
        }
      }
    }
    // the first T (T <= 32: lanes 0..T-1 of x0) are the selection; ascending index order
    int v = lane < T ? (int)(0xFFFFFFFFu - (uint32_t)x0) : 0x7fffffff;
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const int y = __shfl_xor_sync(0xffffffffu, v, j);
        const bool take_min = ((lane & j) == 0) == ((lane & kk) == 0);
        v = take_min ? min(v, y) : max(v, y);
      }
    }
    if (lane < T) dst[lane] = v;
    return;
  }
  __syncwarp();
  // ---- fallback: exact radix select of the T-th key (4 passes of 8 bits)
  uint32_t prefix = 0u, pmask = 0u;
  int need = T;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) hist[lane * 8 + q] = 0u;
    __syncwarp();
#pragma unroll 4
    for (int base = 0; base < ncand; base += 32) {
      const uint32_t k = keyat(base + lane);
      if (k != 0u && (k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t cnt[8], tot = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      cnt[q] = hist[255 - lane * 8 - q];
      tot += cnt[q];
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - tot;
    const unsigned hit = __ballot_sync(0xffffffffu, excl < (uint32_t)need && incl >= (uint32_t)need);
    const int src = __ffs(hit) - 1;
    uint32_t digit = 0u, above = 0u;
    if (lane == src) {
      uint32_t run = excl;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (run + cnt[q] >= (uint32_t)need) {
          digit = 255u - (uint32_t)(lane * 8 + q);
          above = run;
          break;
        }
        run += cnt[q];
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, src);
    above = __shfl_sync(0xffffffffu, above, src);
    need -= (int)above;
    prefix |= digit << shift;
    pmask |= 0xFFu << shift;
    __syncwarp();
  }
  const uint32_t kth = prefix;
  int taken_eq = 0, out = 0;
  for (int base = 0; base < ncand; base += 32) {
    const uint32_t k = keyat(base + lane);
    const bool eq = k == kth;
    const unsigned me = __ballot_sync(0xffffffffu, eq);
    const bool sel = k > kth || (eq && taken_eq + __popc(me & lt) < need);
    taken_eq += __popc(me);
    const unsigned ms = __ballot_sync(0xffffffffu, sel);
    if (sel) dst[out + __popc(ms & lt)] = base + lane;
    out += __popc(ms);
  }
}

// NCH > 0: the row's candidates stay in registers (NCH chunks of 128, b <= 128 NCH):
// one global read instead of two and no re-masking in pass 2.  NCH = 0: stream
// from global twice.  Pass 2 skips the warp scan of chunks without a candidate.
template <int NCH>
__global__ void __launch_bounds__(256) topk_stream4_kernel(const float* __restrict__ scores,
                                                          int32_t* __restrict__ idx, int64_t rows,
                                                          int64_t N, int64_t B_K, int64_t b, int T) {
  __shared__ __align__(16) uint32_t smem_all[8][256];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t row = blockIdx.x * 8ll + wib;
  if (row >= rows) return;
  uint32_t* hist = smem_all[wib];
  // 32-bit index math (rows = h_K N < 2^31): a 64-bit divide is a long
  // emulated sequence, paid once per row
  const int64_t t = (int64_t)((uint32_t)row % (uint32_t)N);
  const int own = (int)((uint32_t)t / (uint32_t)B_K), ncand = own + 1;
  const float* sr = scores + row * b;
  int32_t* dst = idx + row * T;
  const unsigned lt = (1u << lane) - 1u;
  auto keyat = [&](int c) -> uint32_t {
    return c < ncand ? (c == own ? 0xFF800000u : score_key32(__ldg(sr + c))) : 0u;
  };
  // ---- pass 1 (4 consecutive candidates per lane: one 16-byte load).
  // The passes compare floats directly -- the own block as +inf, NaN / -inf
  // unselectable (v > -inf is false for both), fmaxf ignores NaN, -0.0 == 0.0
  // -- and only the candidates get the 32-bit order key.
  const float4* sr4 = reinterpret_cast<const float4*>(sr);
  auto vals4 = [&](int base, float (&v4)[4]) {
    const int c0 = base + 4 * lane;
    const float4 f = c0 < ncand ? __ldg(sr4 + (c0 >> 2)) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    v4[0] = f.x; v4[1] = f.y; v4[2] = f.z; v4[3] = f.w;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (c0 + e >= ncand) v4[e] = -INFINITY;
      if (c0 + e == own) v4[e] = INFINITY;
    }
  };
  // chunks wholly below the own block need no masking: a plain 16-byte load
  auto raw4 = [&](int base, float (&v4)[4]) {
    const float4 f = __ldg(sr4 + (base >> 2) + lane);
    v4[0] = f.x; v4[1] = f.y; v4[2] = f.z; v4[3] = f.w;
  };
  auto load4 = [&](int base, float (&v4)[4]) {
    if (base + 128 <= own) raw4(base, v4);
    else vals4(base, v4);
  };
  auto excl_scan = [&](int v, int& total) {  // warp exclusive prefix sum
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    total = __shfl_sync(0xffffffffu, incl, 31);
    return incl - v;
  };
  // (no separate "<= T selectable" pass: then theta = 1 and every selectable
  // key is a candidate, which the rank path below returns in index order)
  float lmf = -INFINITY;
  float vr[NCH > 0 ? NCH : 1][4];
  if constexpr (NCH > 0) {
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      if (k * 128 < ncand) load4(k * 128, vr[k]);
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      if (k * 128 < ncand) {
#pragma unroll
        for (int e = 0; e < 4; ++e) lmf = fmaxf(lmf, vr[k][e]);
      }
  } else {
    int base = 0;
#pragma unroll 4
    for (; base + 128 <= own; base += 128) {
      float v4[4];
      raw4(base, v4);
      lmf = fmaxf(lmf, fmaxf(fmaxf(v4[0], v4[1]), fmaxf(v4[2], v4[3])));
    }
    for (; base < ncand; base += 128) {  // the chunk(s) holding the own block
      float v4[4];
      vals4(base, v4);
#pragma unroll
      for (int e = 0; e < 4; ++e) lmf = fmaxf(lmf, v4[e]);
    }
  }
  // ---- theta: T-th largest lane maximum (warp bitonic, descending)
  uint32_t lm = score_key32(lmf);  // 0 for an all-unselectable lane
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, lm, j);
      const bool take_max = ((lane & j) == 0) == ((lane & kk) == 0);
      lm = take_max ? max(lm, y) : min(lm, y);
    }
  }
  const uint32_t theta = max(__shfl_sync(0xffffffffu, lm, T - 1), 1u);
  // the float threshold with the same meaning (keys are monotone in the value)
  const float thf = theta == 1u ? -INFINITY
                                : __uint_as_float((theta & 0x80000000u) ? (theta & 0x7FFFFFFFu) : ~theta);
  // ---- pass 2: candidates >= theta, packed so that larger = better
  unsigned long long* slots = reinterpret_cast<unsigned long long*>(hist);
  int cand = 0;
  // v > -inf && v >= thf as one compare (NaN fails both forms)
  const float thf_eff = thf == -INFINITY ? -FLT_MAX : thf;
  auto chunk = [&](int base, const float (&v4)[4]) {
    bool c[4];
    int cnt = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      c[e] = v4[e] >= thf_eff;
      cnt += c[e];
    }
    if (!__any_sync(0xffffffffu, cnt > 0)) return;  // no candidate in this chunk
    int tot;
    int pos = cand + excl_scan(cnt, tot);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (c[e]) {
        if (pos < 64)
          slots[pos] = ((unsigned long long)score_key32(v4[e]) << 32) |
                       (0xFFFFFFFFu - (uint32_t)(base + 4 * lane + e));
        ++pos;
      }
    cand += tot;
  };
  if constexpr (NCH > 0) {
#pragma unroll
    for (int k = 0; k < NCH; ++k)
      if (k * 128 < ncand) chunk(k * 128, vr[k]);
  } else {  // the next chunk's load is in flight while this one is scanned
    float cur[4];
    load4(0, cur);
    for (int base = 0; base < ncand; base += 128) {
      float nxt[4];
      load4(base + 128, nxt);  // -inf past the row (no load)
      chunk(base, cur);
#pragma unroll
      for (int e = 0; e < 4; ++e) cur[e] = nxt[e];
    }
  }
  __syncwarp();
  if (cand <= 32) {
    // typical case (~T..2T candidates): lane L holds candidate L, and the
    // candidates sit in ascending index order.  Rank each by counting the
    // better ones (key desc, index asc -- the packed value is larger); the
    // T best, read in lane order, are the ascending selection.
    const unsigned long long x = lane < cand ? slots[lane] : 0ull;
    int rank = 0;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) rank += __shfl_sync(0xffffffffu, x, j) > x;
    const bool sel = lane < cand && rank < T;
    const unsigned ms = __ballot_sync(0xffffffffu, sel);
    if (sel) dst[__popc(ms & lt)] = (int)(0xFFFFFFFFu - (uint32_t)x);
    const int got = __popc(ms);
    if (lane >= got && lane < T) dst[lane] = -1;
    return;
  }
  if (cand <= 64) {
    unsigned long long x0 = lane < cand ? slots[lane] : 0ull;
    unsigned long long x1 = lane + 32 < cand ? slots[lane + 32] : 0ull;
#pragma unroll
    for (int kk = 2; kk <= 64; kk <<= 1) {
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        if (j == 32) {  // partner in the same lane (only at kk = 64)
          const unsigned long long hi = max(x0, x1), lo = min(x0, x1);
          x0 = hi;
          x1 = lo;
        } else {
          const unsigned long long y0 = __shfl_xor_sync(0xffffffffu, x0, j);
          const unsigned long long y1 = __shfl_xor_sync(0xffffffffu, x1, j);
          const bool lower = (lane & j) == 0;
          const bool d0 = (lane & kk) == 0, d1 = ((lane + 32) & kk) == 0;
          x0 = (lower == d0) ? max(x0, y0) : min(x0, y0);
          x1 = (lower == d1) ? max(x1, y1) : min(x1, y1);
        }
      }
    }
    // the first T (T <= 32: lanes 0..T-1 of x0) are the selection; ascending index order
    int v = lane < T ? (int)(0xFFFFFFFFu - (uint32_t)x0) : 0x7fffffff;
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const int y = __shfl_xor_sync(0xffffffffu, v, j);
        const bool take_min = ((lane & j) == 0) == ((lane & kk) == 0);
        v = take_min ? min(v, y) : max(v, y);
      }
    }
    if (lane < T) dst[lane] = v;
    return;
  }
  __syncwarp();
  // ---- fallback: exact radix select of the T-th key (4 passes of 8 bits)
  uint32_t prefix = 0u, pmask = 0u;
  int need = T;
#pragma unroll 1
  for (int shift = 24; shift >= 0; shift -= 8) {
#pragma unroll
    for (int q = 0; q < 8; ++q) hist[lane * 8 + q] = 0u;
    __syncwarp();
#pragma unroll 4
    for (int base = 0; base < ncand; base += 32) {
      const uint32_t k = keyat(base + lane);
      if (k != 0u && (k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t cnt[8], tot = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      cnt[q] = hist[255 - lane * 8 - q];
      tot += cnt[q];
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - tot;
    const unsigned hit = __ballot_sync(0xffffffffu, excl < (uint32_t)need && incl >= (uint32_t)need);
    const int src = __ffs(hit) - 1;
    uint32_t digit = 0u, above = 0u;
    if (lane == src) {
      uint32_t run = excl;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (run + cnt[q] >= (uint32_t)need) {
          digit = 255u - (uint32_t)(lane * 8 + q);
          above = run;
          break;
        }
        run += cnt[q];
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, src);
    above = __shfl_sync(0xffffffffu, above, src);
    need -= (int)above;
    prefix |= digit << shift;
    pmask |= 0xFFu << shift;
    __syncwarp();
  }
  const uint32_t kth = prefix;
  int taken_eq = 0, out = 0;
  for (int base = 0; base < ncand; base += 32) {
    const uint32_t k = keyat(base + lane);
    const bool eq = k == kth;
    const unsigned me = __ballot_sync(0xffffffffu, eq);
    const bool sel = k > kth || (eq && taken_eq + __popc(me & lt) < need);
    taken_eq += __popc(me);
    const unsigned ms = __ballot_sync(0xffffffffu, sel);
    if (sel) dst[out + __popc(ms & lt)] = base + lane;
    out += __popc(ms);
  }
}


// One CTA per row for T > 32: bitonic sort of all causal candidates in smem.
template <typename S>
__global__ void topk_block_kernel(const S* __restrict__ scores, int32_t* __restrict__ idx,
                                  int64_t N, int64_t B_K, int64_t b, int T, int P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* ksk = reinterpret_cast<uint64_t*>(smem_raw);
  uint32_t* kix = reinterpret_cast<uint32_t*>(ksk + P);
  const int64_t row = blockIdx.x;
  const int64_t t = row % N, own = t / B_K, ncand = own + 1;
  const S* sr = scores + row * b;
  const uint64_t okey = own_key<S>();
  for (int k = threadIdx.x; k < P; k += blockDim.x) {
    ksk[k] = (k < ncand) ? (k == own ? okey : score_key(sr[k])) : 0;
    kix[k] = (uint32_t)k;
  }
  __syncthreads();
  // sort descending under better()
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool desc = (i & k) == 0;
          const bool sw = desc ? better(ksk[l], kix[l], ksk[i], kix[i])
                               : better(ksk[i], kix[i], ksk[l], kix[l]);
          if (sw) {
            uint64_t a = ksk[i]; ksk[i] = ksk[l]; ksk[l] = a;
            uint32_t c = kix[i]; kix[i] = kix[l]; kix[l] = c;
          }
        }
      }
      __syncthreads();
    }
  }
  // keep the first T selectable entries, then sort those by index ascending
  int P2 = 1;
  while (P2 < T) P2 <<= 1;
  uint32_t* v = kix + P;  // reuse: [P2]
  for (int k = threadIdx.x; k < P2; k += blockDim.x)
    v[k] = (k < T && k < P && ksk[k] != 0) ? kix[k] : 0x7fffffffu;
  __syncthreads();
  for (int k = 2; k <= P2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool asc = (i & k) == 0;
          if ((v[i] > v[l]) == asc) {
            uint32_t a = v[i]; v[i] = v[l]; v[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int k = threadIdx.x; k < T; k += blockDim.x)
    idx[row * T + k] = (v[k] == 0x7fffffffu) ? -1 : (int32_t)v[k];
}

// validate_selection: one thread per row; flags OR-reduced per warp.
__global__ void validate_kernel(const int32_t* __restrict__ idx, int64_t rows, int64_t N,
                                int64_t B_K, int64_t b, int T, int32_t* flags) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int f = 0;
  if (row < rows) {
    const int64_t own = (row % N) / B_K;
    const int32_t* r = idx + row * T;
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
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) f |= __shfl_xor_sync(0xffffffffu, f, o);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

template <typename S>
int topk_impl(const fsa_shape* s, const void* scores, int32_t* idx, cudaStream_t st) {
  const int64_t b = s->N / s->B_K, rows = s->h_K * s->N;
  const int T = (int)s->T;
  if (rows == 0) return FSA_OK;
  if (sizeof(S) == 4 && T <= 32 && b % 4 == 0) {
    const unsigned grid = (unsigned)((rows + 7) / 8);
    const float* sc = (const float*)scores;
    if (b <= 512)
      topk_stream4_kernel<4><<<grid, 256, 0, st>>>(sc, idx, rows, s->N, s->B_K, b, T);
    else if (b <= 1024)
      topk_stream4_kernel<8><<<grid, 256, 0, st>>>(sc, idx, rows, s->N, s->B_K, b, T);
    else  // longer rows: 64+ registers of candidates cost more occupancy than the re-read
      topk_stream4_kernel<0><<<grid, 256, 0, st>>>(sc, idx, rows, s->N, s->B_K, b, T);
  } else if (sizeof(S) == 4 && T <= 32) {
    topk_stream_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>((const float*)scores, idx, rows,
                                                                  s->N, s->B_K, b, T);
  } else if (T <= 32) {
    const int warps = 8;
    topk_warp_kernel<S><<<(unsigned)((rows + warps - 1) / warps), warps * 32, 0, st>>>(
        (const S*)scores, idx, rows, s->N, s->B_K, b, T);
  } else {
    int P = 1;
    while (P < b) P <<= 1;
    int P2 = 1;
    while (P2 < T) P2 <<= 1;
    size_t smem = (size_t)P * 12 + (size_t)P2 * 4;
    FSA_REQUIRE(smem <= 200 * 1024, "select_topk: b=%lld too large for T>32 path", (long long)b);
    cudaFuncSetAttribute(topk_block_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    topk_block_kernel<S><<<(unsigned)rows, 256, smem, st>>>((const S*)scores, idx, s->N, s->B_K,
                                                            b, T, P);
  }
  FSA_LAUNCH_CHECK("select_topk");
  return FSA_OK;
}

}  // namespace fsa

extern "C" int fsa_select_topk(const fsa_shape* s, int score_dtype, const void* scores,
                               int32_t* idx, void* stream) {
  switch (score_dtype) {
    case FSA_DT_F32: return fsa::topk_impl<float>(s, scores, idx, (cudaStream_t)stream);
    case FSA_DT_F64: return fsa::topk_impl<double>(s, scores, idx, (cudaStream_t)stream);
    default: fsa::set_error("select_topk: scores must be f32 or f64"); return FSA_ERR_INVALID;
  }
}

extern "C" int fsa_validate_selection(const fsa_shape* s, const int32_t* idx, int32_t* flags,
                                      void* stream) {
  const int64_t rows = s->h_K * s->N;
  if (rows == 0) return FSA_OK;
  fsa::validate_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      idx, rows, s->N, s->B_K, s->N / s->B_K, (int)s->T, flags);
  FSA_LAUNCH_CHECK("validate_selection");
  return FSA_OK;
}
